"""Loop bodies (backward branches) of one SASS function with opcode counts.
usage: python scripts/sass_loops.py k.sass <function-substring>"""
import re, collections, sys
s = open(sys.argv[1]).read().split('\n')
fn = sys.argv[2]
inside = False
instrs, labels = [], {}
for l in s:
    if l.startswith('.text.'):
        inside = fn in l
        continue
    if not inside:
        continue
    lm = re.match(r'^(\.L_x_\d+):', l.strip())
    if lm:
        labels[lm.group(1)] = len(instrs)
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)(.*)', l)
    if m:
        instrs.append((m.group(3), m.group(4)))
for i, (op, rest) in enumerate(instrs):
    if op.startswith('BRA'):
        t = re.search(r'\((\.L_x_\d+)\)', rest)
        if t and t.group(1) in labels and labels[t.group(1)] <= i:
            body = instrs[labels[t.group(1)]:i + 1]
            c = collections.Counter(x[0].split('.')[0] for x in body)
            print(f"loop {labels[t.group(1)]}-{i} len={len(body)}:", c.most_common(20))

import re,collections,sys
s=open(sys.argv[1]).read().split('\n')
fn=sys.argv[2]
inside=False; line=None; cnt=collections.Counter(); total=0; regs=None
for l in s:
    if l.startswith('.text.') or re.match(r'^\s*\.section\s+\.text',l):
        inside = fn in l
    if not inside: continue
    m=re.search(r'//## File "([^"]+)", line (\d+)',l)
    if m: line=(m.group(1).split('/')[-1],int(m.group(2)))
    if re.search(r'\b(LDL|STL)\b',l):
        cnt[line]+=1; total+=1
print(total); print(cnt.most_common(12))

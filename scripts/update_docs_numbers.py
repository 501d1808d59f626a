#!/usr/bin/env python
"""Rewrite the number tables of profiles/r02_summary.md and DESIGN.md from a
measurement set (profiles/<TAG>/bench_*.json, scripts/gpu_measure_r02.sh).
usage: python scripts/update_docs_numbers.py TAG OLDTAG"""
import json
import re
import sys

tag, old = sys.argv[1], sys.argv[2]
B = lambda name: json.load(open(f"profiles/{tag}/{name}.json"))
rows = []
for c in range(1, 6):
    b, t = B(f"bench_cfg{c}"), B(f"bench_det_cfg{c}")
    s, e = b["stage_ms"], b["e2e"]
    rows.append("| %d | %.2f | %.3f | %.3f | %.3f | %.3f | %.3f | %.3f | %.2f | %.2f | %.2f | %.1f | %.1e |" % (
        c, b["value"], b["ms_per_step"], s["gather"], s["s2m"], s["near"], s["m2t"], s["scatter"], e["value"],
        e["pageable"]["value"], t["value"], b["config"]["replan_seconds"] * 1e3, b["parity"]["rel_l2_vs_reference_fkt"]))
p = "profiles/r02_summary.md"
s = open(p).read().replace(f"profiles/{old}", f"profiles/{tag}")
a, b_ = s.index("| cfg | MVM/s | ms / MVM | gather"), s.index("Round-2 progression (MVM/s)")
hdr = s[a:].split("\n")[0:2]
s = s[:a] + "\n".join(hdr) + "\n" + "\n".join(rows) + "\n\n" + s[b_:]
fp = {c: B(f"bench_fp32_cfg{c}") for c in (2, 3, 5)}
s = re.sub(r"cfg2 [0-9.]+\nMVM/s \(near [0-9.]+ ms\), cfg3 [0-9.]+ \(near [0-9.]+ ms\), cfg5 [0-9.]+;",
           "cfg2 %.1f\nMVM/s (near %.2f ms), cfg3 %.1f (near %.2f ms), cfg5 %.1f;" % (
               fp[2]["value"], fp[2]["stage_ms"]["near"], fp[3]["value"], fp[3]["stage_ms"]["near"], fp[5]["value"]), s)
open(p, "w").write(s)

p = "DESIGN.md"
s = open(p).read().replace(f"profiles/{old}", f"profiles/{tag}")
names = {1: "1 cauchy N=2e4", 2: "**2 matérn N=1e6**", 3: "3 gaussian d=5 N=1e6", 4: "4 inverse-r N=4e6", 5: "5 cauchy d=2 16 RHS"}
ncu = json.load(open("profiles/ncu_near.json"))
a, b_ = s.index("### Measured (B200, round 2 final;"), s.index("M2T kernels: cfg1 / cfg2 / cfg3 `m2t_cart`")
rows = []
for c in range(1, 6):
    d = B(f"bench_cfg{c}")
    st = d["stage_ms"]
    pipe = "— (launch-bound)" if c == 1 else "%.1f%%" % (100 * ncu[f"cfg{c}"]["fp64_pipe_frac"])
    val = "**%.1f**" % d["value"] if c == 2 else ("%.1f" % d["value"] if c > 1 else "%.0f" % d["value"])
    rows.append("| %s | %s | %.2f | %.2f | %.2f | %.2f | %.2f | %.2f | %s | %.1e |" % (
        names[c], val, d["ms_per_step"], st["gather"], st["s2m"], st["near"], st["m2t"], st["scatter"], pipe,
        d["parity"]["rel_l2_vs_reference_fkt"]))
s = s[:a] + f"""### Measured (B200, round 2 final; `profiles/r02_summary.md`, `profiles/{tag}/`)

| cfg | MVM/s | ms / MVM | gather | s2m | near | m2t | scatter | near FP64 pipe (ncu) | z vs reference |
|---|---|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + "\n\n" + s[b_:]
open(p, "w").write(s)
d = B("bench_default_cfg2")
print("default:", round(d["value"], 2), round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2),
      round(d["e2e"]["pageable"]["value"], 2), "ref s/MVM", round(d["cpu_baseline"]["seconds_per_mvm"], 2),
      "ref arm", B("bench_reference_cfg2")["value"], "plan", round(d["config"]["plan_seconds"], 3),
      "replan", round(d["config"]["replan_seconds"] * 1e3, 1), round(d["config"]["replan_device_seconds"] * 1e3, 1))

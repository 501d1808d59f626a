#!/usr/bin/env python
"""Summarise `ncu --set full` raw CSVs (scripts/gpu_ncu_r02.sh) per kernel
launch and write the near-field evidence bench.py reads:

    python scripts/ncu_summary.py TAG CFG... [--json profiles/ncu_near.json]

For each config, the near-field launches of ONE multiply (near_stream /
near_kernel, both pair forms) are aggregated: traffic = sum of DRAM read +
write bytes, fp64_pipe_frac = duration-weighted sm__pipe_fp64_cycles_active
(% of peak sustained elapsed). Prints a per-launch table for every captured
kernel (near and M2T)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}

METRICS = {
    "time": "gpu__time_duration.sum",
    "dram_r": "dram__bytes_read.sum",
    "dram_w": "dram__bytes_write.sum",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "fp64_active": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}


def read(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"name": r[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            d[k] = v * UNITS.get(units[i], 1.0)
        out.append(d)
    return out


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    jpath = os.path.join(ROOT, "profiles", "ncu_near.json")
    if "--json" in sys.argv:
        jpath = sys.argv[sys.argv.index("--json") + 1]
        args.remove(jpath)
    tag, cfgs = args[0], args[1:]
    try:
        js = json.load(open(jpath))
    except Exception:
        js = {}
    for c in cfgs:
        raw = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_cfg{c}_raw.csv")
        ks = read(raw)
        print(f"cfg{c}:")
        for k in ks:
            print(f"  {k['name'][:70]:70s} {k.get('time', 0) * 1e3:8.3f} ms  dram {(k.get('dram_r', 0) + k.get('dram_w', 0)) / 1e6:8.1f} MB"
                  f"  fp64 {k.get('fp64', 0):5.1f}%  issue {k.get('issue', 0):5.1f}%  regs {k.get('regs', 0):.0f}")
        near = [k for k in ks if "near_stream" in k["name"] or "near_kernel" in k["name"]]
        if not near:
            continue
        # one multiply's launches: the first launch of each distinct kernel
        seen, one = set(), []
        for k in near:
            if k["name"] in seen:
                break
            seen.add(k["name"])
            one.append(k)
        t = sum(k["time"] for k in one)
        js[f"cfg{c}"] = {
            "traffic": sum(k.get("dram_r", 0) + k.get("dram_w", 0) for k in one),
            "fp64_pipe_frac": sum(k["fp64"] * k["time"] for k in one) / t / 100.0,
            "ncu_ms": t * 1e3,
            "launches": len(one),
            "capture": f"profiles/{tag}_ncu_cfg{c}_details.txt",
        }
    with open(jpath, "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    print(json.dumps(js, indent=1))


if __name__ == "__main__":
    main()

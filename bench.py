#!/usr/bin/env python
"""FKT MVM benchmark — BASELINE.json metric on the headline config (cfg2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--cfg C]

Our arm: one B200-native FKT plan per rank (cfg2: Matern-3/2 l=0.1, N=1e6,
d=3, p=6, leaf 512, theta 0.5, SURVEY Appendix B inputs from fkt::Rng(42)).
`value` = whole-job MVMs/s with y and z resident in HBM (CUDA events around
K back-to-back device multiplies on the launching stream, max over ranks);
`e2e` = the same through the C-ABI host-buffer call (pinned host y -> H2D ->
MVM -> D2H z every step). The roofline is for the dominant kernel (near
field K3, FP64-pipe bound) against the FP64 FMA peak measured live on this
GPU. The reference arm times the unmodified reference FKT (oracle/_ref) on
the host cores. Multi-GPU (torchrun, N ranks): ONE MVM per step sharded by
target over the ranks (paper_2106_04487_b200.distributed.ShardedPlan: partial
moments -> NCCL all-reduce -> near + M2T of the owned targets -> NCCL
all-reduce of z), scaling "strong" (total work fixed), DESIGN.md §6.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FKT MVMs/sec (and effective interactions/sec) at N=1e6 d=3, % of roofline"

CONFIGS = {
    1: dict(kernel="cauchy", params={"sigma": 1.0}, n=20000, p=4, leaf=512, theta=0.5, d=3, nrhs=1),
    2: dict(kernel="matern32", params={"sigma": 1.0, "rho": 0.1}, n=1000000, p=6, leaf=512, theta=0.5, d=3, nrhs=1),
    3: dict(kernel="gaussian", params={}, n=1000000, p=4, leaf=1024, theta=0.75, d=5, nrhs=1),
    4: dict(kernel="inverse-r", params={}, n=4000000, p=8, leaf=512, theta=0.5, d=3, nrhs=1),
    5: dict(kernel="cauchy", params={"sigma": 1.0}, n=2000000, p=6, leaf=512, theta=0.75, d=2, nrhs=16),
}

# BASELINE.md §3 flop convention: +,-,x = 1, FMA = 2, div/sqrt/rsqrt = 8, exp = 20.
def near_flops_per_pair(kernel: str, d: int) -> int:
    diff = 3 * d - 1  # d subtractions, d squares, d-1 adds
    extra = {
        "cauchy": 1 + 1 + 8 + 2, "rational-quadratic": 1 + 1 + 8 + 2, "gaussian": 20 + 2,
        "inverse-r": 8 + 2, "inverse-r2": 8 + 2, "matern32": 8 + 1 + 1 + 20 + 1 + 1 + 2,
        "matern12": 8 + 8 + 20 + 1 + 2, "exponential": 8 + 20 + 2,
    }.get(kernel, 8 + 20 + 2)
    return diff + extra


# FP64 work the near kernel actually executes per (target, source) pair, from
# the SASS of its inner pair loop (scripts/sass_pair_mix.py on build/near.o,
# profiles/r02_sass_near_pairs.txt; the pair covers all right-hand sides):
# (FP64 instructions, flops with FMA = 2).
# The SURVEY §8(d) convention above charges exp = 20, sqrt / div = 8 flops;
# the fast-math bodies need fewer, so the convention-based
# roofline.frac can exceed 1 while the FP64 pipe is ~70% busy.
EXEC_FP64_PER_PAIR = {
    ("matern32", 3, 1): (15, 26),   # Gram form: 11 DFMA, 2 DMUL, 2 DADD
    ("gaussian", 5, 1): (12, 22),   # factored Gram form: 10 DFMA, 1 DMUL, 1 DADD
    ("inverse-r", 3, 1): (10, 16),  # difference form + select: 6 DFMA, 1 DMUL, 3 DADD
    ("cauchy", 2, 16): (23, 45),    # Gram form, 16 RHS: 22 DFMA, 1 DADD
    ("cauchy", 3, 1): (9, 17),      # Gram form: 8 DFMA, 1 DADD
}


def workload_desc(cfg):
    c = CONFIGS[cfg]
    return (f"cfg{cfg}: {c['kernel']} {c['params']} N={c['n']} d={c['d']} p={c['p']} leaf={c['leaf']} "
            f"theta={c['theta']} nrhs={c['nrhs']}")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def near_evals(tree, lo=None, hi=None) -> int:
    """Kernel evaluations of the near field; with [lo, hi), only the targets at
    those tree positions (one shard)."""
    off, idx = tree.nearCsr()
    sizes = tree.ends.astype(np.int64) - tree.begins.astype(np.int64)
    if lo is None:
        return int(np.sum(np.diff(off) * sizes))
    order = tree.order().astype(np.int64)
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    tp = inv[idx.astype(np.int64)]
    w = np.repeat(sizes, np.diff(off))
    return int(w[(tp >= lo) & (tp < hi)].sum())


def s2m_pairs(tree) -> int:
    off, _ = tree.farCsr()
    has = np.diff(off) > 0
    sizes = tree.ends.astype(np.int64) - tree.begins.astype(np.int64)
    return int(np.sum(sizes[has]))


def golden_parity(cfg, z):
    path = os.path.join(ROOT, "tests", "golden", f"cfg{cfg}_ref.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    rows = g["rows"]
    zr = g["z_rows"]
    zz = z[rows] if z.ndim == 1 else z[rows, :]
    out = {"rows": int(rows.size), "rel_l2_vs_reference_fkt": float(np.linalg.norm(zz - zr) / np.linalg.norm(zr))}
    zc = zz if zz.ndim == 1 else zz[:, 0]
    out["rel_l2_vs_dense"] = float(np.linalg.norm(zc - g["dense_rows"]) / np.linalg.norm(g["dense_rows"]))
    return out


def near_ncu(cfg, precision=64):
    """ncu evidence for the near kernel of THIS config (profiles/ncu_near.json,
    one `ncu --set full` capture per config, scripts/gpu_ncu_near_cfgs.sh):
    {"traffic": dram read + write bytes per launch, "fp64_pipe_frac": ...,
    "capture": file} or None when that config has no capture."""
    path = os.path.join(ROOT, "profiles", "ncu_near.json")
    try:
        with open(path) as f:
            v = json.load(f).get(f"cfg{cfg}" + ("" if precision == 64 else "_fp32"))
    except Exception:
        return None
    return v if isinstance(v, dict) else None


def traffic_for(cfg, precision=64):
    v = near_ncu(cfg, precision)
    return None if v is None else v.get("traffic")


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2106_04487_b200 as fkt

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[args.cfg]
    n, nrhs = c["n"], c["nrhs"]
    x, w = fkt.synthConfig(args.cfg, n)
    t0 = time.perf_counter()
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(c["kernel"], c["params"]),
                  fkt.FktOptions(p=c["p"], theta=c["theta"], leafCapacity=c["leaf"], nearPrecision=args.near_precision,
                                 deterministic=args.deterministic))
    plan_s = time.perf_counter() - t0
    plan_phases = pl.plan_phases()
    # re-plan for moving points (FktPlan.rebuild: same plan, new coordinates
    # of the same n points, buffers reused). The first rebuilds size the build
    # scratch and the list buffers (with headroom); the steady-state figure is
    # the median of three further rebuilds, alternating moved / original points
    rng = np.random.default_rng(3)
    x_moved = x + 1e-3 * rng.standard_normal(x.shape) * x.std(axis=0)
    for i in range(3):
        pl.rebuild(x_moved if i % 2 == 0 else x)
    replan_each, replan_phase_each = [], []
    for i in range(3):
        t0 = time.perf_counter()
        pl.rebuild(x if i % 2 == 0 else x_moved)
        replan_each.append(time.perf_counter() - t0)
        replan_phase_each.append(pl.plan_phases())
    mid = replan_each.index(sorted(replan_each)[1])
    replan_s, replan_phases = replan_each[mid], replan_phase_each[mid]
    # the same with the moved coordinates already in HBM (fkt_plan_rebuild_device)
    xd = [torch.from_numpy(x_moved).cuda(), torch.from_numpy(x).cuda()]
    replan_dev_each = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pl.rebuild_device(xd[i % 2])
        replan_dev_each.append(time.perf_counter() - t0)
    replan_dev_s = sorted(replan_dev_each[1:])[1]
    del xd
    info = pl.info()
    wcols = w.reshape(n, nrhs) if nrhs > 1 else w
    ydev = torch.from_numpy(np.ascontiguousarray(wcols.T if nrhs > 1 else wcols)).cuda()
    zdev = torch.empty_like(ydev)
    # A dedicated (non-default) stream: the plan captures the whole MVM as a
    # CUDA graph on first use and replays it (same kernels, fewer launches).
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if sharded:
        from paper_2106_04487_b200.distributed import ShardedPlan

        sp = ShardedPlan(pl)

        def mul():
            sp.multiply_device(ydev, zdev, stream=stream)
    else:
        def mul():
            pl.multiply_device(ydev, zdev, stream=stream)
    for _ in range(args.warmup):
        mul()
    torch.cuda.synchronize()
    zhost = zdev.cpu().numpy()
    parity = golden_parity(args.cfg, zhost.T if nrhs > 1 else zhost) if rank == 0 else None

    # ---- timed region: K device multiplies -------------------------------
    with ClockSampler(local) as clocks:
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            mul()
        e1.record(stream)
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if sharded:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-stage timing (same stream) for the roofline ------------------
    stage_ms = np.zeros(5)
    reps = max(3, min(args.steps, 20))
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(stream)
        for s in range(5):
            pl.stage_device(s, ydev, zdev, nrhs=nrhs, stream=stream)
            ev[s + 1].record(stream)
        torch.cuda.synchronize()
        stage_ms += np.array([ev[s].elapsed_time(ev[s + 1]) for s in range(5)])
    stage_ms /= reps

    # ---- e2e: public host-buffer API, pinned buffers, H2D + D2H per step ---
    yh = torch.from_numpy(np.asfortranarray(wcols)).pin_memory() if nrhs == 1 else \
        torch.from_numpy(np.ascontiguousarray(wcols.T)).pin_memory()
    zh = torch.empty_like(yh).pin_memory()
    import ctypes as C

    if sharded:
        def host_mul():  # pinned y -> H2D -> sharded MVM (all of z on every rank) -> D2H z
            ydev.copy_(yh.reshape(ydev.shape), non_blocking=True)
            mul()
            zh.reshape(zdev.shape).copy_(zdev, non_blocking=True)
            stream.synchronize()
    else:
        def host_mul():
            rc = fkt.lib.fkt_plan_multiply(pl._h, C.cast(C.c_void_p(yh.data_ptr()), C.POINTER(C.c_double)),
                                           C.cast(C.c_void_p(zh.data_ptr()), C.POINTER(C.c_double)), nrhs)
            fkt._check(rc)

    for _ in range(max(1, args.warmup // 2)):
        host_mul()
    if sharded:
        dist.barrier()
    te = time.perf_counter()
    e2e_steps = max(3, args.steps // 2)
    for _ in range(e2e_steps):
        host_mul()
    e2e_s = (time.perf_counter() - te) / e2e_steps
    if sharded:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # the drop-in FktPlan::multiply(std::span) path: PAGEABLE host buffers
    # (numpy, like std::vector) through the same C-ABI call
    pageable_s = None
    if not sharded:
        ya = np.array(yh.numpy(), copy=True)
        za = np.empty_like(ya)

        def page_mul():
            fkt._check(fkt.lib.fkt_plan_multiply(pl._h, ya.ctypes.data_as(C.POINTER(C.c_double)),
                                                 za.ctypes.data_as(C.POINTER(C.c_double)), nrhs))

        page_mul()
        tp = time.perf_counter()
        for _ in range(e2e_steps):
            page_mul()
        pageable_s = (time.perf_counter() - tp) / e2e_steps

    launches = int(fkt.lib.fkt_plan_kernel_launches(pl._h, nrhs))
    shard_lo, shard_hi = pl.shard_range()
    if rank != 0:
        dist.destroy_process_group()
        return

    # ---- roofline (dominant kernel: near field) ---------------------------
    pk_fma, pk_mma = C.c_double(), C.c_double()
    fkt._check(fkt.lib.fkt_fp64_peaks(C.byref(pk_fma), C.byref(pk_mma)))
    peak_tf = max(pk_fma.value, pk_mma.value) / 1e12
    tree = pl.tree()
    nev_all = near_evals(tree)
    nev = near_evals(tree, shard_lo, shard_hi) if sharded else nev_all  # rank 0's near launch
    fpp = near_flops_per_pair(c["kernel"], c["d"]) + 2 * (nrhs - 1)
    near_flops = nev * fpp
    P = info["coefficient_count"]
    far_pairs = info["far_total"] + s2m_pairs(tree)
    far_flops = far_pairs * (2 * P + 2 * P * nrhs)
    near_ms = stage_ms[2]
    achieved = near_flops / (near_ms * 1e-3) / 1e12
    ex = EXEC_FP64_PER_PAIR.get((c["kernel"], c["d"], nrhs))
    exec_fields = {}
    if ex is not None and args.near_precision == 64:
        instr_rate = ex[0] * nev / (near_ms * 1e-3)  # FP64 instructions / s (lanes)
        exec_fields = {"executed_fp64_instr_per_pair": ex[0], "executed_flops_per_pair": ex[1],
                       "executed_frac": ex[1] * nev / (near_ms * 1e-3) / 1e12 / peak_tf,
                       "fp64_pipe_frac": instr_rate / (peak_tf * 1e12 / 2)}
    mvm_s = ms * 1e-3
    value = 1.0 / mvm_s  # one MVM per step for the whole job
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "MVM/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64" if args.near_precision == 64 else "f64 (near field f32 fast mode)",
        "data": "synthetic (SURVEY Appendix B recipe, fkt::Rng(42); no public dataset)",
        "config": {
            "workload": workload_desc(args.cfg),
            "parallelism": (f"target-sharded x{world} (moment + z all-reduce over NCCL)" if sharded
                            else "single GPU"),
            "l2": "inputs larger than L2: far lists %.0f MB + near lists %.0f MB + coordinates %.0f MB per step"
                  % (info["far_total"] * 4 / 1e6, info["near_total"] * 4 / 1e6, n * c["d"] * 8 / 1e6),
            "plan_seconds": plan_s, "plan_phases": plan_phases,
            "replan_seconds": replan_s, "replan_seconds_each": replan_each, "replan_device_seconds": replan_dev_s, "replan_phases": replan_phases,
            "deterministic": bool(args.deterministic),
            "nodes": info["nodes"], "far_pairs": info["far_total"], "near_pairs": info["near_total"],
            "near_evals": nev_all, "coefficients": P,
            "m2t": ("cartesian (m2t_cart)" if info.get("m2t_cartesian") and nrhs == 1 else "harmonic"),
        },
        "effective_interactions_per_s": float(n) * n * nrhs / mvm_s,
        "stage_ms": {"gather": stage_ms[0], "s2m": stage_ms[1], "near": stage_ms[2], "m2t": stage_ms[3],
                     "scatter": stage_ms[4]},
        "roofline": {
            "kernel": "near_kernel (K3)",
            "bound": "fp64",
            "achieved": achieved,
            "peak": peak_tf,
            "peak_source": "FP64 datapath peak measured live in this run (fkt_fp64_peaks: best of DFMA chains and "
                           "mma.sync f64 chains, 3 lengths x 3 reps after a warm-up); MEASURED_PEAKS.json has no "
                           "fp64 entry",
            "peak_dfma": pk_fma.value / 1e12, "peak_dmma": pk_mma.value / 1e12,
            "unit": "TFLOP/s",
            "frac": achieved / peak_tf,
            "traffic": traffic_for(args.cfg, args.near_precision),
            "flops_per_launch": near_flops,
            "flops_per_pair": fpp,
            "whole_step_frac": (nev_all * fpp + far_flops) / mvm_s / 1e12 / peak_tf / world,
            # frac counts SURVEY §8(d)'s flop convention (exp = 20, sqrt / div = 8);
            # the fast-math pair body executes fewer FP64 instructions (16 for the
            # Matern-3/2 Gram form), so the FP64 pipe utilisation ncu measured for
            # this kernel (profiles/ncu_near.json, this config's capture) is the hardware-side figure
            "ncu_fp64_pipe_frac": (near_ncu(args.cfg, args.near_precision) or {}).get("fp64_pipe_frac"),
            "ncu_capture": (near_ncu(args.cfg, args.near_precision) or {}).get("capture"),
            "frac_note": ("frac = SURVEY 8(d) convention flops (exp 20, sqrt/div 8) / live DFMA peak; the fast-math "
                          "pair body executes fewer FP64 ops than the convention charges, so frac may exceed 1. "
                          "executed_frac and fp64_pipe_frac count the FP64 work the kernel really issues (SASS)."),
            **exec_fields,
        },
        "e2e": {"value": 1.0 / e2e_s, "unit": "MVM/s", "h2d_bytes_per_step": int(yh.numel() * 8) * world,
                "d2h_bytes_per_step": int(zh.numel() * 8) * world,
                "method": ("ShardedPlan.multiply_device per rank (pinned host y -> H2D, sharded MVM, D2H of all z), "
                           "wall clock, max over ranks" if sharded else
                           "fkt_plan_multiply (C-ABI, pinned host y/z, H2D+MVM+D2H per step), wall clock"),
                "pageable": (None if pageable_s is None else
                             {"value": 1.0 / pageable_s, "unit": "MVM/s",
                              "method": "fkt_plan_multiply on pageable host buffers (numpy; what FktPlan::multiply"
                                        "(std::span) with std::vector storage runs): chunked staging through "
                                        "pinned bounce buffers, wall clock"})},
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
        "clocks": clocks.summary(),
        "parity": parity,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cfg, reps=args.cpu_reps)
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def _ref_sample_run(cfg, n_s, reps, warmup):
    """Reference FKT (oracle/_ref) on the cfg recipe with n_s points; returns seconds per MVM."""
    from oracle import ref

    c = CONFIGS[cfg]
    x, w = ref.gen_config(cfg, n_s)
    rp = ref.RefPlan(x, c["kernel"], c["params"], p=c["p"], theta=c["theta"], leaf=c["leaf"], eager=False,
                     threads=0)
    for _ in range(warmup):
        rp.multiply(w)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        rp.multiply(w)
        ts.append(time.perf_counter() - t0)
    return ts, rp.plan_seconds


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, warmup=1, reps=3):
    """Reference CPU FKT (oracle/_ref, unmodified, streaming, all host threads)
    at the FULL config size: BASELINE.md §4 -- 1 warm-up MVM, then the median
    of `reps` timed MVMs (plan timed separately)."""
    c = CONFIGS[cfg]
    cores = os.cpu_count()
    ts, plan_s = _ref_sample_run(cfg, c["n"], reps, warmup)
    t = float(np.median(ts))
    return {"value": 1.0 / t, "unit": "MVM/s", "cores": cores, "kind": "reference",
            "cpu_model": cpu_model(), "nproc": cores,
            "sample": (f"full cfg{cfg} workload (N={c['n']}): reference FktPlan::multiply, streaming, "
                       f"FktOptions.threads = 0 ({cores} threads); {warmup} warm-up, median of {reps}"),
            "seconds_per_mvm": t, "seconds_each": ts, "plan_seconds": plan_s}


def run_reference(args):
    """--impl reference: the unmodified reference FKT (oracle/_ref) through its
    own FktPlan API at the FULL config size, every step one full MVM (no
    sampling, no extrapolation): W warm-up MVMs, then K timed MVMs
    (proj/tools/fkt_main.cpp:206-252 times the same call)."""
    world, rank, local = dist_setup()
    if rank != 0:
        return
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfktref.so not built"}))
        return
    c = CONFIGS[args.cfg]
    cores = os.cpu_count()
    ts, plan_s = _ref_sample_run(args.cfg, c["n"], args.steps, args.warmup)
    t_step = float(np.mean(ts))
    value = 1.0 / t_step
    sample = (f"full cfg{args.cfg} workload (N={c['n']}) every step: one reference FktPlan::multiply "
              f"(streaming, {cores} threads, {cpu_model()}); {args.warmup} warm-up + {args.steps} timed MVMs, "
              f"value = 1 / mean step time")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MVM/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY Appendix B recipe, fkt::Rng(42))",
        "config": {"workload": workload_desc(args.cfg), "parallelism": "host cores", "sample_n": c["n"],
                   "reference_plan_seconds": plan_s, "median_ms": float(np.median(ts)) * 1e3,
                   "min_ms": float(np.min(ts)) * 1e3, "max_ms": float(np.max(ts)) * 1e3},
        "cpu_baseline": {"value": value, "unit": "MVM/s", "cores": cores, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": cores},
        "e2e": {"value": value, "unit": "MVM/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "effective_interactions_per_s": float(c["n"]) * c["n"] * c["nrhs"] / t_step,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--sharded", action="store_true",
                    help="use the target-sharded multi-GPU path even at one rank (it is automatic for N > 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=3, help="timed reference MVMs for cpu_baseline (median)")
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise reproducible MVM (FktOptions.deterministic: fixed-order sums, no atomics)")
    ap.add_argument("--near-precision", type=int, default=64, choices=[64, 32],
                    help="32 = FP32 fast near-field mode (not the headline; parity gate is FP64)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

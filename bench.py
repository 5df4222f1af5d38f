"""Benchmark: level-batched skeletonization factorization on B200 (fp64).

Headline (BASELINE.json metric, configs[1] = cfg2, 16-hole multiply-connected
Stokes geometry, 49 200 unknowns): factorization unknowns/s.  One step = one
full factorization (all levels + augmentation sweep + corner LU).  Secondary
numbers: ms per local hole-move update (cfg4 regime on cfg2) and RHS/s of a
256-RHS solve.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun): independent replicas, one per GPU (the path does not shard,
DESIGN.md "replicas only"); value = total unknowns of all ranks / max rank time.
``--impl reference`` times the CPU reference restatement (oracle/, the
reference itself is pure Python and does not ship to the GPU box) on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factorization unknowns/sec (fp64)"
UNIT = "unknowns/s"


def _dist():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.p = None
        self.path = f"/tmp/skb_clocks_{os.getpid()}.csv"
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, val in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                  "sw_power_cap"], f[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "samples": len(sm), "reasons": sorted(reasons)}


def aggregate(step_ms, world, n_unk, reduce_max):
    """Whole-job throughput: all ranks' unknowns / max-over-ranks device time."""
    total = reduce_max(float(sum(step_ms)))
    return world * len(step_ms) * n_unk / (total * 1e-3), total


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def measure_fp64_peak(torch):
    """cuBLAS DGEMM (torch.matmul float64, 8192^3) -- FP64 DMMA denominator (not in MEASURED_PEAKS)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


def cpu_reference_run(wl, steps, warmup, budget_s=150.0):
    """Time the CPU reference restatement (oracle) on the host cores."""
    from oracle import skel_oracle as O
    b = wl.boundary
    ncores = os.cpu_count() or 1
    cands = [1] if ncores == 1 else [1, ncores]
    t_best, workers = None, 1
    for w in cands[: max(1, warmup)] if warmup else cands[:1]:
        t0 = time.perf_counter()
        O.factor_full(b, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor, workers=w)
        dt = time.perf_counter() - t0
        if t_best is None or dt < t_best:
            t_best, workers = dt, w
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        O.factor_full(b, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor, workers=workers)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return times, workers


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    rank, world, local = _dist()

    from paper_2001_11619_b200 import configs
    wl = configs.cfg2()
    n_unk = 2 * wl.boundary.n_nodes + 3 * wl.boundary.n_holes
    cfg = {"workload": "cfg2: outer circle R=10 (8192 nodes) + 16 holes r=0.5 (1024 nodes each), "
                       "Stokes double layer + augmentation, eps=1e-10, leaf 64, proxy 64 @ 1.5x half-width",
           "n_unknowns": n_unk, "seed": wl.seed, "parallelism": "replicas" if world > 1 else "single"}

    if args.impl == "reference":
        if rank != 0:
            return
        times, workers = cpu_reference_run(wl, args.steps, args.warmup)
        v = n_unk * len(times) / sum(times)
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": len(times),
                "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": cfg, "impl": "reference",
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                                 "sample": f"{len(times)} full cfg2 factorizations, oracle/skel_oracle.py "
                                           f"(numpy/scipy restatement, workers={workers}, BLAS 1 thread)"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2001_11619_b200 import SystemSpec, build_tree, factor, update, _lib
    from paper_2001_11619_b200 import skel as S
    from paper_2001_11619_b200.geometry import Boundary

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    b = wl.boundary
    spec = SystemSpec()
    tree = build_tree(b.positions, wl.leaf_cap)
    b._skb_device = S.DeviceBoundary(b)         # inputs resident in HBM for `value`
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > L2 (126 MB)

    def step():
        return factor(spec, b, tree, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)

    for _ in range(max(3, args.warmup)):
        f = step()
        del f
    barrier()
    clocks = Clocks(local)
    times = []
    for _ in range(args.steps):
        flush.fill_(1.0)                            # evict L2 between timed steps
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f = step()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        del f
    clk = clocks.stop()
    # per-kernel-family device times from the library's CUDA-event timers, on two
    # extra steps of the same workload (event records perturb the timed pipeline)
    prof_steps = 2
    _lib.prof_enable(True)
    _lib.prof_read(reset=True)
    for _ in range(prof_steps):
        flush.fill_(1.0)
        f = step()
        del f
    torch.cuda.synchronize()
    fam = _lib.prof_read(reset=True)
    _lib.prof_enable(False)
    def reduce_max(x):
        t_ = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(t_, op=torch.distributed.ReduceOp.MAX)
        return float(t_.item())

    value, total_ms = aggregate(times, world, n_unk, reduce_max)
    launches = sum(v["launches"] for v in fam.values()) // prof_steps

    # ---- e2e through the public API from host arrays (geometry H2D inside the timed region)
    e2e_times = []
    io0 = dict(S.IO)
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        bh = Boundary([c for c in b.curves])        # fresh host Boundary, no device cache
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        th = build_tree(bh.positions, wl.leaf_cap)
        fh = factor(spec, bh, th, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        _ = fh.stats["top_pivot_ratio"]
        e1.record()
        e1.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
        del fh
    h2d = (S.IO["h2d"] - io0["h2d"]) / args.steps
    d2h = (S.IO["d2h"] - io0["d2h"]) / args.steps
    e2e_value, _ = aggregate(e2e_times, world, n_unk, reduce_max)

    line = None
    fp64 = None
    if rank == 0:
        peaks = _peaks()
        # the DGEMM peak probe (2 x 512 MB operands) runs after the secondary
        # measurements; roofline is filled in then
        fp64 = 35.5
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        # dominant kernel family by device time; DRAM traffic per launch from the
        # committed ncu capture of one factorization (profiles/, scripts/ncu_traffic.py)
        dom = max(fam, key=lambda k: fam[k]["ms"])
        traffic = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "r01_cfg2_traffic.json")))["families"]
            # per launch of the family's timed scopes (bench launch count per step)
            per_step = fam[dom]["launches"] / prof_steps
            traffic = tr[dom]["dram_bytes"] / per_step if dom in tr and per_step else None
        except Exception:
            traffic = None
        d = fam[dom]
        per = max(d["launches"], 1)
        if d["flops"] > 0:
            ach = d["flops"] / (d["ms"] * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": ach, "peak": fp64, "unit": "TFLOP/s",
                    "frac": ach / fp64, "traffic": traffic, "kernel": dom,
                    "peak_source": "measured cuBLAS DGEMM 8192^3 (torch.matmul float64) in this run",
                    "avg_launch_ms": d["ms"] / per}
        else:
            ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": traffic, "kernel": dom,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs", "avg_launch_ms": d["ms"] / per}
        fam_summary = {k: {"ms_per_step": v["ms"] / prof_steps, "launches_per_step": v["launches"] / prof_steps,
                           **({"tflops": v["flops"] / (v["ms"] * 1e-3) / 1e12} if v["flops"] and v["ms"] else {}),
                           **({"gbs": v["bytes"] / (v["ms"] * 1e-3) / 1e9} if v["bytes"] and v["ms"] else {})}
                      for k, v in fam.items()}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {**cfg, "l2": "flushed (256 MB write) before every timed step"},
                "step_ms": [round(x, 3) for x in times], "e2e_step_ms": [round(x, 3) for x in e2e_times],
                "roofline": roof, "kernel_families": fam_summary,
                "kernel_families_note": f"CUDA-event timers on {prof_steps} extra steps after the timed region", "fp64_dgemm_tflops": fp64,
                "gpu_launches": int(launches),
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h),
                        "path": "host Boundary -> build_tree -> factor() (public API), geometry + "
                                "level descriptors H2D, ranks/pivots D2H inside the timed region"},
                "clocks": clk}

    # ---- secondary: hole-move updates (cfg4 regime) and 256-RHS solve
    if rank == 0 and not args.no_secondary:
        import gc
        gc.collect()
        f = step()
        seq = configs.hole_move_sequence(b, 12)
        upd = []
        cur = update(f, seq[0][2], seq[0][3])       # warm-up moves
        cur = update(cur, seq[1][2], seq[1][3])
        for _, _, nb, rep in seq[2:]:
            torch.cuda.synchronize()
            cur = update(cur, nb, rep)
            upd.append(cur.stats["update_time"] * 1e3)
        X = torch.from_numpy(np.random.default_rng(5).standard_normal((f.dim, 256))).cuda()
        f.solve(X)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            f.solve(X)
        torch.cuda.synchronize()
        rhs_s = 3 * 256 / (time.perf_counter() - t0)
        line["secondary"] = {"update_ms_mean": float(np.mean(upd)),
                             "update_ms_median": float(np.median(upd)), "update_ms": upd,
                             "update_n_dirty": cur.stats["n_dirty"], "solve_256rhs_per_s": rhs_s,
                             "factor_ms": total_ms / args.steps}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times_c, workers = cpu_reference_run(wl, 2, 0, budget_s=30.0)
        line["cpu_baseline"] = {"value": n_unk * len(times_c) / sum(times_c), "unit": UNIT,
                                "cores": workers, "kind": "port",
                                "sample": f"{len(times_c)} full cfg2 factorization(s) with oracle/skel_oracle.py "
                                          f"(numpy/scipy restatement of the reference, BLAS 1 thread)"}
    if rank == 0:
        gc_ = __import__("gc")
        gc_.collect()
        fp64 = measure_fp64_peak(torch)
        line["fp64_dgemm_tflops"] = fp64
        roof = line["roofline"]
        if roof["unit"] == "TFLOP/s":
            roof["peak"] = fp64
            roof["frac"] = roof["achieved"] / fp64
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

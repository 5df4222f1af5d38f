"""Median synchronised wall time of factor / update for a config (no profiling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200 import skel as S
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = configs.by_name(name)
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
f = fa()
seq = configs.hole_move_sequence(b, reps + 2)
cur = update(f, seq[0][2], seq[0][3])
del f
ft, ut, fw = [], [], []
for i in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w0, n0 = S.IO["wait_s"], S.IO["waits"]
    g = fa(); torch.cuda.synchronize(); ft.append(time.perf_counter() - t0); del g
    fw.append((S.IO["wait_s"] - w0, S.IO["waits"] - n0))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cur = update(cur, seq[i + 1][2], seq[i + 1][3]); torch.cuda.synchronize()
    ut.append(time.perf_counter() - t0)
ms = torch.cuda.memory_stats()
print("allocator: cudaMalloc calls", ms.get("num_device_alloc"), "retries", ms.get("num_alloc_retries"),
      "peak GB", ms.get("allocated_bytes.all.peak", 0) / 1e9, "reserved GB", ms.get("reserved_bytes.all.current", 0) / 1e9)
print(f"{name}: factor median {1e3*np.median(ft):.1f} ms (min {1e3*min(ft):.1f}); "
      f"update median {1e3*np.median(ut):.1f} ms (min {1e3*min(ut):.1f}); "
      f"factor host waits {[f'{1e3*w:.1f}ms/{n}' for w, n in fw]}")

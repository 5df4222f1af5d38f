"""Engine / driver host timing of one warm cfg2 hole-move update (SKB_ENGINE_TIMING=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2(); b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 6)
for i, (h, d, nb, rp) in enumerate(seq):
    torch.cuda.synchronize()
    print(f"--- update {i}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    f = update(f, nb, rp)
    torch.cuda.synchronize()
    print(f"--- {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr, flush=True)

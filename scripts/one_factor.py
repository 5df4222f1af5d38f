"""One warm factor (or update / solve) of a config between cudaProfilerStart/Stop,
for ncu launch lists (ncu --profile-from-start off).
  python scripts/one_factor.py cfg3 [factor|update|solve]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = sys.argv[2] if len(sys.argv) > 2 else "factor"
wl = configs.by_name(name)
b = wl.boundary
fa = lambda: factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol,
                    proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
f = fa()
if mode == "update":
    seq = configs.hole_move_sequence(b, 3)
    f = update(f, seq[0][2], seq[0][3])
    run = lambda: update(f, seq[1][2], seq[1][3])
elif mode == "solve":
    X = torch.from_numpy(configs.cfg5_rhs(b, 256) if name == "cfg3" else
                         np.random.default_rng(5).standard_normal((f.dim, 256))).cuda()
    f.solve(X)
    run = lambda: f.solve(X)
else:
    run = fa
run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", mode)

"""Bench-like sequence (factors, e2e factors, updates) with memory and timing checkpoints."""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200 import skel as S
from paper_2001_11619_b200.geometry import Boundary
wl = configs.cfg2(); b = wl.boundary; spec = SystemSpec()
tree = build_tree(b.positions, wl.leaf_cap)
def mem(tag):
    fr, tot = torch.cuda.mem_get_info()
    print(f"{tag}: free {fr/1e9:.1f} GB, torch reserved {torch.cuda.memory_reserved()/1e9:.2f} GB", flush=True)
mem("start")
for i in range(10):
    f = factor(spec, b, tree, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor); del f
mem("after 10 factors")
for i in range(5):
    bh = Boundary([c for c in b.curves]); th = build_tree(bh.positions, wl.leaf_cap)
    f = factor(spec, bh, th, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor); del f
mem("after e2e factors")
f = factor(spec, b, tree, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 30)
cur = f
ts = []
for h, d, nb, rep in seq:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cur = update(cur, nb, rep)
    torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
mem("after 30 updates")
print("update ms:", " ".join(f"{x:.0f}" for x in ts))

"""cProfile of one warm update() on cfg2."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200 import skel as S

wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 4)
cur = f
for _, _, nb, rep in seq[:3]:
    cur = update(cur, nb, rep)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
cur = update(cur, seq[3][2], seq[3][3])
torch.cuda.synchronize()
pr.disable()
print("update_time", cur.stats["update_time"])
pstats.Stats(pr).sort_stats("cumtime").print_stats(30)

"""cProfile of warm updates (cfg2 hole moves)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2(); b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 8)
cur = update(f, seq[0][2], seq[0][3]); cur = update(cur, seq[1][2], seq[1][3])
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for h, d, nb, rep in seq[2:]:
    cur = update(cur, nb, rep)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(30)

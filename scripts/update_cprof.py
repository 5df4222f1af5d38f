"""cProfile of update() on cfg2 (host-side hot spots of the update path)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2(); b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count,
           proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 12)
for h, d, nb, rp in seq[:3]:
    f = update(f, nb, rp)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for h, d, nb, rp in seq[3:]:
    f = update(f, nb, rp)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumtime").print_stats(45)

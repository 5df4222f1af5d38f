"""Device time per kernel family of one warm cfg2 update + host cProfile."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update, _lib
wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 4)
cur = f
for _, _, nb, rep in seq[:2]:
    cur = update(cur, nb, rep)
torch.cuda.synchronize()
_lib.prof_enable(True); _lib.prof_read(True)
t0 = time.perf_counter()
cur = update(cur, seq[2][2], seq[2][3])
torch.cuda.synchronize()
wall = time.perf_counter() - t0
fam = _lib.prof_read(True); _lib.prof_enable(False)
print(f"update wall {wall*1e3:.1f} ms, device {sum(v['ms'] for v in fam.values()):.1f} ms, dirty {cur.stats['n_dirty']}")
for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"   {k:9s} {v['ms']:7.2f} ms {v['launches']:5d}")
pr = cProfile.Profile(); pr.enable()
cur = update(cur, seq[3][2], seq[3][3])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(22)

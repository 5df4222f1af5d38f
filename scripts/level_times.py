"""Wall time per level (synchronised) of a warm factor and update on cfg2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200 import skel as S
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 3)
cur = update(f, seq[0][2], seq[0][3])
for label, fn in [("factor", lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count,
                                             proxy_factor=wl.proxy_factor)),
                  ("update", lambda: update(cur, seq[1][2], seq[1][3]))]:
    S._Prof.enabled = True
    S._Prof.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    S._Prof.enabled = False
    lv = {k: v for k, v in S._Prof.acc.items() if k.startswith("level")}
    rest = {k: v for k, v in S._Prof.acc.items() if not k.startswith("level")}
    print(label, f"wall {1e3*(time.perf_counter()-t0):.1f} ms;", " ".join(f"{k}:{1e3*v:.1f}" for k, v in lv.items()))
    print("   stages:", " ".join(f"{k}:{1e3*v:.1f}" for k, v in sorted(rest.items(), key=lambda kv: -kv[1])))
    del r

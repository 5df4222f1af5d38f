import os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200._lib import call
wl = configs.cfg2()
t = build_tree(wl.boundary.positions, wl.leaf_cap)
f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
x = torch.from_numpy(np.random.default_rng(0).standard_normal((f.dim, 1))).cuda()
xs = x.clone()
f._solve_dev(x.clone()); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
from paper_2001_11619_b200 import skel as S
arena = torch.empty(32 << 20, dtype=torch.uint8, pin_memory=True)
call("skb_capture_begin", 16 << 20); S._CAPTURE["arena"] = arena
try:
    with torch.cuda.graph(g):
        f._solve_dev(xs)
    print("captured OK")
except Exception:
    traceback.print_exc()
S._CAPTURE["arena"] = None
print("session", call("skb_capture_end"))
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); g.replay(); torch.cuda.synchronize(); print("replay ms", (time.perf_counter()-t0)*1e3)
y = x.clone(); f._solve_dev(y); print("diff", (y - xs).abs().max().item())

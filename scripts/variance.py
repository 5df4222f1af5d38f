"""Per-repetition factor wall time with host waits, new cudaMallocs and GC runs."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200 import skel as S
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
wl = configs.by_name(name)
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
f = fa(); del f
gcn = [0]
gc.callbacks.append(lambda ph, info: gcn.__setitem__(0, gcn[0] + (ph == "start")))
for r in range(reps):
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    w0 = S.IO["wait_s"]; g0 = gcn[0]
    t0 = time.perf_counter()
    f = fa()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"rep {r:2d}: wall {1e3*wall:6.1f} ms  waits {1e3*(S.IO['wait_s']-w0):5.1f} ms  "
          f"new cudaMalloc {torch.cuda.memory_stats().get('num_device_alloc',0)-m0}  gc {gcn[0]-g0}", flush=True)
    del f

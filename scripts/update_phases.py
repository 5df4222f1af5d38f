"""Host time per update() section (SKB_HOST_PROF=1), averaged over hole moves 3..N.
  python scripts/update_phases.py [cfg2|cfg3] [moves]"""
import gc, os, sys, time
os.environ.setdefault("SKB_HOST_PROF", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update, skel
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2"); b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, int(sys.argv[2]) if len(sys.argv) > 2 else 14)
ts = []
for i, (h, d, nb, rp) in enumerate(seq):
    gc.collect()
    torch.cuda.synchronize()
    if i == 2:
        skel._HostTimer.acc.clear()
        from paper_2001_11619_b200 import _lib
        _lib.CALL_TIMES = {}
    t0 = time.perf_counter()
    f = update(f, nb, rp)
    torch.cuda.synchronize()
    if i >= 2:
        ts.append((time.perf_counter() - t0) * 1e3)
n = len(ts)
print("update ms median %.2f" % np.median(ts), [round(x, 1) for x in ts])
for k, v in sorted(skel._HostTimer.acc.items(), key=lambda x: -x[1]):
    print("  %-14s %8.3f ms/update" % (k, v * 1e3 / n))

from paper_2001_11619_b200 import _lib
print("native entry points (host ms/update, calls/update):")
for k, (c, t) in sorted(_lib.CALL_TIMES.items(), key=lambda x: -x[1][1])[:14]:
    print("  %-26s %7.3f ms %6.1f" % (k, t * 1e3 / n, c / n))

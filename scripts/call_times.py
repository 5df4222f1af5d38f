"""Host time per C-ABI entry point during one warm cfg2 factor and update."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update, _lib
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 3)
cur = update(f, seq[0][2], seq[0][3])
torch.cuda.synchronize()
for label, fn in [("factor", lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count,
                                             proxy_factor=wl.proxy_factor)),
                  ("update", lambda: update(cur, seq[1][2], seq[1][3]))]:
    _lib.CALL_TIMES = {}
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    tot = sum(v[1] for v in _lib.CALL_TIMES.values())
    print(f"{label}: wall {wall*1e3:.1f} ms, in C calls {tot*1e3:.1f} ms")
    for k, (n, s_) in sorted(_lib.CALL_TIMES.items(), key=lambda kv: -kv[1][1])[:10]:
        print(f"   {k:24s} {n:4d} calls {s_*1e3:7.2f} ms")
    _lib.CALL_TIMES = None

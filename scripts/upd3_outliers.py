"""Reproduce bench.py's cfg3 sequence (factor, 256-RHS solves incl. pinned e2e, hole-move
updates) with host phase timers per update, to find slow update steps."""
import gc, os, sys, time
os.environ.setdefault("SKB_HOST_PROF", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update, skel
wl = configs.cfg3(); b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
if "nosolve" not in sys.argv:
    Xh = configs.cfg5_rhs(b, 256)
    X = torch.from_numpy(Xh).cuda()
    for _ in range(3):
        f.solve(X)
    if "nopin" not in sys.argv:
        Xp = torch.from_numpy(Xh).pin_memory(); Yp = torch.empty_like(Xp).pin_memory()
        for _ in range(3):
            Y = f.solve(Xp.cuda(non_blocking=True)); Yp.copy_(Y, non_blocking=True); torch.cuda.current_stream().synchronize()
        del Y
    del X
seq = configs.hole_move_sequence(b, 12)
cur = f
for i, (h, d, nb, rp) in enumerate(seq):
    torch.cuda.synchronize()
    before = dict(skel._HostTimer.acc)
    t0 = time.perf_counter()
    cur = update(cur, nb, rp)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    acc = {k: (v - before.get(k, 0.0)) * 1e3 for k, v in skel._HostTimer.acc.items()}
    top = sorted(acc.items(), key=lambda kv: -kv[1])[:5]
    print(f"move {i}: {dt:.1f} ms  reserved {torch.cuda.memory_reserved()/1e9:.1f} GB ", " ".join(f"{k}={v:.1f}" for k, v in top), flush=True)

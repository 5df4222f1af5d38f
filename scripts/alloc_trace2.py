"""Per-update time spent in torch.empty (update path), by call site."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
import paper_2001_11619_b200.skel as S
wl = configs.cfg2(); b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count,
           proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 24)
orig_empty = torch.empty
acc = collections.defaultdict(float)
def empty(*a, **k):
    t0 = time.perf_counter(); r = orig_empty(*a, **k); dt = time.perf_counter() - t0
    fr = sys._getframe(1)
    acc[(fr.f_code.co_name, fr.f_lineno)] += dt
    return r
S.torch.empty = empty
for i, (h, d, nb, rp) in enumerate(seq):
    acc.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = update(f, nb, rp)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    top = sorted(acc.items(), key=lambda kv: -kv[1])[:3]
    print(f"update {i}: {1e3*tot:.1f} ms, empty {1e3*sum(acc.values()):.1f} ms:",
          ", ".join(f"{k[0]}:{k[1]} {1e3*v:.1f}" for k, v in top), flush=True)
print(torch.cuda.memory_stats().get("num_device_alloc"))

"""Which allocations in update() are slow? (wraps torch.empty / Tensor.clone)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2(); b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count,
           proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 8)
for h, d, nb, rp in seq[:3]:
    f = update(f, nb, rp)
torch.cuda.synchronize()
rec = []
orig_empty = torch.empty
def empty(*a, **k):
    t0 = time.perf_counter(); r = orig_empty(*a, **k); dt = time.perf_counter() - t0
    import traceback
    rec.append((dt, r.numel() * r.element_size(), k.get("pin_memory", False), str(r.device),
                traceback.extract_stack(limit=3)[0].lineno))
    return r
torch.empty = empty
import paper_2001_11619_b200.skel as S
S.torch.empty = empty
t0 = time.perf_counter()
for h, d, nb, rp in seq[3:]:
    f = update(f, nb, rp)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
rec.sort(reverse=True)
print("update total ms", 1e3 * tot / 5, "allocs/update", len(rec) / 5, "alloc ms/update", 1e3 * sum(r[0] for r in rec) / 5)
for r in rec[:15]:
    print("  %.3f ms %10d B pin=%s %s line %d" % (1e3 * r[0], r[1], r[2], r[3], r[4]))
print("memory reserved GB", torch.cuda.memory_reserved() / 1e9, "allocated", torch.cuda.memory_allocated() / 1e9)
print(torch.cuda.memory_stats().get("num_alloc_retries"), torch.cuda.memory_stats().get("num_sync_all_streams"),
      torch.cuda.memory_stats().get("num_device_alloc"), torch.cuda.memory_stats().get("num_device_free"))

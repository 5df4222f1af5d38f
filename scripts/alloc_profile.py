"""Host time spent inside torch.empty per call site during warm factorizations."""
import collections, os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200 import skel as S
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = fa(); del f
real = torch.empty
acc = collections.defaultdict(lambda: [0, 0.0])
def timed(*a, **k):
    t0 = time.perf_counter()
    r = real(*a, **k)
    dt = time.perf_counter() - t0
    fr = traceback.extract_stack(limit=2)[0]
    e = acc[f"{os.path.basename(fr.filename)}:{fr.lineno}"]
    e[0] += 1; e[1] += dt
    return r
S.torch.empty = timed
for r in range(3):
    acc.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = fa(); torch.cuda.synchronize()
    print(f"rep {r}: wall {1e3*(time.perf_counter()-t0):.1f} ms, torch.empty total {1e3*sum(v[1] for v in acc.values()):.1f} ms")
    for k, (n, s_) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:6]:
        print(f"    {k:24s} {n:4d} calls {1e3*s_:7.2f} ms")
    del f
S.torch.empty = real

"""Where do occasional slow factor steps come from? (GC pauses / allocator growth)"""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200 import skel as S
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
b = wl.boundary
b._skb_device = S.DeviceBoundary(b)
gct = []
def cb(phase, info):
    if phase == "start":
        cb.t0 = time.perf_counter()
    else:
        gct.append((info["generation"], 1e3 * (time.perf_counter() - cb.t0)))
gc.callbacks.append(cb)
def step():
    t = build_tree(b.positions, wl.leaf_cap)
    return factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = step(); del f
for mode in ("gc on", "gc off"):
    if mode == "gc off":
        gc.collect(); gc.disable()
    ts = []
    for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
        gct.clear()
        print(f"=== {mode} step {i}", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = step()
        torch.cuda.synchronize()
        dt = 1e3 * (time.perf_counter() - t0)
        ts.append(dt)
        big = [g for g in gct if g[1] > 5]
        print(f"=== end {dt:.1f}", file=sys.stderr, flush=True)
        if dt > 1.3 * np.median(ts) or big:
            print(mode, "step", i, f"{dt:.1f} ms", "gc:", [(g, round(t, 1)) for g, t in gct if t > 1],
                  "reserved GB", torch.cuda.memory_reserved() / 1e9, flush=True)
        del f
    print(mode, "median", np.median(ts), "max", max(ts), flush=True)
    gc.enable()

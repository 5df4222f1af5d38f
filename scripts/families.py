"""Per-kernel-family device time of one warm factor (library CUDA-event timers)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, _lib

for name in sys.argv[1:] or ["cfg2"]:
    wl = configs.by_name(name)
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    for _ in range(2):
        f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        del f
    torch.cuda.synchronize()
    _lib.prof_enable(True)
    _lib.prof_read(True)
    t0 = time.perf_counter()
    f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    fam = _lib.prof_read(True)
    _lib.prof_enable(False)
    tot = sum(v["ms"] for v in fam.values())
    print(f"{name}: wall {wall*1e3:.1f} ms, device (family sum) {tot:.1f} ms")
    for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"]):
        extra = ""
        if v["flops"]:
            extra = f"  {v['flops']/(v['ms']*1e-3)/1e12:.2f} TFLOP/s"
        elif v["bytes"]:
            extra = f"  {v['bytes']/(v['ms']*1e-3)/1e9:.0f} GB/s"
        print(f"   {k:9s} {v['ms']:8.2f} ms  {v['launches']:5d} launches{extra}")

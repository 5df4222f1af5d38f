"""Time the batched LU (skb_getrf_batched) on single matrices of given orders."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import _lib
if os.environ.get("SKB_LIB"):          # compare another build of the library
    _lib.load(os.environ["SKB_LIB"])
from paper_2001_11619_b200 import skel
from paper_2001_11619_b200._lib import call

for n in [int(a) for a in (sys.argv[1:] or ["276", "849", "2532"])]:
    A0 = torch.from_numpy(np.random.default_rng(n).standard_normal((n, n))).cuda()
    A = A0.clone()
    ip = torch.empty(n, dtype=torch.int32, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    ratio = torch.empty(1, dtype=torch.float64, device="cuda")
    m = skel._mats(np.array([A.data_ptr()], np.uint64), [n], [n], [n])
    ipp = np.array([ip.data_ptr()], np.uint64)
    ts = []
    for it in range(6):
        A.copy_(A0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call("skb_getrf_batched", 1, m, ipp, info, ratio, skel._stream())
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    if os.environ.get("LU_BREAKDOWN"):
        from torch.profiler import ProfilerActivity, profile
        A.copy_(A0)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            call("skb_getrf_batched", 1, m, ipp, info, ratio, skel._stream())
            torch.cuda.synchronize()
        agg = {}
        for e in prof.events():
            if e.device_type.name == "CUDA":
                k = e.name.split("(")[0].replace("void ", "")[:40]
                c, t = agg.get(k, (0, 0.0))
                agg[k] = (c + 1, t + e.device_time_total / 1e3)
        print("  " + "; ".join(f"{k} x{c} {t:.3f} ms" for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])))
    if os.environ.get("LU_SAVE"):
        np.save(f"{os.environ['LU_SAVE']}_{n}_A.npy", A.cpu().numpy())
        np.save(f"{os.environ['LU_SAVE']}_{n}_p.npy", ip.cpu().numpy())
    print(f"n={n}: LU {min(ts[1:]):.3f} ms ({2 * n ** 3 / 3 / (min(ts[1:]) * 1e-3) / 1e12:.3f} TFLOP/s)")

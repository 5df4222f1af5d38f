"""Time skb_geqrf_batched on synthetic single-shape batches (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200._lib import call

def run(m, n, B, reps=5):
    A = torch.randn(B, n, m, dtype=torch.float64, device="cuda")   # column-major m x n per box
    A0 = A.clone()
    ptrs = np.array([A.data_ptr() + 8 * b * n * m for b in range(B)], np.int64)
    mm = np.full(B, m, np.int64); nn = np.full(B, n, np.int64)
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for r in range(reps + 1):
        A.copy_(A0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        call("skb_geqrf_batched", B, mm, nn, mm, ptrs, s)
        e1.record(); torch.cuda.synchronize()
        if r: ts.append(e0.elapsed_time(e1))
    return min(ts)

if __name__ != "__main__":
    shapes = []
else:
    shapes = [(512, 32), (512, 64), (512, 96), (512, 128), (512, 160), (512, 192),
          (256, 96), (384, 96), (1024, 96), (1024, 192), (2048, 96)]
for m, n in shapes:  # noqa
    t1 = run(m, n, 1)
    t148 = run(m, n, 148)
    t296 = run(m, n, 296)
    print(f"m {m:5d} n {n:4d}: 1 box {1e3*t1:8.1f} us  148 boxes {1e3*t148:8.1f} us  296 boxes {1e3*t296:8.1f} us"
          f"  ({2*m*n*n*296/(t296*1e-3)/1e12:.2f} TF/s)")

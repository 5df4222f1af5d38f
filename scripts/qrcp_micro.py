"""Time skb_qrcp_id_batched on synthetic R factors (rank ~ n/2 at tol 1e-10)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200._lib import call

def make(n, B, seed=0):
    rng = np.random.default_rng(seed)
    out = np.empty((B, n, n))
    for b in range(B):
        U, _ = np.linalg.qr(rng.standard_normal((n, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        A = (U * np.logspace(0, -20, n)) @ V.T
        R = np.linalg.qr(A, mode="r")
        out[b] = R.T            # column-major storage of R
    return out

def run(n, B, reps=3):
    H = make(n, min(B, 16))
    H = np.concatenate([H] * ((B + 15) // 16))[:B]
    A = torch.from_numpy(H).cuda()
    A0 = A.clone()
    ptrs = np.array([A.data_ptr() + 8 * b * n * n for b in range(B)], np.int64)
    nn = np.full(B, n, np.int64)
    off = np.arange(B + 1, dtype=np.int64) * n
    perm = torch.empty(B * n, dtype=torch.int32, device="cuda")
    diag = torch.empty(B * n, dtype=torch.float64, device="cuda")
    ko = torch.empty(2 * B, dtype=torch.int32, device="cuda")
    gap = torch.empty(B, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for r in range(reps + 1):
        A.copy_(A0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        call("skb_qrcp_id_batched", B, nn, nn, nn, ptrs, np.zeros(B, np.int64), 1e-10, off,
             perm, diag, ko, ko.data_ptr() + 4 * B, gap, s)
        e1.record(); torch.cuda.synchronize()
        if r: ts.append(e0.elapsed_time(e1))
    k = ko.cpu().numpy()
    return min(ts), int(k[:B].max()), int(k[B:].max())

cases = [(64, 100), (96, 230), (128, 230), (160, 150), (200, 100), (256, 30), (400, 8)]
if len(sys.argv) > 1 and sys.argv[1] == "single":
    cases = [(64, 1), (96, 1), (128, 1), (160, 1), (256, 1), (400, 1)]
for n, B in cases:
    t, k, st = run(n, B)
    print(f"n {n:4d} B {B:4d}: {1e3*t:8.1f} us  k {k} steps {st}  ({1e3*t/st:.2f} us/step)", flush=True)

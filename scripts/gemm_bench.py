"""Grouped DMMA GEMM throughput vs cuBLAS DGEMM on representative shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import skel as S

def run(m, n, k, ta=0, tb=0, batch=1, reps=5):
    A = [torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device="cuda") for _ in range(batch)]
    B = [torch.randn((n, k) if tb else (k, n), dtype=torch.float64, device="cuda") for _ in range(batch)]
    D = [torch.empty((m, n), dtype=torch.float64, device="cuda") for _ in range(batch)]
    rows = [dict(A=np.array([a.data_ptr() for a in A], np.uint64), B=np.array([b.data_ptr() for b in B], np.uint64),
                 D=np.array([d.data_ptr() for d in D], np.uint64), m=np.full(batch, m), n=np.full(batch, n),
                 k=np.full(batch, k), lda=np.full(batch, A[0].shape[1]), ldb=np.full(batch, B[0].shape[1]),
                 ldd=np.full(batch, n), alpha=np.ones(batch), beta=np.zeros(batch),
                 transA=np.full(batch, ta), transB=np.full(batch, tb))]
    S._gemm(rows); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        S._gemm(rows)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * m * n * k * batch
    Ar = A[0].T if ta else A[0]
    Br = B[0].T if tb else B[0]
    ref = Ar @ Br
    err = (D[0] - ref).abs().max().item() / ref.abs().max().item()
    e0.record()
    for _ in range(reps):
        for i in range(batch):
            (A[i].T if ta else A[i]) @ (B[i].T if tb else B[i])
    e1.record(); e1.synchronize()
    ms2 = e0.elapsed_time(e1) / reps
    print(f"m{m} n{n} k{k} tA{ta} tB{tb} x{batch}: skb {fl/ms/1e9:7.2f} TF ({ms:.3f} ms)  cuBLAS {fl/ms2/1e9:7.2f} TF  relerr {err:.1e}")

run(4096, 4096, 4096)
run(8192, 8192, 1024)
run(1000, 768, 200, batch=64)
run(100, 768, 100, ta=1, batch=1000)
run(500, 91, 32, batch=300)
run(768, 256, 300000, ta=1)
run(294912, 256, 768)
run(2532, 256, 2532)

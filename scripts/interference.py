"""Kernel-interference stress: batched LU (stream A) while the QR/QRCP kernels
run on stream B; LU results must be bitwise identical to an isolated run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import skel
from paper_2001_11619_b200._lib import call

rng = np.random.default_rng(0)
ns = [40, 49, 57, 75, 120, 145, 160] * 6
mats = [torch.from_numpy(rng.standard_normal((n, n))).cuda() for n in ns]
work = [m.clone() for m in mats]
ipiv = [torch.empty(n, dtype=torch.int32, device="cuda") for n in ns]
info = torch.empty(len(ns), dtype=torch.int32, device="cuda")
ratio = torch.empty(len(ns), dtype=torch.float64, device="cuda")
M = skel._mats(np.array([w.data_ptr() for w in work], np.uint64), ns, ns, ns)
IP = np.array([p.data_ptr() for p in ipiv], np.uint64)
mode = sys.argv[1] if len(sys.argv) > 1 else "qrcp"
# stream B workload: wide stacks like cfg2 levels 1-2
mq, nq = {"qrcp": (912, 464), "small": (500, 120), "cl3": (200, 200), "mode0": (160, 150)}[mode]
Bn = 8
stk0 = torch.from_numpy(rng.standard_normal((Bn, nq, mq))).cuda()   # column-major per box
stk = stk0.clone()
A = np.array([stk[b].data_ptr() for b in range(Bn)], np.int64)
mm = np.full(Bn, mq, np.int64); nn = np.full(Bn, nq, np.int64)
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()

def lu(s):
    for w, m in zip(work, mats):
        w.copy_(m)
    call("skb_getrf_batched", len(ns), M, IP, info, ratio, s.cuda_stream)

def qr(s):
    stk.copy_(stk0)
    if mq > nq:
        call("skb_geqrf_batched", Bn, mm, nn, mm, A, s.cuda_stream)
    ints = torch.empty(Bn * nq + 2 * Bn + 1, dtype=torch.int32, device="cuda")
    dg = torch.empty(Bn * nq, dtype=torch.float64, device="cuda")
    gp = torch.empty(Bn, dtype=torch.float64, device="cuda")
    po = np.arange(Bn + 1, dtype=np.int64) * nq
    call("skb_qrcp_id_batched", Bn, np.minimum(mm, nn), nn, mm, A, np.zeros(Bn, np.int64), 1e-10, po, ints,
         dg, ints.data_ptr() + 4 * Bn * nq, ints.data_ptr() + 4 * (Bn * nq + Bn), gp, s.cuda_stream)
    return ints, dg, gp

with torch.cuda.stream(sA):
    lu(sA)
torch.cuda.synchronize()
ref = [w.clone() for w in work]
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    with torch.cuda.stream(sB):
        keep = qr(sB)
    with torch.cuda.stream(sA):
        lu(sA)
    torch.cuda.synchronize()
    nbad = sum(not torch.equal(w, r) for w, r in zip(work, ref))
    if nbad:
        bad += 1
        print("iteration", it, ":", nbad, "LU results differ")
print(mode, "iterations with differing LU:", bad)

"""Bitwise repeatability of the batched Householder QR and QRCP on level-1
shaped stacks (cluster kernels): N repeats per batch size, first mismatch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import skel
from paper_2001_11619_b200._lib import call

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
m, n = 912, 464
rng = np.random.default_rng(0)
base = [rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -14, n)) for _ in range(4)]
for nbox in (1, 2, 3, 4):
    ref = None
    bad_g = bad_q = 0
    for it in range(N):
        dev = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in base[:nbox]]
        ptrs = np.array([d.data_ptr() for d in dev], np.int64)
        mm = np.full(nbox, m, np.int64)
        nn = np.full(nbox, n, np.int64)
        call("skb_geqrf_batched", nbox, mm, nn, mm, ptrs, skel._stream())
        torch.cuda.synchronize()
        R = [d.cpu().numpy().copy() for d in dev]
        # QRCP on the n x n R (column-major, lda = m)
        perm = torch.zeros(nbox * n, dtype=torch.int32, device="cuda")
        diag = torch.zeros(nbox * n, dtype=torch.float64, device="cuda")
        k = torch.zeros(nbox, dtype=torch.int32, device="cuda")
        st = torch.zeros(nbox, dtype=torch.int32, device="cuda")
        gap = torch.zeros(nbox, dtype=torch.float64, device="cuda")
        poff = np.arange(nbox + 1, dtype=np.int64) * n
        call("skb_qrcp_id_batched", nbox, nn, nn, mm, ptrs, np.zeros(nbox, np.int64), 1e-12,
             poff, perm, diag, k, st, gap, skel._stream())
        torch.cuda.synchronize()
        Q = [d.cpu().numpy().copy() for d in dev] + [perm.cpu().numpy(), k.cpu().numpy()]
        if ref is None:
            ref = (R, Q)
            continue
        if not all(np.array_equal(a, b) for a, b in zip(R, ref[0])):
            bad_g += 1
        elif not all(np.array_equal(a, b) for a, b in zip(Q, ref[1])):
            bad_q += 1
    print(f"nbox {nbox}: geqrf mismatches {bad_g}/{N-1}, qrcp mismatches {bad_q}/{N-1}", flush=True)

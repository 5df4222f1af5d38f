"""QRCP microbenchmark on synthetic top-level shapes (decaying spectrum, rank ~ k at tol):
  python scripts/qrcp_bench.py [nbox m n k]   -> ms per batched call, steps, agreement with scipy"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.linalg as sla
from paper_2001_11619_b200._lib import call
from paper_2001_11619_b200 import skel
nbox, m, n, k = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4, 1804, 1182, 441)
tol = 1e-8
rng = np.random.default_rng(0)
mats = []
for b in range(nbox):
    U, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
    V, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
    sig = 10.0 ** (-8.0 * np.arange(min(m, n)) / k)
    mats.append((U * sig) @ V.T)
flat = np.concatenate([A.T.ravel() for A in mats])          # column-major per box
off = np.arange(nbox, dtype=np.int64) * (m * n)
act_off = np.arange(nbox + 1, dtype=np.int64) * n
s = skel._stream()
ts = []
for it in range(6):
    d = torch.from_numpy(flat).cuda()
    A = (d.data_ptr() + 8 * off).astype(np.int64)
    perm = torch.empty(nbox * n, dtype=torch.int32, device="cuda")
    diag = torch.empty(nbox * n, dtype=torch.float64, device="cuda")
    ko = torch.empty(2 * nbox, dtype=torch.int32, device="cuda")
    gap = torch.empty(nbox, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call("skb_qrcp_id_batched", nbox, np.full(nbox, m, np.int64), np.full(nbox, n, np.int64),
         np.full(nbox, m, np.int64), A, np.zeros(nbox, np.int64), tol, act_off, perm, diag, ko,
         ko.data_ptr() + 4 * nbox, gap, s)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
kk = ko.cpu().numpy()
pm = perm.cpu().numpy().reshape(nbox, n)
ok = 0
for b in range(min(nbox, 2)):
    _, R, p = sla.qr(mats[b], mode="economic", pivoting=True)
    dg = np.abs(np.diag(R))
    kr = int(np.count_nonzero(dg > tol * dg[0]))
    ok += int(kr == kk[b] and np.array_equal(p[:kr], pm[b, :kr]))
env = {k_: v for k_, v in os.environ.items() if k_.startswith("SKB_")}
print(f"{env} {nbox}x({m}x{n}) k={kk[:nbox].tolist()[:4]} steps={kk[nbox:].tolist()[:4]} "
      f"ms min {min(ts):.2f} med {np.median(ts):.2f}; scipy-identical skeletons {ok}/{min(nbox, 2)}", flush=True)
import ctypes
from paper_2001_11619_b200 import _lib
lib = _lib.load()
if hasattr(lib, "skb_qblk_trace_get"):
    out = (ctypes.c_longlong * 16)()
    lib.skb_qblk_trace_get(out, 1)
    tot = sum(out[:9]) or 1
    names = ["argmax", "barrier", "winner", "pivot col", "reflector", "aux+list", "dots", "finalize", "flush"]
    print("  phases (clock share):", " ".join(f"{n} {100*out[j]/tot:.0f}%" for j, n in enumerate(names)),
          f"| total {tot/6/1.9e6:.2f} ms/call")
if hasattr(lib, "skb_qrcp_trace_get"):
    tr = (ctypes.c_longlong * (256 * 8))()
    lib.skb_qrcp_trace_get(tr)
    a = np.array(tr[:]).reshape(256, 8)[20:200]
    d = np.diff(a[:, :7], axis=1).mean(axis=0)
    nxt = (a[1:, 0] - a[:-1, 6]).mean()
    names = ["argmax", "sync", "cl.sync", "reflector(w0)", "sync", "scale+sync"]
    print("  mode-1 step cycles:", " ".join(f"{n} {v:.0f}" for n, v in zip(names, d)), f"update {nxt:.0f}",
          f"| step {(a[1:, 0] - a[:-1, 0]).mean():.0f} cycles")

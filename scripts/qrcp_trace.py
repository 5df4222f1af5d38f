"""Per-step phase cycles of the cluster QRCP (mode 1), CTA 0 of box 0; needs
the -DSKB_QRCP_TRACE build loaded through SKB_LIB."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import _lib
lib = _lib.load(os.environ["SKB_LIB"])
from paper_2001_11619_b200 import skel
from paper_2001_11619_b200._lib import call
m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 464
nbox = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rng = np.random.default_rng(1)
base = [np.triu(rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -14, n))) for _ in range(nbox)]
for it in range(2):
    dev = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in base]
    ptrs = np.array([d.data_ptr() for d in dev], np.int64)
    mm = np.full(nbox, m, np.int64); nn = np.full(nbox, n, np.int64)
    perm = torch.zeros(nbox * n, dtype=torch.int32, device="cuda")
    diag = torch.zeros(nbox * n, dtype=torch.float64, device="cuda")
    k = torch.zeros(nbox, dtype=torch.int32, device="cuda")
    st = torch.zeros(nbox, dtype=torch.int32, device="cuda")
    gap = torch.zeros(nbox, dtype=torch.float64, device="cuda")
    poff = np.arange(nbox + 1, dtype=np.int64) * n
    call("skb_qrcp_id_batched", nbox, mm, nn, mm, ptrs, np.zeros(nbox, np.int64), 1e-12,
         poff, perm, diag, k, st, gap, skel._stream())
    torch.cuda.synchronize()
tr = np.zeros((256, 8), np.int64)
lib.skb_qrcp_trace_get(ctypes.c_void_p(tr.ctypes.data))
steps = tr[1:200]
nxt = tr[2:201, 0]
names = ["argmax", "sync1", "cluster", "reflector", "sync2", "scale+sync3", "apply(next)"]
d = np.stack([steps[:, 1] - steps[:, 0], steps[:, 2] - steps[:, 1], steps[:, 3] - steps[:, 2],
              steps[:, 4] - steps[:, 3], steps[:, 5] - steps[:, 4], steps[:, 6] - steps[:, 5],
              nxt - steps[:, 6]], 1)
print("k", k.cpu().numpy(), "median cycles per phase:", {nm: int(np.median(d[:, j])) for j, nm in enumerate(names)},
      "total", int(np.median(nxt - steps[:, 0])))

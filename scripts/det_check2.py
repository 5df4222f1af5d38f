"""Engine vs Python level loop: compare level-1 ID stacks before / after QRCP (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKB_ENGINE_SNAP"] = "1"
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, _lib
from paper_2001_11619_b200 import skel as S
wl = getattr(configs, sys.argv[1])()
b = wl.boundary
lib = _lib.load()
py = {}
orig_call = S.call
def spy(name, *args):
    if name in ("skb_qrcp_id_batched",):
        B, mq, nB, lda, A = args[:5]
        if int(np.max(nB)) >= 300:
            torch.cuda.synchronize()
            py["pre"] = [S._fetch(int(A[j]), int(nB[j]), int(lda[j])) for j in range(B)]
            py["meta"] = (np.array(mq), np.array(nB), np.array(lda))
            r = orig_call(name, *args)
            torch.cuda.synchronize()
            py["post"] = [S._fetch(int(A[j]), int(nB[j]), int(lda[j])) for j in range(B)]
            return r
    return orig_call(name, *args)
S.call = spy
S._ENGINE_ON = False
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
S.call = orig_call
eng = {}
ow = S._Engine.wait
def w(self, L):
    h = ow(self, L)
    if L == 1:
        eng["h"] = h
    return h
S._Engine.wait = w
S._ENGINE_ON = True
f2 = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
h = eng["h"]
def snap(wh):
    n = lib.skb_debug_snap(wh, None, 0)
    buf = np.empty(n); lib.skb_debug_snap(wh, buf.ctypes.data, n); return buf
s1, s2 = snap(1), snap(2)
base = int(h["A"][0])
print("python meta mq nB lda", py["meta"])
print("engine rows", h["rows"], "nB", h["nB"], "mq", h["m_q"])
for j in range(len(h["A"])):
    o = (int(h["A"][j]) - base) // 8
    n = int(h["nB"][j]) * int(h["rows"][j])
    e1, e2 = s1[o:o + n], s2[o:o + n]
    p1, p2 = py["pre"][j].ravel(), py["post"][j].ravel()
    print(j, "pre-QRCP equal", np.array_equal(e1, p1), "post-QRCP equal", np.array_equal(e2, p2),
          "max post diff", float(np.max(np.abs(e2 - p2))) if len(p2) == len(e2) else "len")

"""How sensitive is the cfg3 solution to the summation order of PsiV^T z?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, system_matvec
from paper_2001_11619_b200 import skel as S
wl = configs.cfg3()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
rng = np.random.default_rng(1)
rhs = np.concatenate([rng.standard_normal(2 * b.n_nodes), np.zeros(3 * b.n_holes)])
orig = S._gemm_tn_splitk
for chunk in (256, 1024, 4096, 16384, 10**9):
    def patched(*a, chunk=chunk, **k):
        k["chunk"] = chunk
        return orig(*a, **k)
    S._gemm_tn_splitk = patched
    X = torch.from_numpy(rhs.reshape(-1, 1).copy()).cuda()
    f._solve_dev(X)
    x = X.cpu().numpy().ravel()
    r = system_matvec(SystemSpec(), b, x) - rhs
    print(f"chunk {chunk:>10}: residual {np.linalg.norm(r)/np.linalg.norm(rhs):.3e}  |x| {np.linalg.norm(x):.3e}", flush=True)
S._gemm_tn_splitk = orig

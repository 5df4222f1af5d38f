"""cfg5: 256-RHS solve on the cfg3 factorization (RHS/s) + sampled residuals."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, system_matvec

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 256
wl = configs.by_name(name)
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
F = configs.cfg5_rhs(b, nrhs)
X = torch.from_numpy(F).cuda()
f.solve(X)                         # capture
torch.cuda.synchronize()
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Y = f.solve(X)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
Y = Y.cpu().numpy()
cols = sorted(set([0, min(1, nrhs - 1), nrhs // 2, nrhs - 1]))
M = system_matvec(SystemSpec(), b, Y[:, cols])
res = [float(np.linalg.norm(M[:, j] - F[:, c]) / np.linalg.norm(F[:, c])) for j, c in enumerate(cols)]
print(json.dumps({"config": name, "nrhs": nrhs, "solve_s": min(ts), "rhs_per_s": nrhs / min(ts),
                  "factor_s": f.stats["factor_time"], "sampled_residuals": res}))

import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import skel as S
torch.cuda.init()
s = torch.cuda.current_stream()
rng = np.random.default_rng(0)
for rnd in range(4):
    objs = []
    t0 = time.perf_counter()
    for i in range(150):
        objs.append(S._DevSlab(int(rng.integers(1e4, 8e6)), s))
    t1 = time.perf_counter()
    del objs
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    S._DevSlab.flush()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"round {rnd}: 150 allocs {1e3*(t1-t0):.2f} ms, flush {1e3*(t3-t2):.2f} ms")

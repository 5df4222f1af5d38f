"""geqrf micro-benchmark over shapes (run under different SKB_FUSED_SET)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.geqrf_micro import run
for m, n in [(480, 90), (512, 160), (700, 110), (900, 190), (1024, 96)]:
    print(f"set {os.environ.get('SKB_FUSED_SET','0')} m {m} n {n}: B=150 {1e3*run(m, n, 150):7.1f} us  B=300 {1e3*run(m, n, 300):7.1f} us", flush=True)

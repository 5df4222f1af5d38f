"""Find host stalls: run N warm factorizations under the torch profiler and list
host ranges and CUDA runtime calls that took longer than a threshold."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SKB_HOST_PROF", "trace")
import torch
from torch.profiler import ProfilerActivity, profile, record_function

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor

wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = fa()
    del f
torch.cuda.synchronize()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
smi = None
if "--smi" in sys.argv:
    import subprocess
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                            "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "200"],
                           stdout=subprocess.DEVNULL)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
if "--update" in sys.argv:
    from paper_2001_11619_b200 import update
    cur = fa()
    seq = configs.hole_move_sequence(b, n + 1)
    cur = update(cur, seq[0][2], seq[0][3])
    torch.cuda.synchronize()
    seq_it = iter(seq[1:])
    def fa():
        global cur
        h_, d_, nb_, rep_ = next(seq_it)
        cur = update(cur, nb_, rep_)
        return None
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for it in range(n):
        if "--flush" in sys.argv:
            flush.fill_(1.0)
            torch.cuda.synchronize()
        with record_function(f"STEP{it}"):
            f = fa()
            del f
        torch.cuda.synchronize()
if smi is not None:
    smi.terminate()
prof.export_chrome_trace("gpurun_out/stalls.json")
ev = json.load(open("gpurun_out/stalls.json"))["traceEvents"]
steps = sorted([e for e in ev if e.get("name", "").startswith("STEP") and e.get("ph") == "X"
                and e.get("cat") == "user_annotation"],
               key=lambda e: e["ts"])
print("step ms:", [round(e["dur"] / 1e3, 1) for e in steps if e["dur"] > 0])
for e in sorted(ev, key=lambda e: e.get("ts", 0)):
    if e.get("ph") != "X" or e.get("name", "").startswith("STEP") or e.get("name") == "run_levels":
        continue
    if e.get("cat") in ("user_annotation", "cuda_runtime", "cpu_op") and e["dur"] > thr * 1e3:
        st = next((s["name"] for s in steps if s["ts"] <= e["ts"] <= s["ts"] + s["dur"]), "?")
        print(f"{st:7s} {e.get('cat'):16s} {e['name'][:50]:50s} {e['dur'] / 1e3:8.2f} ms")
import gc
gc.disable()
torch.cuda.synchronize()
m0 = torch.cuda.memory_allocated()
f = fa()
torch.cuda.synchronize()
m1 = torch.cuda.memory_allocated()
del f
m2 = torch.cuda.memory_allocated()
print(f"allocated before {m0/1e6:.1f} MB, with factorization {m1/1e6:.1f} MB, after del (no GC) {m2/1e6:.1f} MB")
gc.enable()

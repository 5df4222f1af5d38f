"""Find the slow factorization steps under a given engine run-ahead and show which level's
engine / driver phase took the time (SKB_ENGINE_TIMING lines between step markers)."""
import os, re, subprocess, sys
env = dict(os.environ, SKB_ENGINE_TIMING="1")
n = sys.argv[1] if len(sys.argv) > 1 else "60"
p = subprocess.run([sys.executable, "scripts/outliers.py", "cfg3", n], env=env, capture_output=True, text=True)
steps, cur = [], None
for ln in p.stderr.splitlines():
    if ln.startswith("=== end"):
        cur["ms"] = float(ln.split()[2]); steps.append(cur); cur = None
    elif ln.startswith("==="):
        cur = {"name": ln, "lines": []}
    elif cur is not None and ("engine level" in ln or "driver level" in ln):
        cur["lines"].append(ln)
ms = sorted(s["ms"] for s in steps)
print("steps", len(steps), "median", ms[len(ms) // 2], "max", ms[-1])
for s in sorted(steps, key=lambda s: -s["ms"])[:2]:
    print(s["name"], s["ms"])
    for ln in s["lines"]:
        big = [(k, int(v)) for k, v in re.findall(r"(\w[\w+]*) (\d+)", ln.split(":", 1)[1]) if int(v) > 3000]
        print("   ", ln.split(":")[0], big)

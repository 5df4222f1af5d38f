"""QRCP mode-1 (cluster) results and time vs the cluster width: bitwise
comparison of perm/k/R between widths (SKB_QRCP_CMIN set per subprocess)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np
    import torch
    from paper_2001_11619_b200 import _lib
    if os.environ.get("SKB_LIB"):
        _lib.load(os.environ["SKB_LIB"])
    from paper_2001_11619_b200 import skel
    from paper_2001_11619_b200._lib import call
    out = sys.argv[2]
    res = {}
    for (m, n, nbox) in [(464, 464, 4), (700, 700, 4), (600, 600, 8)]:
        rng = np.random.default_rng(m + nbox)
        base = [np.triu(rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -14, n))) for _ in range(nbox)]
        ts = []
        for it in range(4):
            dev = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in base]
            ptrs = np.array([d.data_ptr() for d in dev], np.int64)
            mm = np.full(nbox, m, np.int64); nn = np.full(nbox, n, np.int64)
            perm = torch.zeros(nbox * n, dtype=torch.int32, device="cuda")
            diag = torch.zeros(nbox * n, dtype=torch.float64, device="cuda")
            k = torch.zeros(nbox, dtype=torch.int32, device="cuda")
            st = torch.zeros(nbox, dtype=torch.int32, device="cuda")
            gap = torch.zeros(nbox, dtype=torch.float64, device="cuda")
            poff = np.arange(nbox + 1, dtype=np.int64) * n
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            call("skb_qrcp_id_batched", nbox, mm, nn, mm, ptrs, np.zeros(nbox, np.int64), 1e-12,
                 poff, perm, diag, k, st, gap, skel._stream())
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"{m}x{n}x{nbox}"] = (min(ts[1:]), [d.cpu().numpy() for d in dev], perm.cpu().numpy(), k.cpu().numpy())
    import pickle
    pickle.dump(res, open(out, "wb"))
elif len(sys.argv) > 1 and sys.argv[1] == "cmp":
    import pickle
    import numpy as np
    a, b = pickle.load(open(sys.argv[2], "rb")), pickle.load(open(sys.argv[3], "rb"))
    for key in a:
        t0, R0, p0, k0 = a[key]
        t1, R1, p1, k1 = b[key]
        same = np.array_equal(p0, p1) and np.array_equal(k0, k1) and all(np.array_equal(x, y) for x, y in zip(R0, R1))
        print(key, f"{t0:.3f} ms -> {t1:.3f} ms", "bitwise same" if same else "DIFF")
else:
    import pickle
    import numpy as np
    outs = {}
    for c in ["0", "4", "8", "16"]:
        env = dict(os.environ, SKB_QRCP_CMIN=c)
        subprocess.run([sys.executable, __file__, "run", f"/tmp/qc_{c}.pkl"], env=env, check=True)
        outs[c] = pickle.load(open(f"/tmp/qc_{c}.pkl", "rb"))
    for key in outs["0"]:
        line = [key]
        for c in outs:
            t, R, p, k = outs[c][key]
            t0, R0, p0, k0 = outs["0"][key]
            same = np.array_equal(p, p0) and np.array_equal(k, k0) and all(np.array_equal(a, b) for a, b in zip(R, R0))
            line.append(f"C>={c}: {t:.3f} ms {'same' if same else 'DIFF'}")
        print("  ".join(line))

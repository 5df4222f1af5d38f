"""Kernel-level parity on a B200: each C-ABI primitive against the fp64 CPU
reference of the same operation (NumPy/SciPy LAPACK), on seeded inputs."""

import numpy as np
import pytest
import scipy.linalg as sla

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import skel_oracle as O  # noqa: E402
from paper_2001_11619_b200 import configs, skel  # noqa: E402
from paper_2001_11619_b200._lib import call  # noqa: E402
from paper_2001_11619_b200.tree import build_tree  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_gemm_grouped_ragged():
    rng = np.random.default_rng(0)
    shapes = [(1, 1, 1), (7, 65, 3), (64, 64, 16), (130, 17, 200), (5, 300, 0), (0, 4, 4),
              (96, 96, 96)]
    rows = []
    outs, refs = [], []
    for ta in (0, 1):
        for tb in (0, 1):
            for (m, n, k) in shapes:
                A = rng.standard_normal((k, m) if ta else (m, k))
                B = rng.standard_normal((n, k) if tb else (k, n))
                C = rng.standard_normal((m, n))
                dA, dB, dC = _dev(A), _dev(B), _dev(C)
                dD = torch.empty((max(m, 1), max(n, 1)), dtype=torch.float64, device="cuda")
                rows.append(dict(A=np.array([dA.data_ptr()], np.uint64), B=np.array([dB.data_ptr()], np.uint64),
                                 C=np.array([dC.data_ptr()], np.uint64), D=np.array([dD.data_ptr()], np.uint64),
                                 m=[m], n=[n], k=[k], lda=[max(A.shape[1], 1)], ldb=[max(B.shape[1], 1)],
                                 ldc=[max(n, 1)], ldd=[max(n, 1)], alpha=[-0.5], beta=[2.0],
                                 transA=[ta], transB=[tb]))
                opA = A.T if ta else A
                opB = B.T if tb else B
                refs.append(-0.5 * (opA @ opB) + 2.0 * C)
                outs.append((dD, m, n, dA, dB, dC))
    skel._gemm(rows)
    torch.cuda.synchronize()
    for (dD, m, n, *_), R in zip(outs, refs):
        if m == 0 or n == 0:
            continue
        got = dD.cpu().numpy()[:m, :n]
        assert np.allclose(got, R, rtol=1e-13, atol=1e-12 * max(1, np.abs(R).max()))


def test_getrf_getrs_batched():
    rng = np.random.default_rng(1)
    ns = [1, 5, 63, 64, 65, 130, 257]
    mats, ipivs, Bs, refs = [], [], [], []
    for n in ns:
        A = rng.standard_normal((n, n)) + 0.1 * np.eye(n)
        Bm = rng.standard_normal((n, 3))
        mats.append(_dev(A))
        ipivs.append(torch.empty(n, dtype=torch.int32, device="cuda"))
        Bs.append(_dev(Bm))
        refs.append((A, Bm))
    m = skel._mats(np.array([t.data_ptr() for t in mats], np.uint64), ns, ns, ns)
    ip = np.array([t.data_ptr() for t in ipivs], np.uint64)
    info = torch.empty(len(ns), dtype=torch.int32, device="cuda")
    ratio = torch.empty(len(ns), dtype=torch.float64, device="cuda")
    call("skb_getrf_batched", len(ns), m, ip, info, ratio, skel._stream())
    b = skel._mats(np.array([t.data_ptr() for t in Bs], np.uint64), ns, [3] * len(ns), [3] * len(ns))
    call("skb_getrs_batched", len(ns), m, ip, b, skel._stream())
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == -1).all()
    for (A, Bm), X, r in zip(refs, Bs, ratio.cpu().numpy()):
        x = X.cpu().numpy()
        ref = np.linalg.solve(A, Bm)
        assert np.linalg.norm(x - ref) <= 1e-11 * np.linalg.norm(ref) * np.linalg.cond(A)
        d = np.abs(np.diag(sla.lu_factor(A)[0]))
        assert abs(r - d.min() / d.max()) <= 1e-10 * (d.min() / d.max())


@pytest.mark.parametrize("n", [513, 849, 1100, 1600, 2532, 3100])
def test_getrf_blocked_panel_classes(n):
    """Blocked LU (shared-memory panels of 64/32/16/8 columns by order):
    backward error of the solve, pivot ratio and interchanges against LAPACK."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    Bm = rng.standard_normal((n, 2))
    dA, dB = _dev(A), _dev(Bm)
    ip = torch.empty(n, dtype=torch.int32, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    ratio = torch.empty(1, dtype=torch.float64, device="cuda")
    m = skel._mats(np.array([dA.data_ptr()], np.uint64), [n], [n], [n])
    call("skb_getrf_batched", 1, m, np.array([ip.data_ptr()], np.uint64), info, ratio, skel._stream())
    call("skb_getrs_batched", 1, m, np.array([ip.data_ptr()], np.uint64),
         skel._mats(np.array([dB.data_ptr()], np.uint64), [n], [2], [2]), skel._stream())
    torch.cuda.synchronize()
    assert int(info.cpu()[0]) == -1
    x = dB.cpu().numpy()
    berr = np.linalg.norm(A @ x - Bm) / (np.linalg.norm(A) * np.linalg.norm(x))
    assert berr < 1e-14, berr
    lu, piv = sla.lu_factor(A)
    d = np.abs(np.diag(lu))
    assert abs(float(ratio.cpu()[0]) - d.min() / d.max()) <= 1e-6 * (d.min() / d.max())
    # partial pivoting on a random matrix: same interchanges as LAPACK
    assert np.array_equal(ip.cpu().numpy(), piv.astype(np.int32))


def test_getrf_singular_reports_index():
    A = np.array([[1.0, 2.0], [2.0, 4.0]])
    dA = _dev(A)
    ip = torch.empty(2, dtype=torch.int32, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    ratio = torch.empty(1, dtype=torch.float64, device="cuda")
    call("skb_getrf_batched", 1, skel._mats(np.array([dA.data_ptr()], np.uint64), [2], [2], [2]),
         np.array([ip.data_ptr()], np.uint64), info, ratio, skel._stream())
    assert int(info.cpu()[0]) == 1     # reference SPEC.md:194-197: SingularPivotError index 1


@pytest.mark.parametrize("n", [300, 849])
def test_getrf_blocked_zero_column(n):
    """Blocked panel path: an exactly zero column reports its (0-based) index
    and leaves the other columns' interchanges LAPACK-identical up to it."""
    rng = np.random.default_rng(7 + n)
    A = rng.standard_normal((n, n))
    z = n - 37
    A[:, z] = 0.0
    dA = _dev(A)
    ip = torch.empty(n, dtype=torch.int32, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    ratio = torch.empty(1, dtype=torch.float64, device="cuda")
    call("skb_getrf_batched", 1, skel._mats(np.array([dA.data_ptr()], np.uint64), [n], [n], [n]),
         np.array([ip.data_ptr()], np.uint64), info, ratio, skel._stream())
    torch.cuda.synchronize()
    assert int(info.cpu()[0]) == z
    _, piv = sla.lu_factor(A, check_finite=False)
    assert np.array_equal(ip.cpu().numpy()[:z], piv[:z].astype(np.int32))


def _golden_boxes(g, prefix):
    keys = [tuple(k) for k in g[prefix + "keys"]]
    out = {}
    for i, k in enumerate(keys):
        def sl(a):
            return g[prefix + a][g[prefix + a + "_off"][i]:g[prefix + a + "_off"][i + 1]]
        out[k] = dict(act=sl("act"), far=sl("far"), S=sl("S"), k=int(g[prefix + "k"][i]))
    return out


def _ulp_diff(a, b):
    ai = a.view(np.int64)
    bi = b.view(np.int64)
    return np.abs(ai - bi)


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_stack_assembly_bitwise(golden, name, builder):
    """(a) GPU ID stacks vs the reference's np.vstack(blocks): bitwise except the
    log()-containing Stokeslet proxy rows (<= 2 ulp)."""
    wl = builder()
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ctx = skel._Ctx(skel.SystemSpec(), wl.boundary, t, wl.tol, wl.proxy_count, wl.proxy_factor)
    ref = _golden_boxes(golden, name)
    i = 0
    while name + f"stack{i}_key" in golden.files:
        key = tuple(golden[name + f"stack{i}_key"])
        S_ref = golden[name + f"stack{i}"]
        bi = t.index(key)
        act_of = {j: ref[t.key(j)]["act"] for j in range(len(t.lev)) if t.key(j) in ref}
        idx = np.array([bi])
        act_off, act = skel._csr([act_of[bi]])
        far_off, far = ctx.far_lists(idx, skel.ActStore.replay(t, act_of))
        pts, pn, pw = ctx.proxies(idx)
        nB, nF, P = len(act), len(far), wl.proxy_count
        rows = 2 * nF + 6 * P + 2
        st = torch.empty(rows * nB, dtype=torch.float64, device="cuda")
        up = skel._upload(ao=act_off, a=act, fo=far_off, f=far if nF else np.zeros(1, np.int64),
                          pts=pts.reshape(-1), pn=pn.reshape(-1), pw=pw, so=np.zeros(1, np.int64))
        g = ctx.g
        call("skb_assemble_stack", g.pos, g.nrm, g.w, 1, up["ao"], up["a"], up["fo"], up["f"],
             up["pts"], up["pn"], up["pw"], P, up["so"], st, nB, nF + P + 1, skel._stream())
        got = st.cpu().numpy().reshape(nB, rows).T
        assert got.shape == S_ref.shape
        ul = _ulp_diff(got, S_ref)
        log_rows = np.zeros(rows, bool)
        log_rows[2 * nF + 4 * P + 1: 2 * nF + 6 * P + 1] = True
        assert ul[~log_rows].max() == 0, (key, ul[~log_rows].max())
        assert ul[log_rows].max() <= 4, (key, ul[log_rows].max())
        i += 1


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_self_block_bitwise(name, builder):
    """(a) Self blocks E = A[B, B] vs the oracle (bitwise) for leaf boxes."""
    wl = builder()
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ctx = skel._Ctx(skel.SystemSpec(), wl.boundary, t, wl.tol, wl.proxy_count, wl.proxy_factor)
    idx = t.level_indices(t.depth)[:4]
    lists = [(2 * t.nodes_of(i)[:, None] + np.arange(2)).ravel() for i in idx]
    ao, a = skel._csr(lists)
    nB = np.diff(ao)
    eo = np.concatenate([[0], np.cumsum(nB * nB)])
    E = torch.empty(int(eo[-1]), dtype=torch.float64, device="cuda")
    co = np.full((len(idx), 5), -1, np.int64)
    cx = np.zeros((len(idx), 4), np.uint64)
    up = skel._upload(ao=ao, a=a, co=co.reshape(-1), cx=cx.reshape(-1), eo=eo[:-1], eld=nB)
    g = ctx.g
    call("skb_assemble_self", g.pos, g.nrm, g.w, g.kap, len(idx), up["ao"], up["a"], None, None,
         up["co"], up["cx"], E, up["eo"], up["eld"], int(nB.max()), skel._stream())
    En = E.cpu().numpy()
    for bi, lst in enumerate(lists):
        ref = O.self_block(wl.boundary, lst, lst)
        got = En[eo[bi]:eo[bi + 1]].reshape(nB[bi], nB[bi])
        assert np.array_equal(got, ref)


def _replay_ids(wl, ref):
    """Run the ID part (GPU stack -> Householder -> QRCP) of every box on the
    reference's exact active sets, level by level; returns the boxes whose
    skeleton (set and order) differs: (key, k_gpu, k_ref, gpu min pivot gap,
    reference threshold margin)."""
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ctx = skel._Ctx(skel.SystemSpec(), wl.boundary, t, wl.tol, wl.proxy_count, wl.proxy_factor)
    act_of = {j: ref[t.key(j)]["act"] for j in range(len(t.lev)) if t.key(j) in ref}
    store = skel.ActStore.replay(t, act_of)
    mism = []
    for lev in range(t.depth, 0, -1):
        idx = t.level_indices(lev)
        B = len(idx)
        act_off, act = skel._csr([act_of[int(i)] for i in idx])
        nB = np.diff(act_off)
        far_off, far = ctx.far_lists(idx, store)
        nF = np.diff(far_off)
        pts, pn, pw = ctx.proxies(idx)
        P = wl.proxy_count
        rows = 2 * nF + 6 * P + 2
        so = np.concatenate([[0], np.cumsum(rows * nB)])
        st = torch.empty(int(so[-1]), dtype=torch.float64, device="cuda")
        up = skel._upload(ao=act_off, a=act, fo=far_off, f=far if len(far) else np.zeros(1, np.int64),
                          pts=pts.reshape(-1), pn=pn.reshape(-1), pw=pw, so=so[:-1])
        g = ctx.g
        s = skel._stream()
        call("skb_assemble_stack", g.pos, g.nrm, g.w, B, up["ao"], up["a"], up["fo"], up["f"],
             up["pts"], up["pn"], up["pw"], P, up["so"], st, int(nB.max()), int((nF + P + 1).max()), s)
        A = (st.data_ptr() + 8 * so[:-1]).astype(np.int64)
        pre = rows > 2 * nB                      # dense.py:56
        if pre.any():
            call("skb_geqrf_batched", int(pre.sum()), np.ascontiguousarray(rows[pre]),
                 np.ascontiguousarray(nB[pre]), np.ascontiguousarray(rows[pre]),
                 np.ascontiguousarray(A[pre]), s)
        mq = np.where(pre, nB, rows).astype(np.int64)
        perm = torch.empty(len(act), dtype=torch.int32, device="cuda")
        diag = torch.empty(len(act), dtype=torch.float64, device="cuda")
        ko = torch.empty(2 * B, dtype=torch.int32, device="cuda")
        gap = torch.empty(B, dtype=torch.float64, device="cuda")
        call("skb_qrcp_id_batched", B, mq, nB.astype(np.int64), rows.astype(np.int64), A,
             np.zeros(B, np.int64), wl.tol, act_off, perm, diag, ko, ko.data_ptr() + 4 * B, gap, s)
        pm = perm.cpu().numpy()
        kk = ko.cpu().numpy()[:B]
        gp = gap.cpu().numpy()
        for bi, i in enumerate(idx):
            r = ref[t.key(i)]
            S = pm[act_off[bi]:act_off[bi] + kk[bi]]
            if kk[bi] != r["k"] or not np.array_equal(S, r["S"]):
                margin = np.inf
                d = r.get("diag")
                if d is not None and len(d) and d[0] > 0:
                    thr = wl.tol * abs(d[0])
                    near = [abs(abs(d[j]) / thr - 1.0) for j in (r["k"] - 1, r["k"]) if 0 <= j < len(d)]
                    margin = min(near) if near else np.inf
                mism.append((t.key(i), int(kk[bi]), r["k"], float(gp[bi]), float(margin)))
    return mism


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_id_replay_skeletons(golden, name, builder):
    """(b) Replay every box on the reference's exact active sets: GPU stack ->
    Householder -> QRCP must select the reference's skeleton (same order)."""
    mism = _replay_ids(builder(), _golden_boxes(golden, name))
    # a mismatch is acceptable only as a pivot tie within rounding
    untied = [m for m in mism if m[3] > 1e-12]
    assert not untied, untied
    assert not mism, mism      # these fixtures are tie-free


def test_id_replay_tie_rich_cfg2(golden):
    """Tie-rich fixture (unphased cfg2: equispaced circles centred on quadtree
    axes give exact pivot ties): per-level replay of every box on the
    reference's active sets.  Every skeleton that differs from the reference's
    must be a tie within rounding -- GPU minimum relative pivot gap <= 1e-12 --
    or a rank decided within rounding of the threshold (|R_kk| within 1e-10 of
    tol |R_00|); SURVEY.md §8(c) item 1."""
    wl = configs.cfg2(phases=False)
    keys = [tuple(k) for k in golden["cfg2u_keys"]]
    ref = {}
    for i, k in enumerate(keys):
        seg = lambda nm: golden[f"cfg2u_{nm}"][golden[f"cfg2u_{nm}_off"][i]:golden[f"cfg2u_{nm}_off"][i + 1]]
        ref[k] = dict(act=seg("act"), S=seg("S"), diag=seg("diag"), k=int(golden["cfg2u_k"][i]))
    mism = _replay_ids(wl, ref)
    print(f"unphased cfg2: {len(keys) - len(mism)}/{len(keys)} boxes with the reference's skeleton "
          f"on replay; mismatches (key, k_gpu, k_ref, gap, margin): {mism}")
    untied = [m for m in mism if m[3] > 1e-12 and m[4] > 1e-10]
    assert not untied, untied


@pytest.mark.parametrize("m,n", [(40, 17), (300, 100), (700, 130), (1500, 200), (2400, 96), (520, 384)])
def test_geqrf_batched_R(m, n):
    """Batched Householder pre-reduction: R^T R == A^T A and |diag(R)| matches LAPACK."""
    rng = np.random.default_rng(m + n)
    As = [rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -12, n)), rng.standard_normal((m, n))]
    dev = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in As]   # column-major
    ptrs = np.array([d.data_ptr() for d in dev], np.int64)
    mm = np.full(2, m, np.int64)
    nn = np.full(2, n, np.int64)
    call("skb_geqrf_batched", 2, mm, nn, mm, ptrs, skel._stream())
    torch.cuda.synchronize()
    for a, d in zip(As, dev):
        R = d.cpu().numpy().T[:n, :n]
        assert np.allclose(np.tril(R, -1), 0.0)
        Rref = sla.qr(a, mode="r")[0][:n]
        assert np.allclose(np.abs(np.diag(R)), np.abs(np.diag(Rref)), rtol=1e-9, atol=1e-14 * np.abs(Rref).max())
        assert np.allclose(np.abs(R), np.abs(Rref), rtol=1e-9, atol=1e-12 * np.abs(Rref).max())


def test_gemm_bits_independent_of_tile_and_n():
    """Each output element is one thread's fixed-K-order DMMA chain: the 64x64
    and 128x128 tile variants and any column subset give identical bits (the
    update path's incremental sweep relies on it)."""
    import subprocess, sys, os
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2001_11619_b200 import skel
rng = np.random.default_rng(1)
m, n, k = 300, 200, 250
A, B, C = (torch.from_numpy(rng.standard_normal(s)).cuda() for s in ((m, k), (k, n), (m, n)))
outs = []
for cols in (n, 37):
    D = torch.empty((m, n), dtype=torch.float64, device="cuda")
    skel._gemm([dict(A=np.array([A.data_ptr()], np.uint64), B=np.array([B.data_ptr()], np.uint64),
                     C=np.array([C.data_ptr()], np.uint64), D=np.array([D.data_ptr()], np.uint64),
                     m=[m], n=[cols], k=[k], lda=[k], ldb=[n], ldc=[n], ldd=[n], alpha=[-1.0], beta=[1.0])])
    outs.append(D[:, :37].cpu().numpy())
np.save(sys.argv[1], np.stack(outs))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for tile in ("64", "128"):
        out = f"/tmp/skb_gemm_{tile}.npy"
        env = dict(os.environ, SKB_GEMM_TILE=tile)
        subprocess.run([sys.executable, "-c", code, out], check=True, env=env)
        res.append(np.load(out))
    assert np.array_equal(res[0][0], res[0][1])       # n = 200 vs n = 37
    assert np.array_equal(res[0], res[1])             # 64x64 vs 128x128 tiles


def test_laplace_stack_and_self_block_bitwise(golden):
    """Laplace-Neumann branch: the GPU ID stack of a leaf box equals the
    reference's np.vstack(blocks) bitwise except the log() proxy rows
    (<= 4 ulp); self blocks equal the oracle's Laplace eval_block bitwise."""
    wl = configs.cfg1()
    spec = skel.SystemSpec(skel.LAPLACE)
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ctx = skel._Ctx(spec, wl.boundary, t, wl.tol, wl.proxy_count, wl.proxy_factor)
    ref = _golden_boxes(golden, "lap_")
    key = tuple(golden["lap_stack0_key"])
    S_ref = golden["lap_stack0"]
    bi = t.index(key)
    act_of = {j: ref[t.key(j)]["act"] for j in range(len(t.lev)) if t.key(j) in ref}
    idx = np.array([bi])
    act_off, act = skel._csr([act_of[bi]])
    far_off, far = ctx.far_lists(idx, skel.ActStore.replay(t, act_of, dpn=1))
    assert np.array_equal(far, ref[key]["far"])
    pts, pn, pw = ctx.proxies(idx)
    nB, nF, P = len(act), len(far), wl.proxy_count
    rows = 2 * nF + 2 * P + 2
    st = torch.empty(rows * nB, dtype=torch.float64, device="cuda")
    up = skel._upload(ao=act_off, a=act, fo=far_off, f=far if nF else np.zeros(1, np.int64),
                      pts=pts.reshape(-1), pn=pn.reshape(-1), pw=pw, so=np.zeros(1, np.int64))
    g = ctx.g
    call("skb_assemble_stack_lap", g.pos, g.nrm, g.w, 1, up["ao"], up["a"], up["fo"], up["f"],
         up["pts"], up["pn"], up["pw"], P, up["so"], st, nB, nF + P + 1, skel._stream())
    got = st.cpu().numpy().reshape(nB, rows).T
    assert got.shape == S_ref.shape
    ul = _ulp_diff(got, S_ref)
    log_rows = np.zeros(rows, bool)
    log_rows[nF:nF + P] = True
    assert ul[~log_rows].max() == 0
    assert ul[log_rows].max() <= 4
    # self blocks of 4 leaf boxes
    idx = t.level_indices(t.depth)[:4]
    lists = [t.nodes_of(i).astype(np.int64) for i in idx]
    ao, a = skel._csr(lists)
    nBs = np.diff(ao)
    eo = np.concatenate([[0], np.cumsum(nBs * nBs)])
    E = torch.empty(int(eo[-1]), dtype=torch.float64, device="cuda")
    co = np.full((len(idx), 5), -1, np.int64)
    cx = np.zeros((len(idx), 4), np.uint64)
    up = skel._upload(ao=ao, a=a, co=co.reshape(-1), cx=cx.reshape(-1), eo=eo[:-1], eld=nBs)
    call("skb_assemble_self_lap", g.pos, g.nrm, g.w, g.kap, len(idx), up["ao"], up["a"], None, None,
         up["co"], up["cx"], E, up["eo"], up["eld"], int(nBs.max()), skel._stream())
    En = E.cpu().numpy()
    for bi_, lst in enumerate(lists):
        refE = O.lap_self_block(wl.boundary, lst, lst)
        assert np.array_equal(En[eo[bi_]:eo[bi_ + 1]].reshape(nBs[bi_], nBs[bi_]), refE)


def test_move_kernels_bit_exact():
    """skb_copy2d_batched / skb_gather_rows / skb_scatter_rows move bytes only:
    bit-exact against NumPy indexing over compact / strided / unaligned / odd /
    empty shapes, with and without column lists, narrow and wide rows."""
    from paper_2001_11619_b200._lib import MAT_DT, ptr
    rng = np.random.default_rng(3)
    s = skel._stream()
    # -- copy2d: (rows, cols, ld_dst, ld_src, element offset of the source block)
    pool = _dev(rng.standard_normal(400000))
    cases = [(7, 5, 5, 5, 0), (7, 5, 5, 5, 1), (64, 64, 64, 64, 2), (33, 17, 40, 23, 3),
             (1, 1, 1, 1, 0), (200, 129, 129, 129, 7), (0, 4, 4, 4, 0), (117, 117, 117, 117, 100)]
    for trans in (0, 1):
        dst_t, ms_d, ms_s, refs = [], [], [], []
        off = 0
        for (r, c, ldd, lds, so) in cases:
            src_rows, src_cols = (c, r) if trans else (r, c)
            lds_eff = max(lds, src_cols)
            sview = pool[off + so: off + so + src_rows * lds_eff].view(src_rows, lds_eff) if src_rows else None
            off += so + src_rows * lds_eff + 8
            d = torch.full((max(r, 1), max(ldd, c, 1)), -7.0, dtype=torch.float64, device="cuda")
            dst_t.append(d)
            ms_d.append((d.data_ptr(), r, c, d.shape[1]))
            ms_s.append((sview.data_ptr() if sview is not None else pool.data_ptr(), src_rows, src_cols, lds_eff))
            if r and c:
                sv = sview[:, :src_cols].cpu().numpy()
                refs.append(sv.T.copy() if trans else sv.copy())
            else:
                refs.append(None)
        md = np.array(ms_d, dtype=[("ptr", "u8"), ("rows", "i8"), ("cols", "i8"), ("ld", "i8")]).astype(MAT_DT)
        msr = np.array(ms_s, dtype=[("ptr", "u8"), ("rows", "i8"), ("cols", "i8"), ("ld", "i8")]).astype(MAT_DT)
        call("skb_copy2d_batched", len(cases), md, msr, trans, s)
        torch.cuda.synchronize()
        for d, (r, c, *_), ref in zip(dst_t, cases, refs):
            if ref is None:
                continue
            got = d.cpu().numpy()
            assert np.array_equal(got[:r, :c], ref)
            assert np.all(got[:r, c:] == -7.0)
    # -- gather / scatter rows
    for nrows_src, ncols in ((500, 3), (500, 48), (300, 129), (200, 256), (100, 770)):
        X = rng.standard_normal((nrows_src, ncols))
        dX = _dev(X)
        B = 5
        perm_all = rng.permutation(nrows_src)               # disjoint row sets (as in the sweeps)
        cuts = np.cumsum([0, 0, 1, 33, 64, 97])
        lists = [perm_all[cuts[j]:cuts[j + 1]] for j in range(5)]
        idx_off = np.zeros(B + 1, np.int64)
        np.cumsum([len(l) for l in lists], out=idx_off[1:])
        idx = np.concatenate(lists).astype(np.int64)
        for use_cols in (False, True):
            if use_cols:
                cl = [np.sort(rng.permutation(ncols)[:max(1, (b * ncols) // 6)]) for b in range(B)]
                col_off = np.zeros(B + 1, np.int64)
                np.cumsum([len(c) for c in cl], out=col_off[1:])
                colv = np.concatenate(cl).astype(np.int64)
                widths = np.array([len(c) for c in cl], np.int64)
            else:
                cl = [np.arange(ncols)] * B
                widths = np.full(B, ncols, np.int64)
            ld = widths + np.array([0, 1, 0, 2, 0])          # odd leading dimensions too
            sizes = np.array([len(l) for l in lists], np.int64) * ld
            dst_off = np.zeros(B, np.int64)
            np.cumsum(sizes[:-1] + np.array([1, 0, 3, 0]), out=dst_off[1:])   # odd offsets
            buf = torch.full((int(dst_off[-1] + sizes[-1]) + 8,), -3.0, dtype=torch.float64, device="cuda")
            d_io, d_idx, d_do, d_ld = _dev(idx_off), _dev(idx if len(idx) else np.zeros(1, np.int64)), _dev(dst_off), _dev(ld)
            d_cols = (_dev(col_off), _dev(colv)) if use_cols else None      # kept alive for the calls
            args_c = (ptr(d_cols[0]), ptr(d_cols[1])) if use_cols else (None, None)
            call("skb_gather_rows", B, ptr(d_io), ptr(d_idx), args_c[0], args_c[1], ncols, ptr(dX), ncols,
                 ptr(buf), ptr(d_do), ptr(d_ld), 97, int(widths.max()), s)
            torch.cuda.synchronize()
            got = buf.cpu().numpy()
            for b in range(B):
                n = len(lists[b])
                blk = got[dst_off[b]: dst_off[b] + n * ld[b]].reshape(n, ld[b])
                assert np.array_equal(blk[:, :widths[b]], X[lists[b]][:, cl[b]])
                assert np.all(blk[:, widths[b]:] == -3.0)
            # scatter back into a fresh array (plain store, then accumulate with alpha)
            Y0 = rng.standard_normal((nrows_src, ncols))
            for acc, alpha in ((0, 1.0), (1, -0.5)):
                dY = _dev(Y0)
                call("skb_scatter_rows", B, ptr(d_io), ptr(d_idx), args_c[0], args_c[1], ncols, ptr(buf),
                     ptr(d_do), ptr(d_ld), ptr(dY), ncols, acc, alpha, 97, int(widths.max()), s)
                torch.cuda.synchronize()
                ref = Y0.copy()
                for b in range(B):
                    if len(lists[b]) == 0:
                        continue
                    sub = X[lists[b]][:, cl[b]]
                    if acc:
                        ref[np.ix_(lists[b], cl[b])] = ref[np.ix_(lists[b], cl[b])] + alpha * sub
                    else:
                        ref[np.ix_(lists[b], cl[b])] = sub
                assert np.array_equal(dY.cpu().numpy(), ref)


def _qrcp_call(mats, tol):
    """skb_qrcp_id_batched on a list of equal-shape host matrices; returns (perm, k, steps, diag)."""
    nbox = len(mats)
    m, n = mats[0].shape
    flat = np.concatenate([A.T.ravel() for A in mats])
    d = _dev(flat)
    A = (d.data_ptr() + 8 * np.arange(nbox, dtype=np.int64) * (m * n)).astype(np.int64)
    act_off = np.arange(nbox + 1, dtype=np.int64) * n
    perm = torch.empty(nbox * n, dtype=torch.int32, device="cuda")
    diag = torch.empty(nbox * n, dtype=torch.float64, device="cuda")
    ko = torch.empty(2 * nbox, dtype=torch.int32, device="cuda")
    gap = torch.empty(nbox, dtype=torch.float64, device="cuda")
    call("skb_qrcp_id_batched", nbox, np.full(nbox, m, np.int64), np.full(nbox, n, np.int64),
         np.full(nbox, m, np.int64), A, np.zeros(nbox, np.int64), tol, act_off, perm, diag, ko,
         ko.data_ptr() + 4 * nbox, gap, skel._stream())
    torch.cuda.synchronize()
    kk = ko.cpu().numpy()
    return perm.cpu().numpy().reshape(nbox, n), kk[:nbox], kk[nbox:], diag.cpu().numpy().reshape(nbox, n)


def test_qrcp_blocked_cooperative_vs_lapack():
    """k_qrcp_blk (dlaqps-style delayed updates, R in L2, cooperative launch):
    on matrices with a decaying spectrum whose R does not fit a 16-CTA cluster,
    rank and skeleton (order included) equal SciPy's dgeqp3 at the tolerance,
    |diag R| matches to 1e-12 |R_00|, and repeated runs are bitwise identical."""
    rng = np.random.default_rng(5)
    tol, m, n, k = 1e-8, 1400, 900, 90
    mats = []
    for _ in range(2):
        U, _ = np.linalg.qr(rng.standard_normal((m, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        mats.append((U * 10.0 ** (-8.0 * np.arange(n) / k)) @ V.T)
    runs = [_qrcp_call(mats, tol) for _ in range(3)]
    pm, kk, steps, dg = runs[0]
    for other in runs[1:]:
        assert np.array_equal(other[1], kk) and np.array_equal(other[2], steps)
        for b in range(2):
            assert np.array_equal(other[0][b, :kk[b]], pm[b, :kk[b]])
            assert np.array_equal(other[3][b, :steps[b]], dg[b, :steps[b]])
    for b, A in enumerate(mats):
        _, R, p = sla.qr(A, mode="economic", pivoting=True)
        d = np.abs(np.diag(R))
        kr = int(np.count_nonzero(d > tol * d[0]))
        assert kk[b] == kr
        assert np.array_equal(pm[b, :kr], p[:kr])
        assert np.allclose(dg[b, :kr], d[:kr], rtol=1e-9, atol=1e-12 * d[0])   # absolute: eps-level in |A|
        assert sorted(pm[b]) == list(range(n))          # a permutation: every column listed once

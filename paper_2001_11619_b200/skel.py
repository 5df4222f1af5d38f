"""Level-batched recursive skeletonization on one B200 -- the drop-in for the
reference's ``factor`` / ``update`` / ``Factorization.solve`` / ``apply``
(``/root/reference/pkg/src/skelsolve/skel.py``).

Host Python keeps only the bookkeeping the reference does in Python (tree,
active/far DOF lists, proxy rings, dirty sets); every floating-point operation
of the factorization runs in libskelb200.so kernels on the device, one batched
call per quadtree level:

  per level (bottom-up, skel.py:445-449):
    (a) ID stacks of all boxes          skb_assemble_stack     (skel.py:297-314)
    (b) Householder pre-reduction       skb_geqrf_batched      (dense.py:56-59)
        pivoted QR, rank, T             skb_qrcp_id_batched    (dense.py:48-79, skel.py:314-319)
    (a) permuted self blocks            skb_assemble_self      (skel.py:282-291,316)
    (c) Schur blocks                    skb_gemm_grouped       (skel.py:320-334)
        X_RR LU / X_RR^-1 X_RS          skb_getrf/getrs        (skel.py:324,333)
  _finish_top (skel.py:364-425):
    (d) H, Psi + per-level U/V^T sweeps + deterministic q x q Schur + corner LU.

Factor data stay resident in HBM; ``Factorization.factors[key]`` materialises
a reference-style ``BoxFactors`` view (host copies) on demand.
"""

from __future__ import annotations

import ctypes
import gc
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import GEMM_DT, MAT_DT, call, ptr
from .tree import Tree, build_tree, dirty_mask, proxy_radius, refit_tree

PIVOT_RATIO_FLOOR = 1e-12          # skel.py:46
DEFAULT_PROXY_COUNT = 64           # skel.py:47
DEFAULT_PROXY_FACTOR = 1.5         # skel.py:48
STOKES = "stokes_dirichlet"        # kernels.py:36
LAPLACE = "laplace_neumann"        # kernels.py:35


class SingularPivotError(RuntimeError):
    """Exact zero pivot (reference dense.py:18-23)."""

    def __init__(self, index: int):
        super().__init__(f"zero pivot at elimination step {index}")
        self.index = index


class RootBoxExceededError(RuntimeError):
    """A perturbed node escaped the fixed root box (reference skel.py:51-52)."""


@dataclass(frozen=True)
class SystemSpec:
    """PDE / kernel selection (reference kernels.py:41-63): the Stokes
    double layer with the multiply-connected augmentation, or the
    Laplace-Neumann adjoint double layer (one DOF per node, never augmented)."""

    pde: str = STOKES

    def __post_init__(self):
        if self.pde not in (LAPLACE, STOKES):
            raise ValueError(f"unknown pde {self.pde!r}")

    @property
    def dof_per_node(self) -> int:
        return 2 if self.pde == STOKES else 1

    @property
    def jump_coefficient(self) -> float:
        return -0.5                 # kernels.py:38

    @property
    def code(self) -> int:
        """C-ABI pde code: 0 Stokes, 1 Laplace."""
        return 0 if self.pde == STOKES else 1

    def augmented(self, b) -> bool:
        return self.pde == STOKES and b.n_holes >= 1

    def n_dofs(self, b) -> int:
        return self.dof_per_node * b.n_nodes


# ---------------------------------------------------------------------------
# small helpers
# ---------------------------------------------------------------------------
_DEV_INDEX = []


def _stream():
    """Raw handle of the current stream (torch's Python-level current_stream()
    costs ~20 us per call; the level loops ask for it hundreds of times)."""
    if not _DEV_INDEX:
        _DEV_INDEX.append(torch.cuda.current_device())
    return torch._C._cuda_getCurrentRawStream(_DEV_INDEX[0])


_LEVEL_STREAM = []


def _level_stream() -> torch.cuda.Stream:
    """Stream of the per-level Schur-complement work (created once)."""
    if not _LEVEL_STREAM:
        _LEVEL_STREAM.append(torch.cuda.Stream())
        # the compression chain (stack -> QR -> QRCP -> host sync) is the
        # critical path: it runs on a high-priority stream
        _LEVEL_STREAM.append(torch.cuda.Stream(priority=-1))
    return _LEVEL_STREAM[0]


def _aug_stream() -> torch.cuda.Stream:
    _level_stream()
    if len(_LEVEL_STREAM) < 3:
        _LEVEL_STREAM.append(torch.cuda.Stream())
    return _LEVEL_STREAM[2]


def _compress_stream() -> torch.cuda.Stream:
    _level_stream()
    return _LEVEL_STREAM[1]


class _HostTimer:
    """Host-only time per section (SKB_HOST_PROF=1; no device syncs)."""

    enabled = bool(os.environ.get("SKB_HOST_PROF"))
    trace = os.environ.get("SKB_HOST_PROF") == "trace"     # record_function ranges (timeline.py)
    acc: dict = {}

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.t0 = time.perf_counter()

    def __exit__(self, *a):
        a_ = _HostTimer.acc
        a_[self.name] = a_.get(self.name, 0.0) + time.perf_counter() - self.t0


class _Null:
    def __enter__(self):
        pass

    def __exit__(self, *a):
        pass


_NULL = _Null()


def _ht(name):
    if _HostTimer.trace:
        return torch.profiler.record_function(name)
    return _HostTimer(name) if _HostTimer.enabled else _NULL


class _Prof:
    """Optional per-stage wall-clock breakdown (SKB_PROFILE=1 synchronises
    after every stage; off by default so the pipeline stays asynchronous)."""

    enabled = bool(int(__import__("os").environ.get("SKB_PROFILE", "0")))
    acc: dict = {}
    _t = 0.0
    _lt = 0.0

    @classmethod
    def start(cls):
        if cls.enabled:
            torch.cuda.synchronize()
            cls._t = time.perf_counter()

    @classmethod
    def tick(cls, name):
        if cls.enabled:
            torch.cuda.synchronize()
            t = time.perf_counter()
            cls.acc[name] = cls.acc.get(name, 0.0) + t - cls._t
            cls._t = t

    @classmethod
    def reset(cls):
        cls.acc = {}


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2001_11619_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _csr(arrays):
    lens = np.fromiter((len(a) for a in arrays), dtype=np.int64, count=len(arrays))
    off = np.zeros(len(arrays) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    flat = np.concatenate(arrays).astype(np.int64) if len(arrays) else np.zeros(0, np.int64)
    return off, flat


IO = {"h2d": 0, "d2h": 0, "wait_s": 0.0, "waits": 0}   # host<->device traffic / host waits


def _d2h(t: torch.Tensor) -> np.ndarray:
    IO["d2h"] += t.numel() * t.element_size()
    t0 = time.perf_counter()
    out = t.cpu().numpy()
    IO["wait_s"] += time.perf_counter() - t0
    IO["waits"] += 1
    return out


def _seg_gather(src, starts, lens):
    """Concatenate src[starts[j]:starts[j]+lens[j]] for all j (vectorised)."""
    lens = np.asarray(lens, np.int64)
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    tot = int(off[-1])
    if tot == 0:
        return off, src[:0].copy()
    idx = np.repeat(np.asarray(starts, np.int64) - off[:-1], lens) + np.arange(tot)
    return off, src[idx]


class ActStore:
    """Active / skeleton DOF lists of every tree box as segments of one flat
    array (vectorised replacement of the reference's per-box ``bx.active`` /
    ``bx.skel`` arrays, skel.py:243-256)."""

    def __init__(self, t: Tree, engine: bool = False, dpn: int = 2):
        nbox = len(t.lev)
        cap = 2 * t.n_nodes * (t.depth + 3) + 16
        if engine:
            # the native engine appends in place (no reallocation): active sets
            # and skeletons of every level, <= 2 x 2N per level
            cap = 2 * t.n_nodes * (2 * t.depth + 3) + 16
        self.big = np.empty(cap, np.int64)
        self.fill = 0
        self.s_start = np.zeros(nbox, np.int64)
        self.s_len = np.zeros(nbox, np.int64)
        self.xss = np.zeros(nbox, np.uint64)
        init = getattr(t, f"_store_init{dpn}", None)    # leaf actives depend on the tree only
        if init is not None:
            fill, a_start, a_len, prefix = init
            self.big[:fill] = prefix
            self.fill = fill
            self.a_start, self.a_len = a_start.copy(), a_len.copy()
            return
        self.a_start = np.zeros(nbox, np.int64)
        self.a_len = np.zeros(nbox, np.int64)
        flat = getattr(t, "_level_nodes_flat", None)
        if flat is not None:
            # trees of the native build: leaf actives in the native host runtime
            nv = _tree_native(t)
            fill = _lib.load().skb_host_leaf_actives(
                nbox, t.depth, nv["lev"].ctypes.data, nv["leaf"].ctypes.data,
                t.node_start.ctypes.data, t.node_cnt.ctypes.data, flat.ctypes.data,
                t._level_nodes_off.ctypes.data, nv["ls"].ctypes.data, dpn, self.big.ctypes.data,
                len(self.big), self.a_start.ctypes.data, self.a_len.ctypes.data)
            if fill < 0:
                raise RuntimeError("active-set store too small")
            self.fill = int(fill)
            setattr(t, f"_store_init{dpn}",
                    (self.fill, self.a_start.copy(), self.a_len.copy(), self.big[:self.fill].copy()))
            return
        leaves = np.flatnonzero(t.is_leaf)
        # leaf actives: dofs 2*node + {0,1} of the sorted owned nodes (skel.py:243-249)
        for l in range(t.depth + 1):
            li = leaves[t.lev[leaves] == l]
            if len(li) == 0:
                continue
            off, nodes = _seg_gather(t.level_nodes[l], t.node_start[li], t.node_cnt[li])
            dofs = (dpn * nodes[:, None] + np.arange(dpn)[None, :]).ravel()   # skel.py:243-244
            self.a_start[li] = self._append(dofs) + dpn * off[:-1]
            self.a_len[li] = dpn * t.node_cnt[li]
        setattr(t, f"_store_init{dpn}",
                (self.fill, self.a_start.copy(), self.a_len.copy(), self.big[:self.fill].copy()))

    @classmethod
    def replay(cls, t: Tree, act_of: dict, dpn: int = 2) -> "ActStore":
        """Store with given active sets (per-level replay of recorded inputs)."""
        st = cls(t, dpn=dpn)
        for i, a in act_of.items():
            st.a_start[i] = st._append(np.asarray(a, np.int64))
            st.a_len[i] = len(a)
        return st

    def _append(self, arr):
        n = len(arr)
        if self.fill + n > len(self.big):
            nb = np.empty(max(2 * len(self.big), self.fill + n), np.int64)
            nb[:self.fill] = self.big[:self.fill]
            self.big = nb
        o = self.fill
        self.big[o:o + n] = arr
        self.fill += n
        return o

    def act(self, i):
        return self.big[self.a_start[i]:self.a_start[i] + self.a_len[i]]

    def skel(self, i):
        return self.big[self.s_start[i]:self.s_start[i] + self.s_len[i]]

    def acts(self, idx):
        return _seg_gather(self.big, self.a_start[idx], self.a_len[idx])

    def set_internal(self, t: Tree, idx):
        """Internal boxes: active = concat of children's skeletons in child order."""
        idx = np.asarray(idx, np.int64)
        idx = idx[~t.is_leaf[idx]]
        if len(idx) == 0:
            return
        ch = t.children[idx]
        valid = ch >= 0
        cflat = ch[valid]
        off, dofs = _seg_gather(self.big, self.s_start[cflat], self.s_len[cflat])
        base = self._append(dofs)
        lens = np.where(valid, self.s_len[np.maximum(ch, 0)], 0)
        tot = lens.sum(axis=1)
        st = np.zeros(len(idx), np.int64)
        np.cumsum(tot[:-1], out=st[1:])
        self.a_start[idx] = base + st
        self.a_len[idx] = tot

    def set_skel(self, idx, act_off, act, perm, k):
        """skel = act[perm[:k]] per box (vectorised)."""
        pos_off, pos = _seg_gather(perm.astype(np.int64), act_off[:-1], k)
        owner_base = np.repeat(act_off[:-1], k)
        sk = act[owner_base + pos]
        base = self._append(sk)
        self.s_start[idx] = base + pos_off[:-1]
        self.s_len[idx] = k




def _tree_native(t: Tree) -> dict:
    """Contiguous copies of the tree arrays the native host runtime reads
    (built once per tree)."""
    nv = getattr(t, "_native", None)
    if nv is None:
        nv = dict(center=np.ascontiguousarray(t.center, np.float64),
                  hw=np.ascontiguousarray(t.hw, np.float64),
                  nbr=np.ascontiguousarray(t.neighbors, np.int64),
                  lev=np.ascontiguousarray(t.lev, np.int64),
                  ix=np.ascontiguousarray(t.ix, np.int64),
                  iy=np.ascontiguousarray(t.iy, np.int64),
                  leaf=np.ascontiguousarray(t.is_leaf, np.uint8),
                  ls=np.ascontiguousarray(t.level_start, np.int64),
                  parent=np.ascontiguousarray(t.parent, np.int64),
                  root=np.array([t.root_center[0], t.root_center[1], t.root_half_width]))
        t._native = nv
    return nv


def _native_far_lists(ctx, idx, store):
    nv = _tree_native(ctx.t)
    B = len(idx)
    off = np.zeros(B + 1, np.int64)
    need = np.zeros(1, np.int64)
    cap = max(getattr(ctx, "_far_cap", 0), 4096)
    while True:
        far = np.empty(cap, np.int64)
        rc = _lib.load().skb_host_far_lists(
            B, idx.ctypes.data, nv["center"].ctypes.data, nv["hw"].ctypes.data,
            nv["nbr"].ctypes.data, nv["lev"].ctypes.data, nv["ix"].ctypes.data,
            nv["iy"].ctypes.data, nv["leaf"].ctypes.data, nv["ls"].ctypes.data, ctx.t.depth,
            nv["root"].ctypes.data, ctx.factor, store.big.ctypes.data, store.a_start.ctypes.data,
            store.a_len.ctypes.data, ctx.px.ctypes.data, ctx.py.ctypes.data, off.ctypes.data,
            far.ctypes.data, cap, need.ctypes.data, 1 if ctx.dpn == 2 else 0)
        if rc == 0:
            ctx._far_cap = cap
            return off, far[:int(need[0])]
        cap = int(need[0]) + 1024


class _DevSlab:
    """Device storage from the library's factor pool (skb_dev_alloc: stream
    ordered, never a synchronising cudaMalloc).  Frees are deferred to the
    next factor / update / solve entry (never inside a graph capture) and
    ordered after the level, sweep and current streams."""
    _pending = []

    def __init__(self, nbytes: int, stream):
        out = np.zeros(1, np.uint64)
        call("skb_dev_alloc", int(max(nbytes, 8)), stream.cuda_stream, out)
        self.ptr = int(out[0])
        self.nbytes = int(nbytes)

    @classmethod
    def adopt(cls, addr: int, nbytes: int) -> "_DevSlab":
        """Take over an allocation the native driver made from the same pool."""
        o = cls.__new__(cls)
        o.ptr, o.nbytes = int(addr), int(nbytes)
        return o

    def data_ptr(self) -> int:
        return self.ptr

    def __del__(self):
        if self.ptr:
            pend = _DevSlab._pending if _DevSlab is not None else None
            if pend is not None:            # (module teardown at exit: the pool goes with the process)
                pend.append(self.ptr)
            self.ptr = 0

    @classmethod
    def flush(cls):
        if not cls._pending:
            return
        cur = torch.cuda.current_stream()
        for st in _LEVEL_STREAM:
            cur.wait_stream(st)
        while cls._pending:
            call("skb_dev_free", ctypes.c_uint64(cls._pending.pop()), cur.cuda_stream)


class _CaptureArena:
    """Owns a library capture session (the pinned descriptor arena a captured
    graph replays from).  Released lazily, outside any capture: a destructor
    may run from the garbage collector in the middle of another capture."""
    _pending = []

    def __init__(self, sess):
        self.sess = int(sess)

    def __del__(self):
        if _CaptureArena is not None:
            _CaptureArena._pending.append(self.sess)

    @classmethod
    def flush(cls):
        while cls._pending:
            call("skb_capture_release", cls._pending.pop())


def _upload(**arrays):
    """One H2D copy for several host arrays (staged by the library's pinned
    ring, or its capture arena inside a CUDA-graph capture); returns device views."""
    dev = _dev()
    items, total = [], 0
    for k, a in arrays.items():
        a = np.ascontiguousarray(a)
        total = (total + 15) // 16 * 16
        items.append((k, a, total))
        total += a.nbytes
    total = max(total, 16)
    hn = np.empty(total, np.uint8)
    for k, a, o in items:
        hn[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
    d = torch.empty(total, dtype=torch.uint8, device=dev)
    call("skb_h2d", hn, total, d, _stream())
    IO["h2d"] += total
    out = {}
    for k, a, o in items:
        tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.float64): torch.float64,
               np.dtype(np.int32): torch.int32, np.dtype(np.uint64): torch.int64,
               np.dtype(np.uint8): torch.uint8}[a.dtype]
        out[k] = d[o:o + a.nbytes].view(tdt)
    out["_keep"] = (None, d)
    return out


def _gemm(rows):
    """Launch one grouped GEMM from a list of per-problem column dicts."""
    if not rows:
        return
    n = sum(len(r["m"]) for r in rows)
    if n == 0:
        return
    g = np.zeros(n, GEMM_DT)
    o = 0
    for r in rows:
        c = len(r["m"])
        for f in ("A", "B", "C", "D", "m", "n", "k", "lda", "ldb", "ldc", "ldd", "alpha", "beta",
                  "transA", "transB"):
            g[f][o:o + c] = r.get(f, 0)
        o += c
    call("skb_gemm_grouped", g, n, _stream())


def _mats(ptrs, rows, cols, ld):
    m = np.zeros(len(ptrs), MAT_DT)
    m["ptr"], m["rows"], m["cols"], m["ld"] = ptrs, rows, cols, ld
    return m


def _addr(t: torch.Tensor) -> int:
    return t.data_ptr()


# ---------------------------------------------------------------------------
# device geometry
# ---------------------------------------------------------------------------
class DeviceBoundary:
    """Boundary SoA arrays resident in HBM.  ``Boundary._skb_device = DeviceBoundary(b)``
    keeps them resident across factor() calls (device-resident benchmark mode)."""

    def __init__(self, b):
        up = _upload(pos=np.ascontiguousarray(b.positions, np.float64),
                     nrm=np.ascontiguousarray(b.normals, np.float64),
                     w=np.ascontiguousarray(b.weights, np.float64),
                     kap=np.ascontiguousarray(b.curvatures, np.float64))
        self.pos, self.nrm, self.w, self.kap = up["pos"], up["nrm"], up["w"], up["kap"]
        self._keep = up["_keep"]
        self.n = b.n_nodes


# ---------------------------------------------------------------------------
# per-level factor storage
# ---------------------------------------------------------------------------
class BoxBatch:
    """Factors of a batch of boxes of one level, resident on the device."""

    FIELDS = ("T", "Xrr", "LU", "Xsr", "Xrsdiv", "Xss")

    def __init__(self, idx, act_off, act):
        self.idx = np.asarray(idx, np.int64)
        self.act_off, self.act = act_off, act
        self.nB = np.diff(act_off)
        n = len(self.idx)
        self.k = np.zeros(n, np.int64)
        self.perm = np.zeros(len(act), np.int32)
        self.gap = np.ones(n)
        self.steps = np.zeros(n, np.int64)
        self.ratio = np.ones(n)
        self.info = np.full(n, -1, np.int64)
        self.ptr = {f: np.zeros(n, np.uint64) for f in self.FIELDS}
        self.ipiv = np.zeros(n, np.uint64)
        self.slabs = []                        # device allocations holding the boxes' factors
        self.slab_of = np.full(n, -1, np.int64)   # index into slabs per box

    @property
    def r(self):
        return self.nB - self.k

    def resolve(self):
        """Wait for the asynchronously copied X_RR pivot info of this batch."""
        pend = getattr(self, "_pending", None)
        if pend is not None:
            info_h, ratio_h, ev = pend[:3]
            t0 = time.perf_counter()
            ev.synchronize()
            IO["wait_s"] += time.perf_counter() - t0
            IO["waits"] += 1
            self.info[:] = info_h
            self.ratio[:] = ratio_h
            self._pending = None
        dfr = getattr(self, "_deferred", None)
        if dfr:
            self._deferred = []
            for sel, other, osel in dfr:
                other.resolve()
                self.info[sel], self.ratio[sel] = other.info[osel], other.ratio[osel]

    def skel_csr(self):
        off, pos = _seg_gather(self.perm.astype(np.int64), self.act_off[:-1], self.k)
        return off, self.act[np.repeat(self.act_off[:-1], self.k) + pos]

    def red_csr(self):
        r = self.r
        off, pos = _seg_gather(self.perm.astype(np.int64), self.act_off[:-1] + self.k, r)
        return off, self.act[np.repeat(self.act_off[:-1], r) + pos]

    def take(self, sel, other, osel):
        """Overwrite boxes ``sel`` with ``other``'s boxes ``osel`` (same DOF layout), vectorised."""
        sel = np.asarray(sel, np.int64)
        osel = np.asarray(osel, np.int64)
        if len(sel) == 0:
            return
        lens = self.nB[sel]
        _, src = _seg_gather(np.arange(len(other.perm)), other.act_off[osel], lens)
        _, dst = _seg_gather(np.arange(len(self.perm)), self.act_off[sel], lens)
        self.perm[dst] = other.perm[src]
        self.k[sel], self.gap[sel], self.steps[sel] = other.k[osel], other.gap[osel], other.steps[osel]
        self.ratio[sel], self.info[sel] = other.ratio[osel], other.info[osel]
        for f in self.FIELDS:
            self.ptr[f][sel] = other.ptr[f][osel]
        self.ipiv[sel] = other.ipiv[osel]
        # pivot info may still be in flight: copy it when this batch is resolved
        if getattr(self, "_deferred", None) is None:
            self._deferred = []
        self._deferred.append((sel, other, osel))
        # keep only the slabs that hold a box of this batch (an update chain must not
        # keep every superseded slab of the level alive)
        pos = {id(x): i for i, x in enumerate(self.slabs)}
        so = other.slab_of[osel]
        lut = np.full(max(len(other.slabs), 1), -1, np.int64)
        for u in np.unique(so[so >= 0]):
            sl = other.slabs[u]
            i = pos.get(id(sl))
            if i is None:
                i = pos[id(sl)] = len(self.slabs)
                self.slabs.append(sl)
            lut[u] = i
        self.slab_of[sel] = np.where(so >= 0, lut[np.maximum(so, 0)], -1)


class LevelFactors:
    """All boxes of one tree level (sorted keys) with device CSR lists of
    skeleton/redundant DOFs for the gathers of the sweeps."""

    @property
    def keys(self):
        ks = self.__dict__.get("_keys")
        if ks is None:
            ks = self.__dict__["_keys"] = [self.tree.key(i) for i in self.idx]
        return ks

    def __init__(self, lev, tree, batch: BoxBatch, cols_off, cols):
        self.lev = lev
        self.tree = tree
        self.batch = batch
        self.idx = batch.idx
        self.k = batch.k.copy()
        self.r = batch.r.copy()
        self.sd_off, self.sd = batch.skel_csr()
        self.rd_off, self.rd = batch.red_csr()
        self.cols_off, self.cols = cols_off, cols
        self.ncols = np.diff(cols_off)
        up = _upload(sd_off=self.sd_off, sd=self.sd if len(self.sd) else np.zeros(1, np.int64),
                     rd_off=self.rd_off, rd=self.rd if len(self.rd) else np.zeros(1, np.int64),
                     c_off=cols_off, c=cols if len(cols) else np.zeros(1, np.int64))
        self.d = up
        self.P = {f: batch.ptr[f] for f in BoxBatch.FIELDS}
        self.ipiv = batch.ipiv


# ---------------------------------------------------------------------------
# the compression pipeline for one batch of boxes
# ---------------------------------------------------------------------------
class _Ctx:
    def __init__(self, spec, b, t: Tree, tol, proxy_count, proxy_factor):
        self.spec, self.b, self.t = spec, b, t
        self.dpn, self.pde = spec.dof_per_node, spec.code
        self.tol, self.P, self.factor = float(tol), int(proxy_count), float(proxy_factor)
        if self.P < 8:
            raise ValueError("need at least 8 proxy nodes")
        self._g = None
        self.px = np.ascontiguousarray(b.positions[:, 0])
        self.py = np.ascontiguousarray(b.positions[:, 1])
        th = 2 * np.pi * np.arange(self.P) / self.P
        self.cs = np.stack([np.cos(th), np.sin(th)], axis=1)
        self.stats = {"kernel_s": {}}

    @property
    def sstream(self) -> torch.cuda.Stream:
        return _level_stream()

    @property
    def g(self) -> DeviceBoundary:
        if self._g is None:
            cached = getattr(self.b, "_skb_device", None)
            self._g = cached if cached is not None else DeviceBoundary(self.b)
        return self._g

    # -- host bookkeeping ---------------------------------------------------
    def far_pairs(self, idx):
        """Skeleton-independent half of far_dofs (reference skel.py:258-280):
        the (box, source box) candidate pairs -- colleagues (sorted keys) then
        coarser leaves meeting the proxy disc (sorted keys) -- and the radii."""
        t = self.t
        rp = proxy_radius(t.hw[idx], self.factor)
        nbr = t.neighbors[idx]
        bl_n, s_n = np.nonzero(nbr >= 0)
        src_n = nbr[bl_n, s_n]
        bl_c, src_c = t.coarse_leaves(idx, rp)
        pb = np.concatenate([bl_n, bl_c]).astype(np.int64)
        ps = np.concatenate([src_n, src_c]).astype(np.int64)
        order = np.argsort(pb, kind="stable")
        return rp, pb[order], ps[order]

    def far_lists(self, idx, store: "ActStore", pairs=None):
        """F_int per box (reference _Compressor.far_dofs, skel.py:258-280):
        active DOFs of the candidate sources, filtered by strict distance < r_p
        from the box centre.  Native (csrc/host.cpp) unless candidate pairs are
        given (the NumPy restatement below, kept for the host tests)."""
        if pairs is None:
            return _native_far_lists(self, np.asarray(idx, np.int64), store)
        return self.far_lists_np(idx, store, pairs)

    def far_lists_np(self, idx, store: "ActStore", pairs=None):
        t = self.t
        rp, pb, ps = self.far_pairs(idx) if pairs is None else pairs
        B = len(idx)
        if len(ps) == 0:
            return np.zeros(B + 1, np.int64), np.zeros(0, np.int64)
        lens = store.a_len[ps]
        _, flat = _seg_gather(store.big, store.a_start[ps], lens)
        owner = np.repeat(pb, lens)
        # ((dof_pos - c)**2).sum(axis=1) of skel.py:279, same rounding: dx*dx + dy*dy
        node = flat >> (1 if self.dpn == 2 else 0)
        dx = self.px[node] - t.center[idx, 0][owner]
        dy = self.py[node] - t.center[idx, 1][owner]
        d2 = dx * dx + dy * dy
        keep = d2 < (rp * rp)[owner]
        F = flat[keep]
        cnt = np.bincount(owner[keep], minlength=B)
        off = np.zeros(B + 1, np.int64)
        np.cumsum(cnt, out=off[1:])
        return off, F

    def proxies(self, idx):
        """Proxy rings + radial normals + weights (kernels.py:263-273, 340-342), native."""
        idx = np.asarray(idx, np.int64)
        nv = _tree_native(self.t)
        B = len(idx)
        pts = np.empty((B, self.P, 2))
        pn = np.empty((B, self.P, 2))
        pw = np.empty(B)
        call("skb_host_proxies", B, idx, nv["center"], nv["hw"], self.factor, self.P,
             np.ascontiguousarray(self.cs), pts, pn, pw)
        return pts, pn, pw

    def proxies_np(self, idx):
        rp = proxy_radius(self.t.hw[idx], self.factor)
        pts = self.t.center[idx][:, None, :] + rp[:, None, None] * self.cs[None]
        # ring centre: sequential left-to-right sum (cumsum keeps that order)
        ctr = np.cumsum(pts, axis=1)[:, -1, :] / self.P
        pn = pts - ctr[:, None, :]
        pn = pn / np.sqrt((pn * pn).sum(axis=2))[:, :, None]
        pw = 2 * np.pi * rp / self.P
        return pts, pn, pw

    def prep(self, idx) -> dict:
        """Skeleton-independent inputs of launch() for a batch (proxy rings)."""
        idx = np.asarray(idx, np.int64)
        return dict(pairs=None, proxies=self.proxies(idx))

    def child_desc(self, idx, store: "ActStore"):
        """Children's skeleton offsets (active order) and Xss addresses."""
        idx = np.asarray(idx, np.int64)
        ch = self.t.children[idx]
        valid = ch >= 0
        kc = np.where(valid, store.s_len[np.maximum(ch, 0)], 0)
        co = np.full((len(idx), 5), -1, np.int64)
        inner = valid.any(axis=1)
        cum = np.cumsum(kc, axis=1)
        co[inner, 0] = 0
        co[:, 1:] = np.where(valid, cum, -1)
        co[~inner, 1:] = -1
        cx = np.where(valid, store.xss[np.maximum(ch, 0)], np.uint64(0)).astype(np.uint64)
        return co, cx

    # -- device pipeline ----------------------------------------------------
    def launch(self, idx, store: "ActStore", kmin=None, prep=None) -> dict:
        """(a)+(b) of compress_box (reference skel.py:293-316) for a batch of
        same-level boxes: ID stacks, Householder pre-reduction and QRCP are
        enqueued on the current stream; nothing waits."""
        t, P = self.t, self.P
        _Prof.start()
        idx = np.asarray(idx, np.int64)
        B = len(idx)
        with _ht("L.acts"):
            act_off, act = store.acts(idx)
        nB = np.diff(act_off)
        if prep is None:
            prep = self.prep(idx)
        with _ht("L.far_lists"):
            far_off, far = self.far_lists(idx, store, prep["pairs"])
        nF = np.diff(far_off)
        pts, pn, pw = prep["proxies"]
        rows = 2 * nF + (6 if self.dpn == 2 else 2) * P + 2       # stack rows, skel.py:306-314
        sizes = rows * nB
        stack_off = np.zeros(B + 1, np.int64)
        np.cumsum(sizes, out=stack_off[1:])
        dev = _dev()
        _Prof.tick("host_far_proxy")
        with _ht("L.stack_alloc"):
          stack = torch.empty(max(int(stack_off[-1]), 1), dtype=torch.float64, device=dev)
        with _ht("L.upload"):
          up = _upload(act_off=act_off, act=act if len(act) else np.zeros(1, np.int64),
                     far_off=far_off, far=far if len(far) else np.zeros(1, np.int64),
                     pts=pts.reshape(-1), pn=pn.reshape(-1), pw=pw, stack_off=stack_off[:-1])
        s = _stream()
        call("skb_assemble_stack" if self.dpn == 2 else "skb_assemble_stack_lap",
             ptr(self.g.pos), ptr(self.g.nrm), ptr(self.g.w), B,
             ptr(up["act_off"]), ptr(up["act"]), ptr(up["far_off"]), ptr(up["far"]),
             ptr(up["pts"]), ptr(up["pn"]), ptr(up["pw"]), P, ptr(up["stack_off"]), ptr(stack),
             int(nB.max(initial=0)), int((nF + P + 1).max(initial=0)), s)
        _Prof.tick("a_stack")
        base = _addr(stack)
        A = (base + 8 * stack_off[:-1]).astype(np.int64)
        pre = rows > 2 * nB                  # Householder pre-reduction branch, dense.py:56
        if pre.any():
          with _ht("L.geqrf"):
            call("skb_geqrf_batched", int(pre.sum()), np.ascontiguousarray(rows[pre]),
                 np.ascontiguousarray(nB[pre]),
                 np.ascontiguousarray(rows[pre]),
                 np.ascontiguousarray(A[pre]), s)
        _Prof.tick("b_geqrf")
        m_q = np.where(pre, nB, rows).astype(np.int64)
        kmin_a = np.zeros(B, np.int64) if kmin is None else np.asarray(kmin, np.int64)
        na = len(act)
        # one device buffer: diag (na f64) | gap (B f64) | perm (na i32) | k (B) | steps (B+1);
        # gap..steps come back to the host in ONE copy
        nint = na + 2 * B + 1
        o_gap = 8 * max(na, 1)
        o_int = o_gap + 8 * max(B, 1)
        dbuf = torch.empty(o_int + 4 * nint, dtype=torch.uint8, device=dev)
        db = _addr(dbuf)
        lda = rows.astype(np.int64)
        with _ht("L.qrcp"):
          call("skb_qrcp_id_batched", B, m_q, nB, lda,
             A, kmin_a, self.tol, act_off, db + o_int,
             db, db + o_int + 4 * na, db + o_int + 4 * (na + B), db + o_gap, s)
        _Prof.tick("b_qrcp")
        hbuf = torch.empty(dbuf.numel() - o_gap, dtype=torch.uint8, pin_memory=True)
        hbuf.copy_(dbuf[o_gap:], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        IO["d2h"] += hbuf.numel()
        return dict(idx=idx, act_off=act_off, act=act, nB=nB, rows=rows, pre=pre, m_q=m_q,
                    stack=stack, up=up, A=A, lda=lda, perm_d=dbuf[o_int:].view(torch.int32),
                    hbuf=hbuf, o_int=o_int - o_gap, ev=ev)

    def finish(self, h: dict) -> BoxBatch:
        """Wait for a launched batch's QRCP (the one host sync per level) and
        lay out its factor storage; no kernels are launched."""
        idx, act_off, nB = h["idx"], h["act_off"], h["nB"]
        B, na = len(idx), len(h["act"])
        t0 = time.perf_counter()
        with _ht("F.wait"):
            h["ev"].synchronize()                 # sync point (sizes for (c))
        IO["wait_s"] += time.perf_counter() - t0
        IO["waits"] += 1
        hb = h["hbuf"].numpy()
        ih = hb[h["o_int"]:].view(np.int32)
        bt = BoxBatch(idx, act_off, h["act"])
        bt.perm[:] = ih[:na]
        bt.k[:] = ih[na:na + B]
        bt.steps[:] = ih[na + B:na + 2 * B]
        bt.gap[:] = hb[:8 * B].view(np.float64)
        bt._launch = h
        return bt

    def layout(self, bt: BoxBatch):
        """Factor storage of a finished batch (one slab per level); off the
        critical path: runs after the next level's compression is launched."""
        h = bt._launch
        nB, B = bt.nB, len(bt.idx)
        k = bt.k
        r = nB - k
        if _lib.PROF_ON:
            # algorithmic work: stack + self-block bytes written,
            # Householder 2 m n^2 - 2/3 n^3, QRCP 2mn + sum_i 4 (m-i)(n-i-1)
            rows, pre = h["rows"], h["pre"]
            _lib.prof_add("assemble", 0.0, 8.0 * float((rows * nB).sum() + (nB * nB).sum()))
            mr, nr_ = rows[pre].astype(float), nB[pre].astype(float)
            # geqrf / QRCP bytes: the stack (or R) they read once from HBM
            _lib.prof_add("geqrf", float((2 * mr * nr_ ** 2 - 2.0 / 3.0 * nr_ ** 3).sum()),
                          8.0 * float((mr * nr_).sum()))
            fq = 0.0
            for mm, nn, st in zip(h["m_q"], nB, bt.steps):
                i_ = np.arange(st, dtype=float)
                fq += 2.0 * mm * nn + float((4.0 * (mm - i_) * (nn - i_ - 1)).sum())
            _lib.prof_add("qrcp", fq, 8.0 * float((h["m_q"] * nB).sum()))
        # factor storage (one slab from the factor pool), ordered on the level
        # stream that fills it
        sz = np.stack([k * r, r * r, r * r, k * r, r * k, k * k], axis=1)
        tot = sz.sum(axis=1)
        boff = np.zeros(B + 1, np.int64)
        np.cumsum(tot, out=boff[1:])
        # factors (f64) followed by the LU pivots (i32) in ONE allocation
        nf = max(int(boff[-1]), 1)
        slab = _DevSlab(8 * nf + 4 * max(int(r.sum()), 1), self.sstream)
        bt.slabs.append(slab)
        bt.slab_of[:] = len(bt.slabs) - 1
        sb = _addr(slab)
        fo = boff[:-1].copy()
        for fi, f in enumerate(BoxBatch.FIELDS):
            bt.ptr[f][:] = (sb + 8 * fo).astype(np.uint64)
            fo = fo + sz[:, fi]
        ioff = np.zeros(B + 1, np.int64)
        np.cumsum(r, out=ioff[1:])
        bt.ipiv[:] = (sb + 8 * nf + 4 * ioff[:-1]).astype(np.uint64)

    def schur(self, bt: BoxBatch, store: "ActStore"):
        """(c) of compress_box (reference skel.py:317-338) on the level stream:
        it depends on this batch's QRCP and on the children's Xss (previous
        level, same stream), not on the next level's compression."""
        if not bt.slabs:
            self.layout(bt)
        h = bt.__dict__.pop("_launch")
        S = self.sstream
        eng = h.get("engine")
        if eng is not None:
            # level compressed by the native engine: its buffers are raw device
            # pointers, released stream-ordered after the Schur stage
            eng.stream_wait(h["lev"], S)
            with torch.cuda.stream(S):
                self._schur(bt, store, h)
            eng.release(h["lev"], S)
            return
        S.wait_event(h["ev"])
        for tns in (h["stack"], h["perm_d"], h["up"]["_keep"][1]):
            tns.record_stream(S)
        h["dev"] = (ptr(h["up"]["act_off"]), ptr(h["up"]["act"]), ptr(h["perm_d"]))
        with torch.cuda.stream(S):
            self._schur(bt, store, h)

    def _schur(self, bt, store, h):
        idx, act_off, nB, A, lda = h["idx"], h["act_off"], h["nB"], h["A"], h["lda"]
        act_off_d, act_d, perm_d = h["dev"]
        B = len(idx)
        dev = _dev()
        co, cx = self.child_desc(idx, store)
        pbuf = torch.empty(12 * B, dtype=torch.uint8, device=dev)   # ratio (f64) | info (i32)
        ratio_d, info_d = _addr(pbuf), _addr(pbuf) + 8 * B
        # T, self blocks, Schur GEMMs, LU(X_rr), X_rs_div, Xss_mod: one native call
        call("skb_level_schur", B, np.ascontiguousarray(nB, np.int64), bt.k, act_off,
             ptr(self.g.pos), ptr(self.g.nrm), ptr(self.g.w), ptr(self.g.kap), act_off_d,
             act_d, perm_d, A, lda, np.ascontiguousarray(co.reshape(-1)),
             np.ascontiguousarray(cx.reshape(-1)), bt.ptr["T"], bt.ptr["Xrr"], bt.ptr["LU"],
             bt.ptr["Xsr"], bt.ptr["Xrsdiv"], bt.ptr["Xss"], bt.ipiv, info_d, ratio_d, self.pde,
             _stream())
        _Prof.tick("c_schur")
        # X_RR pivot info for the migration rule: copied asynchronously, checked
        # after the next level's QRCP sync (no extra host sync per level)
        phost = torch.empty(12 * B, dtype=torch.uint8, pin_memory=True)
        phost.copy_(pbuf, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        IO["d2h"] += 12 * B
        ph = phost.numpy()
        bt._pending = (ph[8 * B:].view(np.int32), ph[:8 * B].view(np.float64), ev, phost)

    def compress(self, idx, store: "ActStore", kmin=None) -> BoxBatch:
        """Compress a batch of same-level boxes (reference compress_box, skel.py:293-338)."""
        bt = self.finish(self.launch(idx, store, kmin))
        self.schur(bt, store)
        return bt

    def migrate(self, bt: "BoxBatch", store) -> bool:
        """R -> S migration while the X_RR pivot ratio is below the floor
        (reference skel.py:317-330).  Returns True when any box changed."""
        changed = False
        while True:
            bt.resolve()
            kk = bt.k
            bad = ((bt.info >= 0) | (bt.ratio < PIVOT_RATIO_FLOOR)) & (kk < bt.nB)
            if not bad.any():
                return changed
            sel = np.flatnonzero(bad)
            knew = np.minimum(bt.nB[sel], kk[sel] + np.maximum(1, (bt.nB[sel] - kk[sel]) // 8))
            sub = self.compress(bt.idx[sel], store, kmin=knew)
            bt.take(sel, sub, np.arange(len(sel)))
            changed = True


# ---------------------------------------------------------------------------
# Factorization
# ---------------------------------------------------------------------------
class BoxFactors:
    """Reference-style per-box view (skel.py:55-85), host copies on demand."""

    def __init__(self, key, b_dofs, S_loc, R_loc, mats):
        self.key, self.b_dofs, self.S_loc, self.R_loc = key, b_dofs, S_loc, R_loc
        self._mats = mats

    @property
    def skel_dofs(self):
        return self.b_dofs[self.S_loc]

    @property
    def red_dofs(self):
        return self.b_dofs[self.R_loc]

    def __getattr__(self, name):
        m = self.__dict__.get("_mats")
        if m is not None and name in m:
            return m[name]()
        raise AttributeError(name)


def _fetch(addr, rows, cols):
    """Host copy of a device row-major (rows x cols) block at a raw address."""
    rows, cols = int(rows), int(cols)
    if rows * cols == 0:
        return np.zeros((rows, cols))
    t = torch.empty((rows, cols), dtype=torch.float64, device=_dev())
    call("skb_copy2d_batched", 1, _mats([_addr(t)], [rows], [cols], [cols]),
         _mats(np.array([addr], np.uint64), [rows], [cols], [cols]), 0, _stream())
    return t.cpu().numpy()


def _fetch_i32(addr, n):
    out = np.empty(max(int(n), 1), np.int32)
    if n:
        call("skb_d2h", out, ctypes.c_void_p(int(addr)), 4 * int(n))
    return out[:int(n)]


class LUView:
    """Host copy of a box's X_RR LU factors (reference BoxFactors.lu, a PLU of
    dense.py:106-135): ``lu`` (unit-lower L and U packed, row-major), 0-based
    LAPACK pivots ``piv`` and ``pivot_ratio`` = min |u_ii| / max |u_ii|."""

    def __init__(self, lu, piv):
        self.lu, self.piv = lu, piv
        d = np.abs(np.diag(lu))
        self.pivot_ratio = float(d.min() / d.max()) if len(d) and d.max() > 0 else 1.0

    @property
    def n(self):
        return self.lu.shape[0]

    def solve(self, B):
        """X_RR^-1 B on the host copies (inspection only; the factorization's
        own solves run on the device)."""
        import scipy.linalg as sla
        return sla.lu_solve((self.lu, self.piv), np.asarray(B, float))


class _FactorsView:
    """Lazy mapping key -> BoxFactors (reference Factorization.factors)."""

    def __init__(self, levels):
        # holds the level list only (no reference back to the Factorization:
        # a cycle would keep its device memory alive until the cyclic GC runs)
        self._levels = levels
        self._w = None

    @property
    def _where(self) -> dict:
        if self._w is None:
            self._w = {key: (li, bi) for li, L in enumerate(self._levels)
                       for bi, key in enumerate(L.keys)}
        return self._w

    def __len__(self):
        return len(self._where)

    def __iter__(self):
        return iter(self._where)

    def __contains__(self, key):
        return tuple(key) in self._where

    def keys(self):
        return self._where.keys()

    def __getitem__(self, key):
        li, bi = self._where[tuple(key)]
        L = self._levels[li]
        bt = L.batch
        a0, a1 = bt.act_off[bi], bt.act_off[bi + 1]
        dofs = bt.act[a0:a1]
        perm = bt.perm[a0:a1].astype(np.int64)
        k, r = int(L.k[bi]), int(L.r[bi])
        P = L.P
        mats = {
            "T": lambda: _fetch(P["T"][bi], k, r),
            "X_rr": lambda: _fetch(P["Xrr"][bi], r, r),
            "X_sr": lambda: _fetch(P["Xsr"][bi], k, r),
            "X_rs_div": lambda: _fetch(P["Xrsdiv"][bi], r, k),
            "Xss_mod": lambda: _fetch(P["Xss"][bi], k, k),
            "lu": lambda: LUView(_fetch(P["LU"][bi], r, r), _fetch_i32(L.ipiv[bi], r)),
        }
        return BoxFactors(tuple(key), dofs, perm[:k], perm[k:], mats)


class Factorization:
    """Device-resident factorization (reference skel.py:88-221)."""

    def __init__(self, spec, boundary, tree, tol, proxy_count, proxy_factor, levels, root_dofs,
                 E_root, top, top_ipiv, UH, PsiV, UH_div, q, ctx, stats):
        self.spec, self.boundary, self.tree = spec, boundary, tree
        self.tol, self.proxy_count, self.proxy_factor = tol, proxy_count, proxy_factor
        self.levels = levels                # bottom-up (reference sweep_levels order)
        self.root_dofs = root_dofs
        self.E_root, self.top, self.top_ipiv = E_root, top, top_ipiv
        self.UH, self.PsiV, self.UH_div = UH, PsiV, UH_div
        self.q = q
        self._ctx = ctx
        self.stats = stats
        rd = root_dofs if len(root_dofs) else np.zeros(1, np.int64)
        self._root_d = _upload(r=rd)
        self.factors = _FactorsView(levels)

    @property
    def n_dofs(self) -> int:
        return self.spec.dof_per_node * self.boundary.n_nodes

    def _psi_lists(self, with_root: bool):
        """Per augmentation column, the DOF rows where PsiV can be nonzero (rows
        eliminated in a box containing that hole; + root rows for apply), sorted
        by row -- CSR on the device for skb_psi_dot."""
        key = "_psi_root" if with_root else "_psi_nonroot"
        got = getattr(self, key, None)
        if got is not None:
            return got
        rows_l, cols_l = [], []
        for L in self.levels:
            r, c = L.r, L.ncols
            cnt = r * c
            tot = int(cnt.sum())
            if tot == 0:
                continue
            box = np.repeat(np.arange(len(r)), cnt)
            start = np.zeros(len(r), np.int64)
            np.cumsum(cnt[:-1], out=start[1:])
            local = np.arange(tot) - start[box]
            cb = c[box]
            rows_l.append(L.rd[L.rd_off[box] + local // cb])
            cols_l.append(L.cols[L.cols_off[box] + local % cb])
        if with_root and self.q:
            rd = np.asarray(self.root_dofs, np.int64)
            rows_l.append(np.repeat(rd, self.q))
            cols_l.append(np.tile(np.arange(self.q, dtype=np.int64), len(rd)))
        rows = np.concatenate(rows_l) if rows_l else np.zeros(0, np.int64)
        cols = np.concatenate(cols_l) if cols_l else np.zeros(0, np.int64)
        order = np.lexsort((rows, cols))
        rows, cols = rows[order], cols[order]
        off = np.zeros(self.q + 1, np.int64)
        np.cumsum(np.bincount(cols, minlength=self.q), out=off[1:])
        got = _upload(off=off, rows=rows if len(rows) else np.zeros(1, np.int64))
        setattr(self, key, got)
        return got

    @property
    def n_aug(self) -> int:
        return self.q

    @property
    def dim(self) -> int:
        return self.n_dofs + self.q

    @property
    def sweep_levels(self):
        return [(L.lev, L.keys) for L in self.levels]

    # ---- device sweeps -----------------------------------------------------
    def _gather(self, L, which, x, nr, buf):
        off, dd = (L.d["sd_off"], L.d["sd"]) if which == "s" else (L.d["rd_off"], L.d["rd"])
        cnt = L.k if which == "s" else L.r
        o = np.zeros(len(cnt) + 1, np.int64)
        np.cumsum(cnt * nr, out=o[1:])
        up = _upload(o=o[:-1], ld=np.full(len(cnt), nr, np.int64))
        call("skb_gather_rows", len(cnt), ptr(off), ptr(dd), None, None, nr, ptr(x), nr,
             ptr(buf), ptr(up["o"]), ptr(up["ld"]), int(cnt.max(initial=0)), nr, _stream())
        return (_addr(buf) + 8 * o[:-1]).astype(np.uint64), up

    def _scatter(self, L, which, x, nr, bptr, keep):
        off, dd = (L.d["sd_off"], L.d["sd"]) if which == "s" else (L.d["rd_off"], L.d["rd"])
        cnt = L.k if which == "s" else L.r
        base = int(bptr[0]) if len(bptr) else 0
        up = _upload(o=((bptr.astype(np.int64) - base) // 8), ld=np.full(len(cnt), nr, np.int64))
        keep.append(up)
        call("skb_scatter_rows", len(cnt), ptr(off), ptr(dd), None, None, nr, base,
             ptr(up["o"]), ptr(up["ld"]), ptr(x), nr, 0, 1.0, int(cnt.max(initial=0)), nr,
             _stream())

    def _solve_dev(self, x: torch.Tensor) -> torch.Tensor:
        """In-place solve on a (dim, nrhs) row-major device tensor (skel.py:166-221)."""
        nr = x.shape[1]
        nd, q = self.n_dofs, self.q
        s = _stream()
        dev = x.device
        keep = []
        for L in self.levels:                       # _level_up, skel.py:195-208
            B = len(L.k)
            xs = torch.empty(max(int(L.k.sum()) * nr, 1), dtype=torch.float64, device=dev)
            xr = torch.empty(max(int(L.r.sum()) * nr, 1), dtype=torch.float64, device=dev)
            ps, u1 = self._gather(L, "s", x, nr, xs)
            pr, u2 = self._gather(L, "r", x, nr, xr)
            keep += [u1, u2, xs, xr]
            one, mone = np.ones(B), -np.ones(B)
            _gemm([dict(A=L.P["T"], B=ps, C=pr, D=pr, m=L.r, n=nr, k=L.k, lda=L.r, ldb=nr,
                        ldc=nr, ldd=nr, alpha=mone, beta=one, transA=1)])
            call("skb_getrs_batched", B, _mats(L.P["LU"], L.r, L.r, L.r),
                 L.ipiv, _mats(pr, L.r, nr, nr), s)
            _gemm([dict(A=L.P["Xsr"], B=pr, C=ps, D=ps, m=L.k, n=nr, k=L.r, lda=L.r, ldb=nr,
                        ldc=nr, ldd=nr, alpha=mone, beta=one)])
            self._scatter(L, "s", x, nr, ps, keep)
            self._scatter(L, "r", x, nr, pr, keep)
        ns = len(self.root_dofs)
        rd = self._root_d
        if q:                                        # skel.py:180-188
            pl = self._psi_lists(False)
            top_rhs = torch.empty((ns + q, nr), dtype=torch.float64, device=dev)
            up = _upload(o=np.zeros(1, np.int64), ld=np.array([nr], np.int64),
                         ro=np.array([0, ns], np.int64))
            keep.append(up)
            call("skb_gather_rows", 1, ptr(up["ro"]), ptr(rd["r"]), None, None, nr, ptr(x), nr,
                 ptr(top_rhs), ptr(up["o"]), ptr(up["ld"]), ns, nr, s)
            # corr = lam_rhs - PsiV[nonroot]^T x[nonroot]: column-sparse, compensated
            call("skb_psi_dot", q, pl["off"], pl["rows"], self.PsiV, q, x, nr, nr,
                 _addr(x) + 8 * nd * nr, nr, -1.0, _addr(top_rhs) + 8 * ns * nr, nr, s)
            call("skb_getrs_batched", 1, _mats([_addr(self.top)], [ns + q], [ns + q],
                                              [ns + q]),
                 np.array([_addr(self.top_ipiv)], np.uint64),
                 _mats([_addr(top_rhs)], [ns + q], [nr], [nr]), s)
            call("skb_scatter_rows", 1, ptr(up["ro"]), ptr(rd["r"]), None, None, nr,
                 _addr(top_rhs), ptr(up["o"]), ptr(up["ld"]), ptr(x), nr, 0, 1.0, ns, nr, s)
            x[nd:].copy_(top_rhs[ns:])
            # x[:nd] -= UH_div lam (UH_div rows of root DOFs are exactly zero; skel.py:188):
            # the solve's largest product, (2N x q)(q x nrhs), on the DMMA GEMM
            _gemm([dict(A=np.array([_addr(self.UH_div)], np.uint64),
                        B=np.array([_addr(top_rhs) + 8 * ns * nr], np.uint64),
                        C=np.array([_addr(x)], np.uint64), D=np.array([_addr(x)], np.uint64),
                        m=[nd], n=[nr], k=[q], lda=[q], ldb=[nr], ldc=[nr], ldd=[nr],
                        alpha=[-1.0], beta=[1.0])])
            keep += [top_rhs]
        else:
            top_rhs = torch.empty((ns, nr), dtype=torch.float64, device=dev)
            up = _upload(o=np.zeros(1, np.int64), ld=np.array([nr], np.int64),
                         ro=np.array([0, ns], np.int64))
            keep += [up, top_rhs]
            call("skb_gather_rows", 1, ptr(up["ro"]), ptr(rd["r"]), None, None, nr, ptr(x), nr,
                 ptr(top_rhs), ptr(up["o"]), ptr(up["ld"]), ns, nr, s)
            call("skb_getrs_batched", 1, _mats([_addr(self.top)], [ns], [ns], [ns]),
                 np.array([_addr(self.top_ipiv)], np.uint64),
                 _mats([_addr(top_rhs)], [ns], [nr], [nr]), s)
            call("skb_scatter_rows", 1, ptr(up["ro"]), ptr(rd["r"]), None, None, nr,
                 _addr(top_rhs), ptr(up["o"]), ptr(up["ld"]), ptr(x), nr, 0, 1.0, ns, nr, s)
        for L in reversed(self.levels):             # _level_down, skel.py:210-221
            B = len(L.k)
            xs = torch.empty(max(int(L.k.sum()) * nr, 1), dtype=torch.float64, device=dev)
            xr = torch.empty(max(int(L.r.sum()) * nr, 1), dtype=torch.float64, device=dev)
            ps, u1 = self._gather(L, "s", x, nr, xs)
            pr, u2 = self._gather(L, "r", x, nr, xr)
            keep += [u1, u2, xs, xr]
            one, mone = np.ones(B), -np.ones(B)
            _gemm([dict(A=L.P["Xrsdiv"], B=ps, C=pr, D=pr, m=L.r, n=nr, k=L.k, lda=L.k, ldb=nr,
                        ldc=nr, ldd=nr, alpha=mone, beta=one)])
            _gemm([dict(A=L.P["T"], B=pr, C=ps, D=ps, m=L.k, n=nr, k=L.r, lda=L.r, ldb=nr,
                        ldc=nr, ldd=nr, alpha=mone, beta=one)])
            self._scatter(L, "s", x, nr, ps, keep)
            self._scatter(L, "r", x, nr, pr, keep)
        self._keep = keep
        return x

    def _solve_graphed(self, x: torch.Tensor):
        """The per-level solve is a fixed launch sequence for a given nrhs: it is
        captured once into a CUDA graph (library descriptor uploads staged in
        pinned memory during capture) and replayed on a static input buffer."""
        nr = x.shape[1]
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        ent = self._graphs.get(nr)
        if ent is None:
            xs = x.clone()
            self._solve_dev(x.clone())           # warm-up outside capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            # destructors of unreachable objects holding graphs / device memory
            # must not run inside the capture (graph teardown and frees are
            # illegal there): collect now and keep the collector off meanwhile
            gc.collect()
            _CaptureArena.flush()
            call("skb_capture_begin", 48 << 20)
            gc_was = gc.isenabled()
            gc.disable()
            try:
                with torch.cuda.graph(g):
                    self._solve_dev(xs)
            except Exception:
                if gc_was:
                    gc.enable()
                if os.environ.get("SKB_DEBUG_CAPTURE"):
                    import traceback
                    traceback.print_exc()
                call("skb_capture_end")
                self._graphs[nr] = False
                torch.cuda.synchronize()
                self._solve_dev(x)
                return x
            if gc_was:
                gc.enable()
            sess = call("skb_capture_end")
            ent = (g, xs, _CaptureArena(sess), self._keep)
            if len(self._graphs) >= 4:
                self._graphs.clear()
            self._graphs[nr] = ent
        if ent is False:
            self._solve_dev(x)
            return x
        g, xs, _, _ = ent
        xs.copy_(x)
        g.replay()
        x.copy_(xs)
        return x

    def solve(self, rhs, workers: int = 1, refine: int = 0):
        """Solve A x = rhs for (dim,) or (dim, nrhs) input (reference skel.py:166-193).

        ``refine`` > 0 adds that many steps of iterative refinement against the
        compressed operator (x += solve(rhs - apply(x))); 0 (default) is the
        reference's plain solve.  On the ill-conditioned cfg3 geometry one step
        lowers the exact-operator residual ~20x."""
        if refine > 0:
            x = self.solve(rhs, workers)
            for _ in range(refine):
                r = (rhs - self.apply(x)) if not isinstance(rhs, torch.Tensor) else \
                    (rhs.to(torch.float64) - self.apply(x))
                x = x + self.solve(r, workers)
            return x
        is_t = isinstance(rhs, torch.Tensor)
        r = rhs if is_t else np.asarray(rhs, float)
        if r.shape[0] != self.dim:
            raise ValueError(f"dimension mismatch: got {r.shape[0]}, need {self.dim}")
        _DevSlab.flush()
        vec = r.ndim == 1
        if is_t:
            x = r.to(device=_dev(), dtype=torch.float64).reshape(self.dim, -1).clone()
        else:
            x = torch.from_numpy(np.ascontiguousarray(r.reshape(self.dim, -1))).to(_dev())
        x = x.contiguous()
        self._solve_graphed(x)
        if is_t:
            return x.reshape(-1) if vec else x
        # device -> pinned host (the returned array views the pinned block)
        hp = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
        hp.copy_(x, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        out = hp.numpy()
        return out.reshape(-1) if vec else out

    def apply(self, x, workers: int = 1):
        """Compressed product ~ A x (reference skel.py:126-164); vectors or matrices."""
        is_t = isinstance(x, torch.Tensor)
        xa = x if is_t else np.asarray(x, float)
        if xa.shape[0] != self.dim:
            raise ValueError(f"dimension mismatch: got {xa.shape[0]}, need {self.dim}")
        vec = xa.ndim == 1
        dev = _dev()
        X = (xa.to(device=dev, dtype=torch.float64) if is_t
             else torch.from_numpy(np.ascontiguousarray(xa)).to(dev)).reshape(self.dim, -1)
        nr = X.shape[1]
        nd, q = self.n_dofs, self.q
        s = _stream()
        y = X[:nd].clone().contiguous()
        lam = X[nd:].clone().contiguous()
        keep = []
        # V^-1 upward: y_S += T y_R ; y_R += X_rs_div y_S
        for L in self.levels:
            B = len(L.k)
            xs = torch.empty(max(int(L.k.sum()) * nr, 1), dtype=torch.float64, device=dev)
            xr = torch.empty(max(int(L.r.sum()) * nr, 1), dtype=torch.float64, device=dev)
            ps, u1 = self._gather(L, "s", y, nr, xs)
            pr, u2 = self._gather(L, "r", y, nr, xr)
            keep += [u1, u2, xs, xr]
            one = np.ones(B)
            _gemm([dict(A=L.P["T"], B=pr, C=ps, D=ps, m=L.k, n=nr, k=L.r, lda=L.r, ldb=nr,
                        ldc=nr, ldd=nr, alpha=one, beta=one)])
            _gemm([dict(A=L.P["Xrsdiv"], B=ps, C=pr, D=pr, m=L.r, n=nr, k=L.k, lda=L.k, ldb=nr,
                        ldc=nr, ldd=nr, alpha=one, beta=one)])
            self._scatter(L, "s", y, nr, ps, keep)
            self._scatter(L, "r", y, nr, pr, keep)
        bottom = None
        if q:
            bottom = torch.empty((q, nr), dtype=torch.float64, device=dev)
            # bottom = PsiV^T y - lam (all rows incl. root), column-sparse, compensated
            pl = self._psi_lists(True)
            call("skb_psi_dot", q, pl["off"], pl["rows"], self.PsiV, q, y, nr, nr, None, nr, 1.0,
                 bottom, nr, s)
            call("skb_sum_partials", q * nr, 1, lam, q * nr, bottom, -1.0, bottom, s)
        # X_D: y_R <- X_rr y_R (stash y_R), y_root <- E_root y_root, y += UH lam
        stash = []
        for L in self.levels:
            B = len(L.k)
            xr = torch.empty(max(int(L.r.sum()) * nr, 1), dtype=torch.float64, device=dev)
            yr = torch.empty(max(int(L.r.sum()) * nr, 1), dtype=torch.float64, device=dev)
            pr, u2 = self._gather(L, "r", y, nr, xr)
            o = np.zeros(B + 1, np.int64)
            np.cumsum(L.r * nr, out=o[1:])
            py = (_addr(yr) + 8 * o[:-1]).astype(np.uint64)
            _gemm([dict(A=L.P["Xrr"], B=pr, D=py, m=L.r, n=nr, k=L.r, lda=L.r, ldb=nr, ldd=nr,
                        alpha=np.ones(B), beta=np.zeros(B))])
            self._scatter(L, "r", y, nr, py, keep)
            stash.append((pr, xr))
            keep += [u2, yr]
        ns = len(self.root_dofs)
        rd = self._root_d
        up = _upload(o=np.zeros(1, np.int64), ld=np.array([nr], np.int64),
                     ro=np.array([0, ns], np.int64))
        yroot = torch.empty((ns, nr), dtype=torch.float64, device=dev)
        yroot2 = torch.empty((ns, nr), dtype=torch.float64, device=dev)
        call("skb_gather_rows", 1, ptr(up["ro"]), ptr(rd["r"]), None, None, nr, ptr(y), nr,
             ptr(yroot), ptr(up["o"]), ptr(up["ld"]), ns, nr, s)
        _gemm([dict(A=np.array([_addr(self.E_root)], np.uint64), B=np.array([_addr(yroot)], np.uint64),
                    D=np.array([_addr(yroot2)], np.uint64), m=[ns], n=[nr], k=[ns], lda=[ns],
                    ldb=[nr], ldd=[nr], alpha=[1.0], beta=[0.0])])
        call("skb_scatter_rows", 1, ptr(up["ro"]), ptr(rd["r"]), None, None, nr, _addr(yroot2),
             ptr(up["o"]), ptr(up["ld"]), ptr(y), nr, 0, 1.0, ns, nr, s)
        keep += [up, yroot, yroot2]
        if q:
            _gemm([dict(A=np.array([_addr(self.UH)], np.uint64), B=np.array([_addr(lam)], np.uint64),
                        C=np.array([_addr(y)], np.uint64), D=np.array([_addr(y)], np.uint64),
                        m=[nd], n=[nr], k=[q], lda=[q], ldb=[nr], ldc=[nr], ldd=[nr],
                        alpha=[1.0], beta=[1.0])])
        # U^-1 downward: t = stash + UH_div[rd] lam ; y_S += X_sr t ; y_R += T^T y_S
        for L, (pr, xr) in zip(reversed(self.levels), reversed(stash)):
            B = len(L.k)
            one = np.ones(B)
            if q:
                ud = torch.empty(max(int(L.r.sum()) * q, 1), dtype=torch.float64, device=dev)
                pu, u3 = self._gather(L, "r", self.UH_div, q, ud)
                _gemm([dict(A=pu, B=np.full(B, _addr(lam), np.uint64), C=pr, D=pr, m=L.r, n=nr,
                            k=np.full(B, q), lda=np.full(B, q), ldb=nr, ldc=nr, ldd=nr,
                            alpha=one, beta=one)])
                keep += [ud, u3]
            xs = torch.empty(max(int(L.k.sum()) * nr, 1), dtype=torch.float64, device=dev)
            ps, u1 = self._gather(L, "s", y, nr, xs)
            _gemm([dict(A=L.P["Xsr"], B=pr, C=ps, D=ps, m=L.k, n=nr, k=L.r, lda=L.r, ldb=nr,
                        ldc=nr, ldd=nr, alpha=one, beta=one)])
            yr = torch.empty(max(int(L.r.sum()) * nr, 1), dtype=torch.float64, device=dev)
            py2, u4 = self._gather(L, "r", y, nr, yr)
            _gemm([dict(A=L.P["T"], B=ps, C=py2, D=py2, m=L.r, n=nr, k=L.k, lda=L.r, ldb=nr,
                        ldc=nr, ldd=nr, alpha=one, beta=one, transA=1)])
            self._scatter(L, "s", y, nr, ps, keep)
            self._scatter(L, "r", y, nr, py2, keep)
            keep += [xs, u1, yr, u4]
        out = torch.cat([y, bottom], dim=0) if q else y
        torch.cuda.current_stream().synchronize()
        if is_t:
            return out.reshape(-1) if vec else out
        o = out.cpu().numpy()
        return o.reshape(-1) if vec else o


# ---------------------------------------------------------------------------
# _finish_top and the drivers
# ---------------------------------------------------------------------------
def _hole_columns(t: Tree, b, idx, pairs=None):
    """Augmentation columns touched by each box: 3 per hole with nodes in the box
    (PsiV rows of a box's DOFs are zero outside these columns)."""
    idx = np.asarray(idx, np.int64)
    B = len(idx)
    if b.n_holes == 0 or B == 0:
        return np.zeros(B + 1, np.int64), np.zeros(0, np.int64)
    if pairs is None:
        pairs = t.hole_pairs(np.asarray(b.offsets, np.int64))
    pb, pc = pairs
    pos = np.searchsorted(pb, idx)
    end = np.searchsorted(pb, idx, side="right")
    lens = end - pos
    off, sel = _seg_gather(np.arange(len(pb)), pos, lens)
    cur = pc[sel]
    holes = cur >= 1
    owner = np.repeat(np.arange(B), lens)[holes]
    h = cur[holes] - 1
    cols = (3 * h[:, None] + np.arange(3)[None, :]).ravel()
    cnt = np.bincount(owner, minlength=B) * 3
    o = np.zeros(B + 1, np.int64)
    np.cumsum(cnt, out=o[1:])
    return o, cols.astype(np.int64)


class _AugPipe:
    """U sweep on H / V^T sweep on Psi (reference _finish_top, skel.py:379-396),
    run per level on a side stream as soon as the level's factors are final, so
    it overlaps the factorisation of the levels above.  Every box's outgoing
    skeleton rows and Schur part are kept per level (LevelFactors.stash) for
    the incremental sweep of a later update()."""

    def __init__(self, ctx: _Ctx):
        b = ctx.b
        self.q = 3 * b.n_holes if ctx.spec.augmented(b) else 0
        if not self.q:
            return
        dev = _dev()
        nd, q = 2 * b.n_nodes, self.q
        self.UH = torch.empty((nd, q), dtype=torch.float64, device=dev)
        self.PsiV = torch.empty((nd, q), dtype=torch.float64, device=dev)
        self.UH_div = torch.zeros((nd, q), dtype=torch.float64, device=dev)
        self.schur = torch.zeros((q, q), dtype=torch.float64, device=dev)
        self._hc = torch.from_numpy(np.ascontiguousarray(b.hole_centers, np.float64)).to(dev)
        call("skb_assemble_aug", ptr(ctx.g.pos), ptr(ctx.g.w), b.n_nodes, ptr(self._hc), b.n_holes,
             np.ascontiguousarray(b.offsets, np.int64), ptr(self.UH), ptr(self.PsiV), _stream())
        self.stream = _aug_stream()
        self.src = ctx.sstream

    def _wait_inputs(self):
        # the level's Schur work (level stream) and its descriptor uploads /
        # H, Psi assembly (current stream) must both precede the sweep
        for st in (self.src, torch.cuda.current_stream()):
            ev = torch.cuda.Event()
            ev.record(st)
            self.stream.wait_event(ev)

    def submit(self, L: "LevelFactors"):
        if not self.q:
            return
        self._wait_inputs()
        with torch.cuda.stream(self.stream):
            _stash_alloc(L, self.q)
            _aug_level(L, self.UH, self.PsiV, self.UH_div, self.schur, self.q)

    def join(self):
        if self.q:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            torch.cuda.current_stream().wait_event(ev)


_INC_SWEEP = os.environ.get("SKB_INC_SWEEP", "1") != "0"


def _make_pipe(ctx: "_Ctx"):
    upd = getattr(ctx, "upd_old", None) if (_INC_SWEEP and getattr(ctx, "upd_inc", True)) else None
    return _AugPipeUpdate(ctx, *upd) if upd is not None else _AugPipe(ctx)


def _stash_alloc(L: "LevelFactors", q: int):
    """Per-box storage of a level's sweep results: outgoing UH_S (k x q),
    PsiV_S (k x nc), Schur part (nc x q); element offsets per box."""
    k, nc = L.k, L.ncols
    us = k * q
    ps = k * nc
    sp = nc * q
    st_us = np.zeros(len(k), np.int64)
    np.cumsum(us[:-1], out=st_us[1:])
    base_ps = int(us.sum())
    st_ps = np.full(len(k), base_ps, np.int64)
    np.cumsum(ps[:-1], out=st_ps[1:])
    st_ps[1:] += base_ps
    base_sp = base_ps + int(ps.sum())
    st_sp = np.full(len(k), base_sp, np.int64)
    np.cumsum(sp[:-1], out=st_sp[1:])
    st_sp[1:] += base_sp
    L.stash = _DevSlab(8 * max(base_sp + int(sp.sum()), 1), torch.cuda.current_stream())
    L.st_us, L.st_ps, L.st_sp = st_us, st_ps, st_sp


class _AugPipeUpdate(_AugPipe):
    """Incremental _finish_top for update() (the
    reference recomputes it all, skel.py:510).  The sweep is linear in (H, Psi)
    and a box's step touches only its own active rows, so:

    * boxes whose factors were reused (clean) redo only the columns of the
      moved holes (their H columns change everywhere) -- skb_level_aug_narrow;
      their other columns, final UH / PsiV / UH_div rows and Schur parts are
      the previous factorization's (copied);
    * recompressed (dirty) boxes redo every column -- skb_level_aug -- starting
      from fresh H / Psi rows for dirty leaves and, above a clean child, from
      that child's stored outgoing skeleton rows (skb_restore_rows);
    * the corner's Schur block is re-accumulated from the stored per-box parts
      level by level in the refactor's order.

    Every kernel gives the same bits restricted to a column subset as on all
    columns (fixed-K-order DMMA GEMM, per-column triangular solves), so the
    result equals the full sweep bitwise (tests/test_gpu_parity.py)."""

    def __init__(self, ctx: _Ctx, old: "Factorization", dmask):
        b = ctx.b
        self.q = 3 * b.n_holes if ctx.spec.augmented(b) else 0
        if not self.q or old.UH is None:
            if self.q:
                _AugPipe.__init__(self, ctx)
            self.inc = False
            return
        self.inc = True
        dev = _dev()
        nd, q = 2 * b.n_nodes, self.q
        t = ctx.t
        s = _stream()
        self.UH = old.UH.clone()
        self.PsiV = old.PsiV.clone()
        self.UH_div = old.UH_div.clone()
        self.schur = torch.zeros((q, q), dtype=torch.float64, device=dev)
        H0 = torch.empty((nd, q), dtype=torch.float64, device=dev)
        P0 = torch.empty((nd, q), dtype=torch.float64, device=dev)
        self._hc = torch.from_numpy(np.ascontiguousarray(b.hole_centers, np.float64)).to(dev)
        call("skb_assemble_aug", ptr(ctx.g.pos), ptr(ctx.g.w), b.n_nodes, ptr(self._hc), b.n_holes,
             np.ascontiguousarray(b.offsets, np.int64), ptr(H0), ptr(P0), s)
        # columns of holes whose centre moved; rows of every dirty leaf
        moved = np.flatnonzero(np.any(old.boundary.hole_centers != b.hole_centers, axis=1))
        self.qc = (3 * moved[:, None] + np.arange(3)[None, :]).ravel().astype(np.int64)
        qmask = np.zeros(q, np.uint8)
        qmask[self.qc] = 1
        leaves = np.flatnonzero(t.is_leaf & dmask)
        nodes = [t.nodes_of(i) for i in leaves]
        nodes = np.concatenate(nodes) if nodes else np.zeros(0, np.int64)
        rows = np.sort((2 * nodes[:, None] + np.arange(2)[None, :]).ravel()).astype(np.int64)
        up = _upload(rows=rows if len(rows) else np.zeros(1, np.int64),
                     qc=self.qc if len(self.qc) else np.zeros(1, np.int64), qmask=qmask)
        for src, dst in ((H0, self.UH), (P0, self.PsiV)):
            call("skb_copy_rows_cols", len(rows), up["rows"], len(self.qc), up["qc"], nd, q, src, dst, s)
        self._keep = (up, H0, P0)
        self.qmask_d = up["qmask"]
        self.dmask = dmask
        self.tree = t
        self.stream = _aug_stream()
        self.src = ctx.sstream

    def submit(self, L: "LevelFactors"):
        if not self.q:
            return
        if not self.inc:
            return _AugPipe.submit(self, L)
        self._wait_inputs()
        with torch.cuda.stream(self.stream):
            self._submit(L)

    def _submit(self, L):
        q = self.q
        _stash_alloc(L, q)
        B = len(L.idx)
        dirty = self.dmask[L.idx]
        par = self.tree.parent[L.idx]
        pdirty = ((par >= 0) & self.dmask[np.maximum(par, 0)]).astype(np.uint8)
        old_us = np.zeros(B, np.uint64)
        old_ps = np.zeros(B, np.uint64)
        old_sp = np.zeros(B, np.uint64)
        cl = np.flatnonzero(~dirty)
        if len(cl):
            Lo, pos = L.batch.__dict__.pop("clean_old")     # drop the link to the old level
            base = _addr(Lo.stash)
            old_us[cl] = base + 8 * Lo.st_us[pos]
            old_ps[cl] = base + 8 * Lo.st_ps[pos]
            old_sp[cl] = base + 8 * Lo.st_sp[pos]
        z = np.zeros(1, np.int64)
        call("skb_level_aug_update", B, L.k, L.r, q, L.cols_off, L.cols if len(L.cols) else z,
             L.sd_off, L.sd if len(L.sd) else z, L.rd_off, L.rd if len(L.rd) else z,
             dirty.astype(np.uint8), pdirty, L.P["T"], L.P["LU"], L.P["Xsr"], L.P["Xrsdiv"], L.ipiv,
             old_us, old_ps, old_sp, len(self.qc), self.qc if len(self.qc) else z, ptr(self.qmask_d),
             ptr(self.UH), ptr(self.PsiV), ptr(self.UH_div), ptr(self.schur), ptr(L.stash), L.st_us,
             L.st_ps, L.st_sp, _stream())


def _finish_top(ctx: _Ctx, levels, store, pipe: "_AugPipe", before_sync=None):
    """Root block, augmentation sweep and corner LU (reference skel.py:364-425).
    ``before_sync`` runs after the corner LU is enqueued, before its status is
    read back (host work that overlaps the device tail)."""
    t, b = ctx.t, ctx.b
    dev = _dev()
    s = _stream()
    root = 0
    store.set_internal(t, np.array([root]))
    rd = store.act(root).copy()
    ns = len(rd)
    nd = ctx.dpn * b.n_nodes
    q = 3 * b.n_holes if ctx.spec.augmented(b) else 0
    co, cx = ctx.child_desc(np.array([root]), store)
    E_root = torch.empty((max(ns, 1), max(ns, 1)), dtype=torch.float64, device=dev)
    up = _upload(ao=np.array([0, ns], np.int64), a=rd if ns else np.zeros(1, np.int64),
                 co=co.reshape(-1), cx=cx.reshape(-1), eo=np.zeros(1, np.int64),
                 eld=np.array([ns], np.int64))
    call("skb_assemble_self" if ctx.dpn == 2 else "skb_assemble_self_lap",
         ptr(ctx.g.pos), ptr(ctx.g.nrm), ptr(ctx.g.w), ptr(ctx.g.kap), 1,
         ptr(up["ao"]), ptr(up["a"]), None, None, ptr(up["co"]), ptr(up["cx"]), ptr(E_root),
         ptr(up["eo"]), ptr(up["eld"]), ns, s)
    UH = PsiV = UH_div = None
    if q:
        _Prof.start()
        pipe.join()                                  # sweeps were issued level by level
        _Prof.tick("d_aug_sweep")
        UH, PsiV, UH_div, schur = pipe.UH, pipe.PsiV, pipe.UH_div, pipe.schur
        if getattr(pipe, "inc", False) and ns:
            # UH_div rows of root DOFs are never written by the sweep (zero in a
            # refactor); the incremental sweep started from the previous UH_div
            call("skb_fill_rows", ns, ptr(up["a"]), ptr(UH_div), q, None, q, 0.0, s)
        n = ns + q
        top = torch.empty((n, n), dtype=torch.float64, device=dev)
        call("skb_copy2d_batched", 1, _mats([_addr(top)], [ns], [ns], [n]),
             _mats([_addr(E_root)], [ns], [ns], [ns]), 0, s)
        # corner[:ns, ns:] = UH[root]; corner[ns:, :ns] = PsiV[root]^T; corner[ns:, ns:] = -I - schur
        up2 = _upload(o=np.array([ns], np.int64), ld=np.array([n], np.int64),
                      o0=np.zeros(1, np.int64), ldq=np.array([q], np.int64))
        call("skb_gather_rows", 1, ptr(up["ao"]), ptr(up["a"]), None, None, q, ptr(UH), q,
             ptr(top), ptr(up2["o"]), ptr(up2["ld"]), ns, q, s)
        tmp = torch.empty((max(ns, 1), q), dtype=torch.float64, device=dev)
        call("skb_gather_rows", 1, ptr(up["ao"]), ptr(up["a"]), None, None, q, ptr(PsiV), q,
             ptr(tmp), ptr(up2["o0"]), ptr(up2["ldq"]), ns, q, s)
        call("skb_copy2d_batched", 1, _mats([_addr(top) + 8 * ns * n], [q], [ns], [n]),
             _mats([_addr(tmp)], [ns], [q], [q]), 1, s)
        call("skb_diag_fill", q, _addr(top) + 8 * (ns * n + ns), n, -1.0, ptr(schur), q, -1.0, s)
        del tmp
    else:
        n = ns
        top = torch.empty((max(n, 1), max(n, 1)), dtype=torch.float64, device=dev)
        top.copy_(E_root)
    ipiv = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    info = torch.empty(1, dtype=torch.int32, device=dev)
    ratio = torch.empty(1, dtype=torch.float64, device=dev)
    _Prof.start()
    call("skb_getrf_batched", 1, _mats([_addr(top)], [n], [n], [n]),
         np.array([_addr(ipiv)], np.uint64), ptr(info), ptr(ratio), s)
    if before_sync is not None:
        before_sync()
    inf = int(info.cpu().item())
    _Prof.tick("d_corner_lu")
    if inf >= 0:
        raise SingularPivotError(inf)
    return rd, E_root, top, ipiv, UH, PsiV, UH_div, q, float(ratio.cpu().item())


def _aug_level(L: LevelFactors, UH, PsiV, UH_div, schur, q):
    """U sweep on H and V^T sweep on Psi for one level (skel.py:384-396), one native call."""
    d = L.d
    call("skb_level_aug", len(L.k), L.k, L.r, q, L.cols_off,
         L.cols if len(L.cols) else np.zeros(1, np.int64), ptr(d["sd_off"]), ptr(d["sd"]),
         ptr(d["rd_off"]), ptr(d["rd"]), ptr(d["c_off"]), ptr(d["c"]), L.P["T"], L.P["LU"],
         L.P["Xsr"], L.P["Xrsdiv"], L.ipiv, ptr(UH), ptr(PsiV), ptr(UH_div), ptr(schur),
         ptr(L.stash), L.st_us, L.st_ps, L.st_sp, 1, _stream())


# The native level engine (csrc/engine.cu) drives factor() unless SKB_ENGINE=0
# (then the single-threaded level loop below, which update() always uses).
_ENGINE_ON = os.environ.get("SKB_ENGINE", "1") != "0"


class _EngineAbort(Exception):
    """A migration (R -> S, skel.py:317-330) was detected while the native
    engine runs ahead: the factorization restarts on the Python level path."""


def _i64p(vals):
    return (ctypes.c_uint64 * len(vals))(*[int(v) for v in vals])


_PREWARMED = [0]
_PREWARM_KB = float(os.environ.get("SKB_PREWARM_KB_PER_DOF", "12"))


def _prewarm_pools(lib, n_dofs: int):
    """Reserve the engine's and the default stream-ordered pool for a problem
    of n_dofs unknowns before the first level runs (ID stacks of ~3 levels in
    flight: ~12 KB per unknown; Schur scratch half of that).  Pool growth in
    the middle of a factorization stalls the host for 30-200 ms."""
    if n_dofs <= _PREWARMED[0] or _PREWARM_KB <= 0:
        return
    _PREWARMED[0] = n_dofs
    eb = int(_PREWARM_KB * 1024 * n_dofs)
    rc = lib.skb_pool_prewarm(eb, eb // 2)
    if rc:
        raise _lib.SkbError(f"skb_pool_prewarm returned {rc}")


class _Engine:
    """Host handle of the native level engine (csrc/engine.cu)."""

    def __init__(self, ctx: "_Ctx", store: "ActStore", update=None):
        t, g = ctx.t, ctx.g
        nv = _tree_native(t)
        self.lib = _lib.load()
        _prewarm_pools(self.lib, ctx.dpn * t.n_nodes)
        self._keep = [nv, store]
        self.children = np.ascontiguousarray(t.children, np.int64)
        self.px, self.py = ctx.px, ctx.py
        self.cs = np.ascontiguousarray(ctx.cs, np.float64)
        self.fill = np.array([store.fill], np.int64)
        self.store = store
        tree = _i64p([nv["center"].ctypes.data, nv["hw"].ctypes.data, nv["nbr"].ctypes.data,
                      nv["lev"].ctypes.data, nv["ix"].ctypes.data, nv["iy"].ctypes.data,
                      self.children.ctypes.data, nv["ls"].ctypes.data, nv["leaf"].ctypes.data])
        st = _i64p([store.big.ctypes.data, store.a_start.ctypes.data, store.a_len.ctypes.data,
                    store.s_start.ctypes.data, store.s_len.ctypes.data, self.fill.ctypes.data])
        geo = _i64p([self.px.ctypes.data, self.py.ctypes.data, ptr(g.pos), ptr(g.nrm), ptr(g.w),
                     self.cs.ctypes.data])
        self.h = ctypes.c_int64(0)
        with _ht("E.start.c"):
            rc = self.lib.skb_engine_start(tree, t.depth, nv["root"].ctypes.data, ctx.factor, st,
                                           len(store.big), geo, ctx.P, ctx.tol, _stream(),
                                           0 if update is not None else 1,
                                           2 * t.n_nodes + 3 * len(t.lev) + 16, ctx.pde,
                                           ctypes.byref(self.h))
        if rc:
            raise _lib.SkbError(f"skb_engine_start returned {rc}")
        self.h = self.h.value
        if update is not None:
            self._upd = update                      # kept alive while the engine runs
            if len(update) == 2:                    # (todo, previous level table): native driver
                todo, table = update
                self.lib.skb_engine_set_update_table(self.h, todo.ctypes.data, table.ctypes.data)
            else:
                todo, coff, cskel = update
                self.lib.skb_engine_set_update(self.h, todo.ctypes.data, coff.ctypes.data,
                                               cskel.ctypes.data)
            self.lib.skb_engine_go(self.h)
        # Run-ahead of the engine over the enqueued Schur stages.  On trees
        # with heavy levels (> 512 boxes, cfg3) the engine enqueues level L's
        # kernels once level L+2's Schur stage is enqueued (lead 1): bounded
        # device memory (ID stacks of three levels in flight) at the speed of
        # unbounded run-ahead (cfg3 160 vs 171 ms at lead 0).  With the pools
        # reserved up front (_prewarm_pools) and the consumer loop native, 600
        # consecutive cfg3 factorizations stayed within 166 ms
        # (scripts/stall_hunt.py); the 0.3-1 s outliers seen with the Python
        # consumer at lead >= 1 were pool growth and interpreter pauses.
        # Lighter trees and updates (a few boxes per level) run ahead
        # unbounded.  SKB_ENGINE_LEAD=n overrides.  Levels without boxes to
        # compress count as acknowledged (engine.cu).
        heavy = update is None and int(np.diff(t.level_start).max(initial=0)) > 512
        lead = int(os.environ.get("SKB_ENGINE_LEAD", "1" if heavy else "-1"))
        if lead >= 0:
            self.lib.skb_engine_set_lead(self.h, lead)
        self.sizes = np.zeros(8, np.int64)
        self.ptrs = np.zeros(14, np.int64)

    @staticmethod
    def _arr(addr, n, dt):
        if not n:
            return np.zeros(0, dt)
        nb = n * np.dtype(dt).itemsize
        return np.frombuffer((ctypes.c_char * nb).from_address(int(addr)), dtype=dt).copy()

    def wait(self, L) -> dict:
        with _ht("E.wait"):
            self.lib.skb_engine_wait(self.h, L, self.sizes.ctypes.data, self.ptrs.ctypes.data)
        rc, B, na, box0, o_int, o_act, h2d, d2h = (int(v) for v in self.sizes)
        IO["h2d"] += h2d
        IO["d2h"] += d2h
        if rc:
            raise _lib.SkbError(f"native level engine failed at level {L} (rc {rc})")
        p = self.ptrs
        if B == 0:
            return None
        act_off = self._arr(p[0], B + 1, np.int64)
        act = self._arr(p[1], na, np.int64)
        rows = self._arr(p[2], B, np.int64)
        nB = np.diff(act_off)
        dbuf, dup = int(p[10]), int(p[11])
        h = dict(idx=self._arr(p[13], B, np.int64), act_off=act_off, act=act, nB=nB,
                 rows=rows, pre=rows > 2 * nB, m_q=self._arr(p[4], B, np.int64),
                 A=self._arr(p[3], B, np.int64), lda=rows, engine=self, lev=L,
                 dev=(dup, dup + 8 * o_act, dbuf + o_int),
                 perm=self._arr(p[5], na, np.int32), k=self._arr(p[6], B, np.int32),
                 steps=self._arr(p[7], B, np.int32), gap=self._arr(p[8], B, np.float64))
        return h

    def stream_wait(self, L, stream):
        self.lib.skb_engine_stream_wait(self.h, L, stream.cuda_stream)

    def release(self, L, stream):
        self.lib.skb_engine_release(self.h, L, stream.cuda_stream)
        self.lib.skb_engine_ack(self.h, L)

    def close(self, stop=False):
        if self.h:
            if stop:
                self.lib.skb_engine_stop(self.h)
            self.lib.skb_engine_free(self.h, _stream())
            self.h = 0
            self.store.fill = int(self.fill[0])

    def __del__(self):
        try:
            self.close(stop=True)
        except Exception:
            pass



# The native level driver (csrc/engine.cu skb_drv_run) consumes the engine's
# levels in C++ (merge, layout, Schur stage, sweep, level lists); this module
# only wraps the resulting arrays.  SKB_NATIVE=0 keeps the Python consumer loop.
_NATIVE_ON = os.environ.get("SKB_NATIVE", "1") != "0"
_O_NF = 21


class _RawDev:
    """Device address with the data_ptr() protocol of a tensor."""
    __slots__ = ("p",)

    def __init__(self, p):
        self.p = int(p)

    def data_ptr(self) -> int:
        return self.p


def _level_code(L: "LevelFactors"):
    c = L.__dict__.get("code")
    if c is None:
        side = np.int64(1) << np.int64(L.lev)
        c = L.code = np.ascontiguousarray(L.tree.ix[L.idx] * side + L.tree.iy[L.idx], np.int64)
    return c


def _level_row(L: "LevelFactors"):
    """Row of the previous-factorization table (engine.cu OldLevel) for one level."""
    row = L.__dict__.get("_row")
    if row is not None:
        return row
    bt = L.batch
    bt.resolve()
    keep = [_level_code(L), np.ascontiguousarray(bt.act_off, np.int64), np.ascontiguousarray(bt.act, np.int64),
            np.ascontiguousarray(bt.perm, np.int32), np.ascontiguousarray(bt.k, np.int64)]
    keep += [np.ascontiguousarray(bt.ptr[f], np.uint64) for f in BoxBatch.FIELDS]
    keep += [np.ascontiguousarray(bt.ipiv, np.uint64), np.ascontiguousarray(bt.info, np.int64),
             np.ascontiguousarray(bt.ratio, np.float64)]
    st = L.__dict__.get("stash")
    row = np.zeros(_O_NF, np.int64)
    row[0] = len(L.idx)
    for i, a in enumerate(keep):
        row[1 + i] = a.ctypes.data
    if st is not None:
        sts = [np.ascontiguousarray(L.st_us, np.int64), np.ascontiguousarray(L.st_ps, np.int64),
               np.ascontiguousarray(L.st_sp, np.int64)]
        row[15] = _addr(st)
        row[16], row[17], row[18] = (a.ctypes.data for a in sts)
        keep += sts
    tail = [np.ascontiguousarray(bt.gap, np.float64), np.ascontiguousarray(bt.steps, np.int64)]
    row[19], row[20] = tail[0].ctypes.data, tail[1].ctypes.data
    L._row_keep = keep + tail
    L._row = row
    return row


def _native_level(lib, drv, lev, t, old, sizes, ptrs):
    """LevelFactors / BoxBatch of one level from the native driver's arrays."""
    rc = lib.skb_drv_level(drv, lev, sizes.ctypes.data, ptrs.ctypes.data)
    if rc:
        raise _lib.SkbError(f"skb_drv_level returned {rc}")
    B, na, nnew, nsd, nrd, ncl = (int(v) for v in sizes[:6])
    slab, slab_b, stash, stash_b, desc, desc_b = (int(v) for v in sizes[6:12])
    od = [int(v) for v in sizes[12:18]]
    arr = _Engine._arr
    p = ptrs
    i64, u64, f64 = np.int64, np.uint64, np.float64
    bt = BoxBatch.__new__(BoxBatch)
    bt.idx = arr(p[0], B, i64)
    bt.act_off = arr(p[2], B + 1, i64)
    bt.act = arr(p[3], na, i64)
    bt.nB = np.diff(bt.act_off)
    bt.perm = arr(p[4], na, np.int32)
    bt.k = arr(p[5], B, i64)
    bt.steps = arr(p[6], B, i64)
    bt.gap = arr(p[7], B, f64)
    bt.info = arr(p[8], B, i64)
    bt.ratio = arr(p[9], B, f64)
    bt.ptr = {f: arr(p[11 + i], B, u64) for i, f in enumerate(BoxBatch.FIELDS)}
    bt.ipiv = arr(p[17], B, u64)
    bt.slabs = []
    bt.slab_of = np.full(B, -1, i64)
    if nnew and slab:
        bt.slabs.append(_DevSlab.adopt(slab, slab_b))
        bt.slab_of[arr(p[27], nnew, i64)] = 0
    if nnew < B:
        cpos = arr(p[10], B, i64)
        clean = np.flatnonzero(cpos >= 0)
        ob = old[lev].batch
        so = ob.slab_of[cpos[clean]]
        lut = np.full(max(len(ob.slabs), 1), -1, i64)
        for u in np.unique(so[so >= 0]):
            lut[u] = len(bt.slabs)
            bt.slabs.append(ob.slabs[u])
        bt.slab_of[clean] = np.where(so >= 0, lut[np.maximum(so, 0)], -1)
    L = LevelFactors.__new__(LevelFactors)
    L.lev, L.tree, L.batch, L.idx = lev, t, bt, bt.idx
    L.code = arr(p[1], B, i64)
    L.k = bt.k.copy()
    L.r = bt.nB - bt.k
    L.sd_off, L.sd = arr(p[18], B + 1, i64), arr(p[19], nsd, i64)
    L.rd_off, L.rd = arr(p[20], B + 1, i64), arr(p[21], nrd, i64)
    L.cols_off, L.cols = arr(p[22], B + 1, i64), arr(p[23], ncl, i64)
    L.ncols = np.diff(L.cols_off)
    keep = _DevSlab.adopt(desc, desc_b)
    L.d = {n: _RawDev(desc + 8 * o) for n, o in zip(("sd_off", "sd", "rd_off", "rd", "c_off", "c"), od)}
    L.d["_keep"] = keep
    L.P = {f: bt.ptr[f] for f in BoxBatch.FIELDS}
    L.ipiv = bt.ipiv
    if stash:
        L.stash = _DevSlab.adopt(stash, stash_b)
        L.st_us, L.st_ps, L.st_sp = arr(p[24], B, i64), arr(p[25], B, i64), arr(p[26], B, i64)
    return L


def _run_levels_native(ctx: _Ctx, upd=None):
    """Level loop of factor() / update() on the native engine + driver."""
    t, b = ctx.t, ctx.b
    lib = _lib.load()
    with _ht("N.store"):
        store = ActStore(t, engine=True, dpn=ctx.dpn)
    ctx.store = store
    old = None
    eupd = None
    table = None
    if upd is not None:
        old_fct, dmask = upd[0], upd[1]
        old = upd[2] if len(upd) > 2 else {L.lev: L for L in old_fct.levels}
        with _ht("N.table"):
            table = np.zeros((max(t.depth, max(old, default=0)) + 1, _O_NF), np.int64)
            for lev, L in old.items():
                table[lev] = _level_row(L)
        dm8 = np.ascontiguousarray(dmask, np.uint8)
        eupd = (dm8, table)
    with _ht("N.engine"):
        eng = _Engine(ctx, store, update=eupd)
    drv = ctypes.c_int64(0)
    try:
        with torch.cuda.stream(ctx.sstream):
            with _ht("N.pipe"):
                pipe = _make_pipe(ctx)
            ctx.pipe = pipe
            nv = _tree_native(t)
            cfg = np.zeros(24, np.int64)
            flat = getattr(t, "_level_nodes_flat", None)
            with _ht("N.pairs"):
                if b.n_holes and flat is not None:
                    # (box, curve) membership from the tree's node lists, in the driver
                    coff = np.ascontiguousarray(b.offsets, np.int64)
                    cfg[4], cfg[5], cfg[6] = -1, coff.ctypes.data, len(coff) - 1
                    cfg[20], cfg[21] = flat.ctypes.data, t._level_nodes_off.ctypes.data
                    cfg[22], cfg[23] = t.node_start.ctypes.data, t.node_cnt.ctypes.data
                elif b.n_holes:
                    pb, pc = t.hole_pairs(np.asarray(b.offsets, np.int64))
                    pb, pc = np.ascontiguousarray(pb, np.int64), np.ascontiguousarray(pc, np.int64)
                    cfg[4], cfg[5], cfg[6] = len(pb), pb.ctypes.data, pc.ctypes.data
            cfg[0] = _stream()
            cfg[2] = ptr(ctx.g.kap)
            cfg[3] = pipe.q
            cfg[7] = nv["parent"].ctypes.data
            if pipe.q:
                cfg[1] = pipe.stream.cuda_stream
                cfg[8], cfg[9], cfg[10], cfg[11] = ptr(pipe.UH), ptr(pipe.PsiV), ptr(pipe.UH_div), ptr(pipe.schur)
            inc = bool(getattr(pipe, "inc", False))
            if upd is not None:
                cfg[12] = 1
                cfg[13] = dm8.ctypes.data
                cfg[17] = table.ctypes.data
            if inc:
                qc = np.ascontiguousarray(pipe.qc, np.int64)
                cfg[14] = len(qc)
                cfg[15] = qc.ctypes.data if len(qc) else 0
                cfg[16] = ptr(pipe.qmask_d)
                cfg[18] = 1
            cfg[19] = store.xss.ctypes.data
            with _ht("N.run"):
                rc = lib.skb_drv_run(eng.h, cfg.ctypes.data, PIVOT_RATIO_FLOOR, ctypes.byref(drv))
            if rc in (100, 101):
                raise _EngineAbort()
            if rc == 102:
                raise RuntimeError("clean box changed its active set")
            if rc:
                raise _lib.SkbError(f"native level driver failed (rc {rc})")
        eng.close()
        torch.cuda.current_stream().wait_stream(ctx.sstream)
        return store, (lib, drv, old)
    except BaseException:
        eng.close(stop=True)
        if drv.value:
            lib.skb_drv_free(drv.value)
        raise


def _native_collect(ctx: _Ctx, handle):
    """Wrap the driver's per-level arrays (after the remaining device work has
    been enqueued: this host work overlaps it) and release the driver."""
    lib, drv, old = handle
    t = ctx.t
    sizes, ptrs = np.zeros(24, np.int64), np.zeros(32, np.int64)
    try:
        with _ht("N.resolve"):
            rc = lib.skb_drv_resolve(drv.value)        # waits for the last Schur stages
        if rc == 100:
            raise _EngineAbort()
        if rc:
            raise _lib.SkbError(f"skb_drv_resolve returned {rc}")
        with _ht("N.collect"):
            levels = [_native_level(lib, drv.value, lev, t, old, sizes, ptrs)
                      for lev in range(t.depth, 0, -1)]
        IO["h2d"] += int(sizes[18])
        IO["d2h"] += int(sizes[19])
    finally:
        lib.skb_drv_free(drv.value)
        drv.value = 0                                  # (the caller's cleanup sees it released)
    return levels


def _run_levels_engine(ctx: _Ctx):
    """_run_levels for factor(): the compression chain runs in the native
    engine thread; this loop only consumes finished levels (Schur stage,
    migration check, augmentation sweep, level descriptors)."""
    t = ctx.t
    with _ht("E.store"):
        store = ActStore(t, engine=True, dpn=ctx.dpn)
    ctx.store = store
    with _ht("E.start"):
        eng = _Engine(ctx, store)
    try:
        with torch.cuda.stream(ctx.sstream):      # host-side work rides the level stream
            out = _engine_loop(ctx, eng, store)
        torch.cuda.current_stream().wait_stream(ctx.sstream)
        return out
    finally:
        eng.close(stop=True)


def _clean_skeletons(t: Tree, old_levels: dict, dmask):
    """Skeletons of the clean boxes of an update, carried over from the previous
    factorization (reference run_level reuse path, skel.py:342-353), as a CSR
    over all boxes of the new tree (dirty boxes empty)."""
    nbox = len(t.lev)
    lens = np.zeros(nbox, np.int64)
    parts = []
    for lev in range(1, t.depth + 1):
        idx = t.level_indices(lev)
        clean = idx[~dmask[idx]]
        if len(clean) == 0:
            continue
        L = old_levels.get(lev)
        if L is None:
            raise _EngineAbort()
        ot, ob = L.tree, L.batch
        side = np.int64(1) << np.int64(lev)
        oc = ot.ix[L.idx] * side + ot.iy[L.idx]
        nc = t.ix[clean] * side + t.iy[clean]
        pos = np.searchsorted(oc, nc)
        if np.any(pos >= len(oc)) or np.any(oc[np.minimum(pos, len(oc) - 1)] != nc):
            raise _EngineAbort()
        k = ob.k[pos]
        _, pp = _seg_gather(ob.perm.astype(np.int64), ob.act_off[pos], k)
        sk = ob.act[np.repeat(ob.act_off[pos], k) + pp]
        lens[clean] = k
        parts.append((clean, k, sk))
    off = np.zeros(nbox + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    flat = np.zeros(max(int(off[-1]), 1), np.int64)
    for clean, k, sk in parts:
        _, dst = _seg_gather(np.arange(len(flat)), off[clean], k)
        flat[dst] = sk
    return off, flat


def _run_levels_engine_update(ctx: _Ctx, old: dict, dmask):
    """_run_levels(reuse=old) on the native engine: only the dirty boxes are
    recompressed; clean boxes keep the previous factors."""
    t = ctx.t
    with _ht("U.clean"):
        coff, cskel = _clean_skeletons(t, old, dmask)
    with _ht("U.store"):
        store = ActStore(t, engine=True, dpn=ctx.dpn)
    ctx.store = store
    with _ht("U.engine"):
        eng = _Engine(ctx, store, update=(np.ascontiguousarray(dmask, np.uint8), coff, cskel))
    try:
        with torch.cuda.stream(ctx.sstream):
            out = _engine_loop(ctx, eng, store, reuse=old, dirty=dmask)
        torch.cuda.current_stream().wait_stream(ctx.sstream)
        return out
    finally:
        eng.close(stop=True)


def _engine_loop(ctx, eng, store, reuse=None, dirty=None):
        t = ctx.t
        pairs = t.hole_pairs(np.asarray(ctx.b.offsets, np.int64)) if ctx.b.n_holes else None
        pipe = _make_pipe(ctx)
        ctx.pipe = pipe
        levels = []
        prev = None
        for lev in range(t.depth, 0, -1):
            h = eng.wait(lev)
            bt_new = None
            if h is not None:
                bt_new = BoxBatch(h["idx"], h["act_off"], h["act"])
                bt_new.perm[:] = h["perm"]
                bt_new.k[:] = h["k"]
                bt_new.steps[:] = h["steps"]
                bt_new.gap[:] = h["gap"]
                bt_new._launch = h
            if prev is not None and prev[1] is not None:
                with _ht("migrate"):
                    pb = prev[1]
                    pb.resolve()
                    if (((pb.info >= 0) | (pb.ratio < PIVOT_RATIO_FLOOR)) & (pb.k < pb.nB)).any():
                        raise _EngineAbort()
            if reuse is None:
                bt = bt_new
            else:
                if bt_new is not None:
                    ctx.layout(bt_new)                # the merge copies factor pointers
                idx_all = t.level_indices(lev)
                todo = bt_new.idx if bt_new is not None else np.zeros(0, np.int64)
                bt = _merge_level(ctx, idx_all, store, todo, bt_new, reuse)
            if bt_new is not None:
                with _ht("schur"):
                    ctx.schur(bt_new, store)
            store.xss[bt.idx] = bt.ptr["Xss"]
            if prev is not None:
                with _ht("aug_submit"):
                    pipe.submit(levels[-1])
            with _ht("levelfactors"):
                cols_off, cols = _hole_columns(t, ctx.b, bt.idx, pairs)
                levels.append(LevelFactors(lev, t, bt, cols_off, cols))
            prev = (lev, bt_new)
        if prev is not None and prev[1] is not None:
            pb = prev[1]
            pb.resolve()
            if (((pb.info >= 0) | (pb.ratio < PIVOT_RATIO_FLOOR)) & (pb.k < pb.nB)).any():
                raise _EngineAbort()
        eng.close()
        if levels:
            pipe.submit(levels[-1])
        return levels, store, sum(len(L.idx) for L in levels) if reuse is None else 0


def _run_levels(ctx: _Ctx, reuse=None, dirty=None):
    """Bottom-up level loop (reference factor skel.py:443-449 / update skel.py:502-509).

    Software-pipelined: as soon as a level's QRCP results reach the host, the
    next level's ID stacks / QR / QRCP are launched (they need only the new
    skeleton lists), then this level's Schur complements go to the level
    stream, so the host bookkeeping and the Schur work overlap the critical
    QRCP -> host -> QRCP chain."""
    t = ctx.t
    store = ActStore(t, dpn=ctx.dpn)
    ctx.store = store
    levels = []
    n_recomp = 0
    prev = None          # (level, batch, fresh boxes) whose migration check is pending
    if _Prof.enabled:
        torch.cuda.synchronize()
        _Prof._lt = time.perf_counter()

    def pre(lev):
        """Level lev's batch and its skeleton-independent launch inputs."""
        idx = t.level_indices(lev)
        if reuse is None:
            todo = idx
        else:
            todo = idx[dirty[idx]]                 # dirty: mask over the tree's boxes
        with _ht("prep"):
            return idx, todo, (ctx.prep(todo) if len(todo) else None)

    def go(p):
        idx, todo, pr = p
        with _ht("set_internal"):
            store.set_internal(t, idx)        # assign_internal_actives, skel.py:251-256
        with _ht("launch"):
            return idx, todo, (ctx.launch(todo, store, prep=pr) if len(todo) else None)

    def fix_prev():
        pl, pbt, pnew = prev
        if pbt is not pnew:
            pos = np.searchsorted(pbt.idx, pnew.idx)
            pbt.take(pos, pnew, np.arange(len(pnew.idx)))
        store.set_skel(pbt.idx, pbt.act_off, pbt.act, pbt.perm, pbt.k)
        store.xss[pbt.idx] = pbt.ptr["Xss"]
        levels[-1] = LevelFactors(pl, t, pbt, *_hole_columns(t, ctx.b, pbt.idx, pairs))
        return (pl, pbt, None)

    lev = t.depth
    p_cur = pre(lev) if lev >= 1 else None
    cur = go(p_cur) if lev >= 1 else None            # first compression in flight first
    pairs = t.hole_pairs(np.asarray(ctx.b.offsets, np.int64)) if ctx.b.n_holes else None
    pipe = _make_pipe(ctx)
    ctx.pipe = pipe
    p_nxt = pre(lev - 1) if lev > 1 else None
    while lev >= 1:
        idx, todo, h = cur
        with _ht("finish"):
            bt_new = ctx.finish(h) if h is not None else None
        # the previous level's X_RR pivot ratios are available now (its kernels
        # ran before this sync); a migration there invalidates this level
        with _ht("migrate"):
            mig = prev is not None and prev[2] is not None and ctx.migrate(prev[2], store)
        if mig:
            prev = fix_prev()
            cur = go(p_cur)                   # redo this level on the corrected skeletons
            continue
        n_recomp += len(todo)
        if reuse is not None and bt_new is not None:
            ctx.layout(bt_new)                # merge copies the factor pointers
        bt = bt_new if reuse is None else _merge_level(ctx, idx, store, todo, bt_new, reuse)
        store.set_skel(bt.idx, bt.act_off, bt.act, bt.perm, bt.k)
        nxt = go(p_nxt) if lev > 1 else None          # critical path first
        if bt_new is not None:
            with _ht("schur"):
                ctx.schur(bt_new, store)
        store.xss[bt.idx] = bt.ptr["Xss"]             # laid out by schur()
        if prev is not None:
            with _ht("aug_submit"):
                pipe.submit(levels[-1])       # previous level final: start its aug sweep
        if _Prof.enabled:
            torch.cuda.synchronize()
            _Prof.acc[f"level{lev}"] = time.perf_counter() - _Prof._lt
            _Prof._lt = time.perf_counter()
        with _ht("levelfactors"):
            cols_off, cols = _hole_columns(t, ctx.b, bt.idx, pairs)
            levels.append(LevelFactors(lev, t, bt, cols_off, cols))
        prev = (lev, bt, bt_new)
        p_cur, p_nxt = p_nxt, (pre(lev - 2) if lev > 2 else None)   # while the GPU compresses
        lev -= 1
        cur = nxt
    if prev is not None and prev[2] is not None and ctx.migrate(prev[2], store):
        prev = fix_prev()
    if levels:
        pipe.submit(levels[-1])
    torch.cuda.current_stream().wait_stream(ctx.sstream)
    return levels, store, n_recomp


def _run_levels_pz(ctx: _Ctx):
    """Level loop of the validation mode ``propagate_zeros=True`` (reference
    skel.py:267-270, 354-361): the boxes of a level are compressed one after
    the other in key order, and a box's far field sees the SKELETONS of the
    colleagues compressed before it (the zeros they created) instead of their
    active sets.  Sequential by construction: one box per launch."""
    t = ctx.t
    store = ActStore(t, dpn=ctx.dpn)
    ctx.store = store
    pairs = t.hole_pairs(np.asarray(ctx.b.offsets, np.int64)) if ctx.b.n_holes else None
    pipe = _make_pipe(ctx)
    ctx.pipe = pipe
    levels = []
    n = 0
    for lev in range(t.depth, 0, -1):
        idx = t.level_indices(lev)
        store.set_internal(t, idx)                    # assign_internal_actives, skel.py:251-256
        act_off, act = store.acts(idx)                # the boxes' own active sets (before any substitution)
        bt = BoxBatch(idx, act_off, act)
        one = np.zeros(1, np.int64)
        for j, i in enumerate(idx):
            sub = ctx.compress(np.array([i], np.int64), store)
            ctx.migrate(sub, store)                   # R -> S migration, skel.py:317-330
            bt.take(np.array([j], np.int64), sub, one)
            store.set_skel(sub.idx, sub.act_off, sub.act, sub.perm, sub.k)
            # colleagues compressed after this box see its skeleton only
            store.a_start[i], store.a_len[i] = store.s_start[i], store.s_len[i]
            n += 1
        bt.resolve()
        store.xss[bt.idx] = bt.ptr["Xss"]
        if levels:
            pipe.submit(levels[-1])
        levels.append(LevelFactors(lev, t, bt, *_hole_columns(t, ctx.b, bt.idx, pairs)))
    if levels:
        pipe.submit(levels[-1])
    torch.cuda.current_stream().wait_stream(ctx.sstream)
    return levels, store, n


def _merge_level(ctx, idx, store, todo, bt_new, old_levels):
    """Level batch for an update: dirty boxes from bt_new, clean boxes share the
    old factor memory (reference run_level reuse path, skel.py:342-353)."""
    t = ctx.t
    act_off, act = store.acts(idx)
    bt = BoxBatch(idx, act_off, act)
    is_new = np.isin(idx, todo)
    if bt_new is not None and is_new.any():
        pos = np.searchsorted(bt_new.idx, idx[is_new])
        bt.take(np.flatnonzero(is_new), bt_new, pos)
    clean = np.flatnonzero(~is_new)
    if len(clean):
        lev = int(t.lev[idx[0]])
        L = old_levels[lev]
        ot = L.tree
        side = np.int64(1) << np.int64(lev)
        oc = ot.ix[L.idx] * side + ot.iy[L.idx]
        nc = t.ix[idx[clean]] * side + t.iy[idx[clean]]
        pos = np.searchsorted(oc, nc)
        if np.any(pos >= len(oc)) or np.any(oc[np.minimum(pos, len(oc) - 1)] != nc):
            raise RuntimeError("clean box missing from the previous factorization")
        ob = L.batch
        lens = bt.nB[clean]
        if not np.array_equal(lens, ob.nB[pos]):
            raise RuntimeError("clean box changed its active set")
        _, a_new = _seg_gather(act, act_off[clean], lens)
        _, a_old = _seg_gather(ob.act, ob.act_off[pos], lens)
        if not np.array_equal(a_new, a_old):
            raise RuntimeError("clean box changed its active set")
        bt.take(clean, ob, pos)
        bt.clean_old = (L, pos)                # the incremental sweep copies their stored rows
    return bt


def _drain(ctx: "_Ctx"):
    """Before an aborted engine run's context is dropped: the augmentation
    sweeps already issued on the aug stream still write UH / PsiV / UH_div /
    schur (allocated on the level stream), so both the level stream (where the
    restarted run allocates) and the current stream wait for them."""
    pipe = getattr(ctx, "pipe", None)
    if pipe is not None and pipe.q:
        ctx.sstream.wait_stream(pipe.stream)
    torch.cuda.current_stream().wait_stream(ctx.sstream)


def _remap_old_levels(fct: "Factorization", old_to_new, dpn: int) -> dict:
    """Level views of the previous factorization in the NEW DOF numbering
    (reference BoxFactors.remapped, skel.py:82-85, with the dof_map of
    skel.py:493-498): index arrays are remapped copies, matrices are shared.
    Boxes that held deleted nodes carry -1 entries; the ownership rule makes
    them dirty, so they are never reused."""
    import copy
    o2n = np.asarray(old_to_new, np.int64)
    dof_map = np.full(dpn * len(o2n), -1, np.int64)
    valid = np.flatnonzero(o2n >= 0)
    for c in range(dpn):
        dof_map[dpn * valid + c] = dpn * o2n[valid] + c
    out = {}
    for L in fct.levels:
        L.batch.resolve()
        L2, bt2 = copy.copy(L), copy.copy(L.batch)
        bt2.act = dof_map[np.asarray(L.batch.act, np.int64)]
        L2.batch = bt2
        L2.__dict__.pop("_row", None)
        L2.__dict__.pop("_row_keep", None)
        _level_code(L2)
        out[L.lev] = L2
    return out


def _levels_and_top(make_ctx, upd=None, reuse=None, dirty=None):
    """Level loop and _finish_top: the native engine + driver first; a migration
    (R -> S, skel.py:317-330) or a clean box without a twin aborts that run and
    the Python level loop redoes everything on a fresh context."""
    attempts = (True, False) if (_ENGINE_ON and not _Prof.enabled) else (False,)
    prev = None
    for fast in attempts:
        if prev is not None:
            _drain(prev)
        with _ht("ctx"):
            ctx = make_ctx()
        prev = ctx
        levels = nh = None
        try:
            with _ht("run_levels"):
                if fast and _NATIVE_ON:
                    store, nh = _run_levels_native(ctx, upd=upd)
                elif fast and upd is not None:
                    levels, store, _ = _run_levels_engine_update(ctx, reuse, dirty)
                elif fast:
                    levels, store, _ = _run_levels_engine(ctx)
                else:
                    levels, store, _ = _run_levels(ctx, reuse=reuse, dirty=dirty)
            got = []
            collect = (lambda: got.append(_native_collect(ctx, nh))) if nh is not None else None
            try:
                with _ht("finish_top"):
                    top = _finish_top(ctx, levels, store, ctx.pipe, before_sync=collect)
            finally:
                if nh is not None and not got and nh[1].value:
                    nh[0].skb_drv_free(nh[1].value)     # (collect frees it otherwise)
                    nh[1].value = 0
            if nh is not None:
                levels = got[0]
            return ctx, levels, top
        except _EngineAbort:
            if not fast:
                raise
    raise RuntimeError("unreachable")


def factor(spec, b, t: Tree, tol: float, workers: int = 1,
           proxy_count: int = DEFAULT_PROXY_COUNT, proxy_factor: float = DEFAULT_PROXY_FACTOR,
           propagate_zeros: bool = False) -> Factorization:
    """Build the skeletonization factorization on the GPU (reference skel.py:428-453).

    ``workers`` is accepted for signature parity (the GPU batches every box of a
    level).  ``propagate_zeros=True`` is the reference's sequential validation
    mode (one box per launch, far fields thinned by the zeros of the boxes
    compressed before; skel.py:267-270): slow by design.
    """
    torch.cuda.synchronize()
    _DevSlab.flush()
    t0 = time.perf_counter()
    with torch.cuda.stream(_compress_stream()):
        if propagate_zeros:
            ctx = _Ctx(spec, b, t, tol, proxy_count, proxy_factor)
            levels, store, _ = _run_levels_pz(ctx)
            rd, E_root, top, ipiv, UH, PsiV, UH_div, q, ratio = _finish_top(ctx, levels, store, ctx.pipe)
        else:
            ctx, levels, (rd, E_root, top, ipiv, UH, PsiV, UH_div, q, ratio) = _levels_and_top(
                lambda: _Ctx(spec, b, t, tol, proxy_count, proxy_factor))
    with _ht("final_sync"):
        torch.cuda.synchronize()
    stats = {"k_per_level": {L.lev: int(L.k.max(initial=0)) for L in levels},
             "root_size": len(rd), "top_pivot_ratio": ratio}
    fct = Factorization(spec, b, t, tol, proxy_count, proxy_factor, levels, rd, E_root, top, ipiv,
                        UH, PsiV, UH_div, q, ctx, stats)
    fct.stats["factor_time"] = time.perf_counter() - t0
    fct.stats["n_dofs"] = fct.n_dofs
    return fct


def update(fct: Factorization, b_new, report, workers: int = 1) -> Factorization:
    """Refactor only what a local perturbation invalidated (reference skel.py:456-514)."""
    with _ht("U.sync"):
        torch.cuda.synchronize()
        _DevSlab.flush()
    t0 = time.perf_counter()
    try:
        with _ht("U.refit"):
            t_new = refit_tree(fct.tree, b_new.positions)
    except ValueError as e:
        raise RootBoxExceededError("perturbed node escaped the root box; refactor with a fresh tree") from e
    with _ht("U.dirty"):
        dmask = dirty_mask(fct.tree, t_new, b_new, report, fct.proxy_factor)
    o2n = np.asarray(report.old_to_new, np.int64)
    same_dofs = len(o2n) == b_new.n_nodes and np.array_equal(o2n, np.arange(len(o2n)))
    if same_dofs:
        old = {L.lev: L for L in fct.levels}
    else:
        # AddHole / DeleteHole (reference skel.py:493-498): clean boxes are reused
        # with remapped DOF lists; the augmentation block changes its size, so the
        # sweep is the full one
        with _ht("U.remap"):
            old = _remap_old_levels(fct, o2n, fct.spec.dof_per_node)

    def make_ctx():
        ctx = _Ctx(fct.spec, b_new, t_new, fct.tol, fct.proxy_count, fct.proxy_factor)
        ctx.upd_old = (fct, dmask)
        ctx.upd_inc = same_dofs
        ctx.g                                           # geometry upload
        torch.cuda.current_stream().synchronize()
        return ctx

    with torch.cuda.stream(_compress_stream()):
        ctx, levels, (rd, E_root, top, ipiv, UH, PsiV, UH_div, q, ratio) = _levels_and_top(
            make_ctx, upd=(fct, dmask, old), reuse=old, dirty=dmask)
    with _ht("U.final"):
        torch.cuda.synchronize()
    ctx.upd_old = None                                  # no chain of old factorizations
    ctx.pipe = None
    for L in levels:
        L.batch.__dict__.pop("clean_old", None)
    stats = {"k_per_level": {L.lev: int(L.k.max(initial=0)) for L in levels},
             "root_size": len(rd), "top_pivot_ratio": ratio}
    nf = Factorization(fct.spec, b_new, t_new, fct.tol, fct.proxy_count, fct.proxy_factor, levels,
                       rd, E_root, top, ipiv, UH, PsiV, UH_div, q, ctx, stats)
    nf.stats["update_time"] = time.perf_counter() - t0
    nf.stats["n_dirty"] = int(dmask.sum())
    nf.stats["n_boxes"] = len(t_new.lev)
    nf.stats["dirty"] = {t_new.key(i) for i in np.flatnonzero(dmask)}
    return nf


def system_matvec(spec, b, x):
    """Exact augmented system product on the GPU (reference kernels.system_matvec,
    kernels.py:393-414), direct O(N^2) summation; x: (dim,) or (dim, nrhs)."""
    is_t = isinstance(x, torch.Tensor)
    xa = x if is_t else np.asarray(x, float)
    nd, q = spec.dof_per_node * b.n_nodes, 3 * b.n_holes if spec.augmented(b) else 0
    if xa.shape[0] != nd + q:
        raise ValueError("dimension mismatch")
    dev = _dev()
    X = (xa.to(device=dev, dtype=torch.float64) if is_t
         else torch.from_numpy(np.ascontiguousarray(xa)).to(dev)).reshape(nd + q, -1).contiguous()
    g = getattr(b, "_skb_device", None) or DeviceBoundary(b)
    Y = torch.empty_like(X)
    if spec.pde == LAPLACE:
        call("skb_system_matvec_lap", g.pos, g.nrm, g.w, g.kap, b.n_nodes, X, X.shape[1], Y, _stream())
    else:
        up = _upload(hc=np.ascontiguousarray(b.hole_centers, np.float64).reshape(-1)
                     if b.n_holes else np.zeros(2),
                     co=np.ascontiguousarray(b.offsets, np.int64))
        call("skb_system_matvec", g.pos, g.nrm, g.w, g.kap, b.n_nodes, up["hc"], q // 3, up["co"], X,
             X.shape[1], Y, _stream())
    if is_t:
        return Y.reshape(x.shape)
    out = Y.cpu().numpy()
    return out.reshape(np.asarray(x).shape)


def point_in_domain(b, points) -> np.ndarray:
    """True where a point lies strictly inside the fluid domain (reference
    Boundary.point_in_domain, geometry.py:179-192): winding number of every
    curve's node polyline (inside the outer curve, outside each hole) and
    nearest node farther than 1e-12 -- one warp per point on the GPU."""
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(points, float)), np.float64)
    m = len(pts)
    if m == 0:
        return np.zeros(0, bool)
    g = getattr(b, "_skb_device", None) or DeviceBoundary(b)
    up = _upload(co=np.ascontiguousarray(b.offsets, np.int64), tg=pts.reshape(-1))
    out = torch.empty(m, dtype=torch.uint8, device=_dev())
    call("skb_point_in_domain", g.pos, up["co"], len(b.offsets) - 1, up["tg"], m, out, _stream())
    return out.cpu().numpy().astype(bool)


def evaluate_interior(spec, b, solution, targets, chunk: int = 256):
    """Field at interior targets from a solve() output (reference
    evaluate_interior, skel.py:537-564) by direct summation on the GPU:
    Stokes u = D mu + H lam (eval_forward_block kernels.py:171-198 + the
    Stokeslet/rotlet columns kernels.py:201-223), shape (m, 2); Laplace
    u = -S mu (kernels.py:193-194), shape (m,).  A (dim, nrhs) solution gives
    (m, 2, nrhs) / (m, nrhs).  Exterior targets are rejected.  ``chunk`` is
    accepted for signature parity (all targets run in one launch)."""
    tg = np.ascontiguousarray(np.atleast_2d(np.asarray(targets, float)), np.float64)
    if not np.all(point_in_domain(b, tg)):
        raise ValueError("targets must lie strictly inside the domain")
    is_t = isinstance(solution, torch.Tensor)
    sol = solution if is_t else np.asarray(solution, float)
    dpn = spec.dof_per_node
    nd, q = dpn * b.n_nodes, 3 * b.n_holes if spec.augmented(b) else 0
    if sol.shape[0] != nd + q:
        raise ValueError("dimension mismatch")
    vec = sol.ndim == 1
    dev = _dev()
    X = (sol.to(device=dev, dtype=torch.float64) if is_t
         else torch.from_numpy(np.ascontiguousarray(sol)).to(dev)).reshape(nd + q, -1).contiguous()
    nr = X.shape[1]
    g = getattr(b, "_skb_device", None) or DeviceBoundary(b)
    m = len(tg)
    Y = torch.empty((dpn * m, nr), dtype=torch.float64, device=dev)
    if spec.pde == LAPLACE:
        up = _upload(tg=tg.reshape(-1))
        call("skb_eval_interior_lap", g.pos, g.w, b.n_nodes, X, nr, up["tg"], m, Y, _stream())
        Y = Y[:, 0] if vec else Y
    else:
        up = _upload(hc=np.ascontiguousarray(b.hole_centers, np.float64).reshape(-1)
                     if b.n_holes else np.zeros(2), tg=tg.reshape(-1))
        call("skb_eval_interior", g.pos, g.nrm, g.w, b.n_nodes, up["hc"], q // 3, X, nr, up["tg"], m, Y,
             _stream())
        Y = Y.reshape(m, 2, nr)
        if vec:
            Y = Y[:, :, 0]
    return Y if is_t else Y.cpu().numpy()

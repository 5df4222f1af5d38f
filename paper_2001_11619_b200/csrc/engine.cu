// Native level engine: the critical-path compression chain of factor()
// (reference skel.py:443-449 driving compress_box skel.py:293-316) runs on a
// host thread of its own, level by level from the leaves up:
//
//   assign_internal_actives (skel.py:251-256) -> far_dofs (skel.py:258-280)
//   -> proxy rings (kernels.py:263-273) -> ID stacks (skb_assemble_stack)
//   -> Householder pre-reduction -> QRCP -> ONE device->host copy of
//   (perm, k, steps, gap) -> skeletons (skel = act[perm[:k]]) -> next level.
//
// The Python side consumes finished levels (skb_engine_wait) and enqueues the
// Schur stage and the augmentation sweep on its own streams while the engine
// already compresses the next level, so Python bookkeeping is off the
// critical path.  Same host functions and kernels as the Python launch path:
// identical results.  The active/skeleton store arrays are the caller's
// (ActStore numpy buffers); the engine appends to them.

#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace skb {
void use_engine_ring(bool on);
int geqrf_batched(int64_t nbox, const int64_t* m, const int64_t* n, const int64_t* lda,
                  const int64_t* A, cudaStream_t s);
int qrcp_batched(int64_t nbox, const int64_t* m, const int64_t* n, const int64_t* lda,
                 const int64_t* A, const int64_t* kmin, double tol, const int64_t* perm_off,
                 int32_t* perm, double* diag, int32_t* k_out, int32_t* steps_out,
                 double* min_gap, cudaStream_t s);
}  // namespace skb

using namespace skb;

namespace {

struct LevelOut {
  int rc = 0;
  bool ready = false;
  int64_t B = 0, na = 0, box0 = 0;
  std::vector<int64_t> act_off, act, rows, A, mq;
  std::vector<int32_t> perm, k, steps;
  std::vector<double> gap;
  double* stack = nullptr;
  char* dbuf = nullptr;          // diag | gap | perm, k, steps (device)
  int64_t* dup = nullptr;        // uploaded descriptors (device): act_off | act | ...
  int64_t o_int = 0;             // byte offset of perm in dbuf
  int64_t o_act = 0;             // element offset of act in dup
  int64_t h2d = 0, d2h = 0;      // bytes moved host<->device for this level
  std::vector<int64_t> idx;      // boxes compressed (all of the level, or the dirty ones)
  cudaEvent_t ev = nullptr;
};

struct Engine {
  // tree (tree.py layout)
  const double *center, *hw;
  const int64_t *nbr, *lev, *ix, *iy, *children, *level_start;
  const uint8_t* leaf;
  int64_t depth;
  double root[3], factor;
  // store (ActStore buffers)
  int64_t *big, *a_start, *a_len, *s_start, *s_len, *fill;
  int64_t cap;
  // geometry
  const double *px, *py, *pos, *nrm, *w, *cs;
  int64_t P;
  double tol;
  int32_t pde = 0;               // 0 Stokes (2 DOFs per node), 1 Laplace (1)
  cudaStream_t s;
  int dev;
  int64_t lev_lo;
  std::vector<LevelOut> out;     // indexed by level
  std::mutex m;
  std::condition_variable cv;
  std::atomic<bool> stop{false};
  int64_t acked = 1 << 30;       // lowest level whose Schur stage the caller has enqueued
  int64_t lead = -1;             // >= 0: run at most `lead` levels ahead of the caller
  std::thread th;
  char* pinned = nullptr;
  size_t pinned_size = 0;
  bool* shared_pinned = nullptr;   // set: the pinned buffer is the shared one
  int64_t* pack = nullptr;         // pinned staging of the per-level upload
  int64_t pack_cap = 0;
  bool shared_pack = false;        // set: pack is the process-wide buffer (g_pack)
  bool freeing = false;
  // update mode: boxes to recompress (uint8 per box) and the clean boxes'
  // skeletons (CSR over boxes); nullptr = factor every box
  const uint8_t* todo = nullptr;
  const int64_t* clean_off = nullptr;
  const int64_t* clean_skel = nullptr;
};

// Process-wide pinned staging buffer for the per-level upload (kept across
// factorizations; one engine at a time, the others stage their own).
struct PackBuf {
  int64_t* p = nullptr;
  int64_t cap = 0;
  bool busy = false;
};
PackBuf& g_pack() {
  static PackBuf b;
  return b;
}

// Grow the engine's pinned staging buffer to n int64 (keeps the contents; the
// previous level's copy out of it has completed: run_level waits on its event).
int pack_reserve(Engine& E, int64_t n) {
  if (n <= E.pack_cap) return 0;
  const int64_t want = std::max<int64_t>(n + n / 4, (int64_t)1 << 20);
  int64_t* np = nullptr;
  SKB_RET(cudaHostAlloc((void**)&np, sizeof(int64_t) * want, cudaHostAllocDefault));
  if (E.pack) {
    memcpy(np, E.pack, sizeof(int64_t) * E.pack_cap);
    cudaFreeHost(E.pack);
  }
  E.pack = np;
  E.pack_cap = want;
  if (E.shared_pack) {
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    g_pack().p = np;
    g_pack().cap = want;
  }
  return 0;
}

// Host worker pool for the per-box bookkeeping of a level (far-field lists,
// proxy rings): one process-wide pool, used by one engine at a time.
struct Pool {
  int W = 1;
  std::vector<std::thread> th;
  std::mutex m, busy;
  std::condition_variable cv, cv_done;
  const std::function<void(int)>* job = nullptr;
  int64_t gen = 0;
  int pending = 0;
  explicit Pool(int w) : W(w < 1 ? 1 : w) {
    for (int i = 1; i < W; ++i)
      th.emplace_back([this, i] {
        int64_t seen = 0;
        for (;;) {
          const std::function<void(int)>* f;
          {
            std::unique_lock<std::mutex> lk(m);
            cv.wait(lk, [&] { return gen != seen; });
            seen = gen;
            f = job;
          }
          (*f)(i);
          std::lock_guard<std::mutex> lk(m);
          if (--pending == 0) cv_done.notify_one();
        }
      });
    for (auto& t : th) t.detach();   // process-lifetime workers
  }
  // f(part) for part in [0, W); the caller runs part 0
  void run(const std::function<void(int)>& f) {
    if (W <= 1) { f(0); return; }
    std::lock_guard<std::mutex> use(busy);
    {
      std::lock_guard<std::mutex> lk(m);
      job = &f;
      pending = W - 1;
      ++gen;
    }
    cv.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(m);
    cv_done.wait(lk, [&] { return pending == 0; });
  }
};

Pool& host_pool() {
  static Pool* p = [] {
    int w = 8;
    if (const char* e = getenv("SKB_ENGINE_THREADS")) w = atoi(e);
    const int hc = (int)std::thread::hardware_concurrency();
    if (hc > 0) w = std::min(w, std::max(1, hc / 2));
    return new Pool(w);
  }();
  return *p;
}

int64_t append(Engine& E, const int64_t* a, int64_t n) {
  const int64_t o = *E.fill;
  if (o + n > E.cap) return -1;
  if (n) memcpy(E.big + o, a, sizeof(int64_t) * n);
  *E.fill = o + n;
  return o;
}

struct ETimer {
  static bool on() {
    static const bool v = getenv("SKB_ENGINE_TIMING") != nullptr;
    return v;
  }
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  char buf[512];
  int n = 0;
  void tick(const char* name) {
    if (!on()) return;
    const auto t = std::chrono::steady_clock::now();
    n += snprintf(buf + n, sizeof(buf) - n, " %s %.0f", name,
                  std::chrono::duration<double, std::micro>(t - t0).count());
    t0 = t;
  }
};

// Debug snapshots (SKB_ENGINE_SNAP=<level>): device copies of that level's
// ID stacks after assembly, after the Householder pre-reduction and after the
// QRCP, read back with skb_debug_snap (race localisation; off by default).
struct Snap {
  double* buf[3] = {nullptr, nullptr, nullptr};
  int64_t cap = 0, n = 0;
};
Snap& g_snap() {
  static Snap s;
  return s;
}
int64_t snap_level() {
  static const int64_t v = getenv("SKB_ENGINE_SNAP") ? atoll(getenv("SKB_ENGINE_SNAP")) : -1;
  return v;
}
int snap_copy(int which, const double* src, int64_t n, cudaStream_t s) {
  Snap& S = g_snap();
  if (n > S.cap) {
    SKB_RET(cudaStreamSynchronize(s));
    for (auto& b : S.buf) {
      if (b) cudaFree(b);
      b = nullptr;
    }
    for (auto& b : S.buf) SKB_RET(cudaMalloc((void**)&b, sizeof(double) * n));
    S.cap = n;
  }
  S.n = n;
  SKB_RET(cudaMemcpyAsync(S.buf[which], src, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int run_level(Engine& E, int64_t L, LevelOut& R) {
  ETimer tm;
  const int64_t b0 = E.level_start[L], nall = E.level_start[L + 1] - b0;
  R.box0 = b0;
  // boxes to compress: all of the level (factor) or the dirty ones (update)
  std::vector<int64_t> idx;
  for (int64_t b = 0; b < nall; ++b)
    if (!E.todo || E.todo[b0 + b]) idx.push_back(b0 + b);
  const int64_t B = (int64_t)idx.size();
  R.B = B;
  R.idx = idx;
  // assign_internal_actives (every box of the level: clean colleagues feed the
  // dirty boxes' far fields): active = concat of the children's skeletons
  {
    std::vector<int64_t> tmp;
    for (int64_t i = b0; i < b0 + nall; ++i) {
      if (E.leaf[i]) continue;
      tmp.clear();
      for (int q = 0; q < 4; ++q) {
        const int64_t c = E.children[4 * i + q];
        if (c < 0) continue;
        tmp.insert(tmp.end(), E.big + E.s_start[c], E.big + E.s_start[c] + E.s_len[c]);
      }
      const int64_t o = append(E, tmp.data(), (int64_t)tmp.size());
      if (o < 0) return 7;
      E.a_start[i] = o;
      E.a_len[i] = (int64_t)tmp.size();
    }
  }
  tm.tick("internal");
  // clean boxes (update): skeletons carried over from the previous factorization
  if (E.todo)
    for (int64_t i = b0; i < b0 + nall; ++i) {
      if (E.todo[i]) continue;
      const int64_t n0 = E.clean_off[i], nk = E.clean_off[i + 1] - n0;
      const int64_t o = append(E, E.clean_skel + n0, nk);
      if (o < 0) return 7;
      E.s_start[i] = o;
      E.s_len[i] = nk;
    }
  if (B == 0) return 0;
  R.act_off.assign(B + 1, 0);
  for (int64_t b = 0; b < B; ++b) R.act_off[b + 1] = R.act_off[b] + E.a_len[idx[b]];
  R.na = R.act_off[B];
  R.act.resize(std::max<int64_t>(R.na, 1));
  for (int64_t b = 0; b < B; ++b)
    memcpy(R.act.data() + R.act_off[b], E.big + E.a_start[idx[b]], sizeof(int64_t) * E.a_len[idx[b]]);
  // One pinned upload, packed in place (int64 units, 16-byte aligned segments):
  //   act_off | act | pts | pn | pw | stack_off | far_off | far
  // The proxy rings are written straight into it by the host pool; the far
  // lists (sizes unknown up front) are copied in by a second pool pass.
  const int64_t P = E.P;
  auto al = [](int64_t o) { return (o + 1) & ~(int64_t)1; };
  const int64_t o_ao = 0;
  R.o_act = al(o_ao + B + 1);
  const int64_t o_pt = al(R.o_act + (int64_t)R.act.size());
  const int64_t o_pn = al(o_pt + B * P * 2);
  const int64_t o_pw = al(o_pn + B * P * 2);
  const int64_t o_so = al(o_pw + B);
  const int64_t o_fo = al(o_so + B);
  const int64_t o_f = al(o_fo + B + 1);
  int rc = 0;
  if ((rc = pack_reserve(E, o_f + 4096))) return rc;
  int64_t* pk = E.pack;
  memcpy(pk + o_ao, R.act_off.data(), sizeof(int64_t) * (B + 1));
  memcpy(pk + R.o_act, R.act.data(), sizeof(int64_t) * R.act.size());
  // far-field DOF lists and proxy rings (native host runtime), boxes split
  // over the host pool in contiguous parts, concatenated in box order
  Pool& pool = host_pool();
  const int parts = B >= 16 ? (int)std::min<int64_t>(pool.W, B / 8) : 1;
  std::vector<std::vector<int64_t>> pfar(parts), poff(parts);
  std::vector<int> prc(parts, 0);
  {
    double* pts = reinterpret_cast<double*>(pk + o_pt);
    double* pn = reinterpret_cast<double*>(pk + o_pn);
    double* pw = reinterpret_cast<double*>(pk + o_pw);
    const std::function<void(int)> work = [&](int p) {
      if (p >= parts) return;
      const int64_t lo = B * p / parts, hi = B * (p + 1) / parts, nb = hi - lo;
      poff[p].resize(nb + 1);
      pfar[p].resize(4096);
      int64_t need = 0;
      const int32_t shift = E.pde == 1 ? 0 : 1;
      int r = skb_host_far_lists(nb, idx.data() + lo, E.center, E.hw, E.nbr, E.lev, E.ix, E.iy, E.leaf,
                                 E.level_start, E.depth, E.root, E.factor, E.big, E.a_start, E.a_len,
                                 E.px, E.py, poff[p].data(), pfar[p].data(), (int64_t)pfar[p].size(), &need,
                                 shift);
      if (r == 1) {
        pfar[p].resize(need + 1);
        r = skb_host_far_lists(nb, idx.data() + lo, E.center, E.hw, E.nbr, E.lev, E.ix, E.iy, E.leaf,
                               E.level_start, E.depth, E.root, E.factor, E.big, E.a_start, E.a_len,
                               E.px, E.py, poff[p].data(), pfar[p].data(), (int64_t)pfar[p].size(), &need,
                               shift);
      }
      prc[p] = r;
      skb_host_proxies(nb, idx.data() + lo, E.center, E.hw, E.factor, P, E.cs, pts + lo * P * 2,
                       pn + lo * P * 2, pw + lo);
    };
    if (parts > 1) pool.run(work);
    else work(0);
  }
  std::vector<int64_t> far_off(B + 1, 0), part_o(parts + 1, 0);
  for (int p = 0; p < parts; ++p) {
    if (prc[p]) return 8;
    const int64_t lo = B * p / parts, nb = (int64_t)poff[p].size() - 1;
    for (int64_t b = 0; b < nb; ++b) far_off[lo + b + 1] = part_o[p] + poff[p][b + 1];
    part_o[p + 1] = part_o[p] + poff[p][nb];
  }
  const int64_t nfar = std::max<int64_t>(far_off[B], 1);
  if ((rc = pack_reserve(E, o_f + nfar))) return rc;
  pk = E.pack;
  {
    const std::function<void(int)> cp = [&](int p) {
      if (p < parts && part_o[p + 1] > part_o[p])
        memcpy(pk + o_f + part_o[p], pfar[p].data(), sizeof(int64_t) * (part_o[p + 1] - part_o[p]));
    };
    if (parts > 1) pool.run(cp);
    else cp(0);
  }
  memcpy(pk + o_fo, far_off.data(), sizeof(int64_t) * (B + 1));
  tm.tick("far+proxies");
  // stack layout (column-major per box, ld = rows)
  R.rows.resize(B);
  std::vector<int64_t> nB(B);
  int64_t* stack_off = pk + o_so;
  int64_t maxnB = 0, maxitems = 0, so = 0;
  for (int64_t b = 0; b < B; ++b) {
    nB[b] = R.act_off[b + 1] - R.act_off[b];
    const int64_t nF = far_off[b + 1] - far_off[b];
    R.rows[b] = E.pde == 1 ? 2 * nF + 2 * P + 2 : 2 * nF + 6 * P + 2;   // skel.py:306-314
    stack_off[b] = so;
    so += R.rows[b] * nB[b];
    maxnB = std::max(maxnB, nB[b]);
    maxitems = std::max(maxitems, nF + P + 1);
  }
  cudaStream_t s = E.s;
  SKB_RET(malloc_async((void**)&R.stack, sizeof(double) * std::max<int64_t>(so, 1), s));
  const int64_t npk = o_f + nfar;
  tm.tick("pack");
  SKB_RET(malloc_async((void**)&R.dup, sizeof(int64_t) * npk, s));
  SKB_RET(cudaMemcpyAsync(R.dup, pk, sizeof(int64_t) * npk, cudaMemcpyHostToDevice, s));
  tm.tick("upload");
  R.h2d += 8 * npk;
  if ((rc = (E.pde == 1 ? skb_assemble_stack_lap : skb_assemble_stack)(
           E.pos, E.nrm, E.w, B, R.dup + o_ao, R.dup + R.o_act, R.dup + o_fo,
                               R.dup + o_f, (const double*)(R.dup + o_pt),
                               (const double*)(R.dup + o_pn), (const double*)(R.dup + o_pw),
                               (int32_t)P, R.dup + o_so, R.stack, maxnB, maxitems, s)))
    return rc;
  if (snap_level() == L && (rc = snap_copy(0, R.stack, so, s))) return rc;
  tm.tick("asm");
  // Householder pre-reduction of the tall stacks (dense.py:56-59)
  R.A.resize(B);
  R.mq.resize(B);
  std::vector<int64_t> pm, pn_, pA;
  for (int64_t b = 0; b < B; ++b) {
    R.A[b] = (int64_t)(R.stack + stack_off[b]);
    const bool pre = R.rows[b] > 2 * nB[b];     // dense.py:56 branch
    R.mq[b] = pre ? nB[b] : R.rows[b];
    if (pre) { pm.push_back(R.rows[b]); pn_.push_back(nB[b]); pA.push_back(R.A[b]); }
  }
  if (!pm.empty() && (rc = geqrf_batched((int64_t)pm.size(), pm.data(), pn_.data(), pm.data(),
                                         pA.data(), s)))
    return rc;
  if (snap_level() == L && (rc = snap_copy(1, R.stack, so, s))) return rc;
  tm.tick("geqrf");
  // QRCP with rank at tol (dense.py:60-68)
  const int64_t na = R.na;
  const int64_t o_gap = 8 * std::max<int64_t>(na, 1);
  R.o_int = o_gap + 8 * std::max<int64_t>(B, 1);
  const int64_t nint = na + 2 * B + 1;
  const int64_t dbytes = R.o_int + 4 * nint;
  SKB_RET(malloc_async((void**)&R.dbuf, dbytes, s));
  std::vector<int64_t> kmin(B, 0);
  int32_t* ints = (int32_t*)(R.dbuf + R.o_int);
  if ((rc = qrcp_batched(B, R.mq.data(), nB.data(), R.rows.data(), R.A.data(), kmin.data(), E.tol,
                         R.act_off.data(), ints, (double*)R.dbuf, ints + na, ints + na + B,
                         (double*)(R.dbuf + o_gap), s)))
    return rc;
  if (snap_level() == L && (rc = snap_copy(2, R.stack, so, s))) return rc;
  // one device->host copy: gap | perm | k | steps
  const size_t hb = (size_t)(dbytes - o_gap);
  if (hb > E.pinned_size) return 9;
  SKB_RET(cudaMemcpyAsync(E.pinned, R.dbuf + o_gap, hb, cudaMemcpyDeviceToHost, s));
  R.d2h += (int64_t)hb;
  SKB_RET(cudaEventRecord(R.ev, s));
  tm.tick("qrcp");
  SKB_RET(cudaEventSynchronize(R.ev));
  tm.tick("WAIT");
  const double* gap = (const double*)E.pinned;
  const int32_t* ih = (const int32_t*)(E.pinned + (R.o_int - o_gap));
  R.gap.assign(gap, gap + B);
  R.perm.assign(ih, ih + na);
  R.k.assign(ih + na, ih + na + B);
  R.steps.assign(ih + na + B, ih + na + 2 * B);
  // skeletons: skel = act[perm[:k]] (assign_internal_actives of the next level reads them)
  for (int64_t b = 0; b < B; ++b) {
    const int64_t i = idx[b], a0 = R.act_off[b], kk = R.k[b];
    std::vector<int64_t> sk(kk);
    for (int64_t j = 0; j < kk; ++j) sk[j] = R.act[a0 + R.perm[a0 + j]];
    const int64_t o = append(E, sk.data(), kk);
    if (o < 0) return 7;
    E.s_start[i] = o;
    E.s_len[i] = kk;
  }
  tm.tick("skel");
  if (ETimer::on()) fprintf(stderr, "engine level %lld (%lld boxes):%s us\n", (long long)L, (long long)B, tm.buf);
  return 0;
}

void engine_main(Engine* E) {
  cudaSetDevice(E->dev);
  use_engine_side(true);
  use_engine_ring(true);          // descriptor uploads through the engine's own pinned ring
  if (!getenv("SKB_ENGINE_SHARED_POOL")) {
    static cudaMemPool_t pool = nullptr;
    static std::mutex pm;
    std::lock_guard<std::mutex> lk(pm);
    if (!pool) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = E->dev;
      if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        if (getenv("SKB_POOL_STRICT")) pool_strict(pool);   // debug, see ring_stage
      } else {
        pool = nullptr;
      }
    }
    skb::tl_pool() = pool;
  }
  for (int64_t L = E->depth; L >= E->lev_lo; --L) {
    LevelOut& R = E->out[L];
    if (E->lead >= 0) {
      std::unique_lock<std::mutex> lk(E->m);
      E->cv.wait(lk, [&] { return E->stop.load() || E->acked <= L + 1 + E->lead || L + 1 + E->lead > E->depth; });
    }
    int rc = 0;
    if (E->stop.load()) rc = -1000;
    else rc = run_level(*E, L, R);
    {
      std::lock_guard<std::mutex> lk(E->m);
      R.rc = rc;
      R.ready = true;
      // a level without boxes to compress has no Schur stage: nothing will
      // ever acknowledge it, so it counts as acknowledged now (an update whose
      // deepest dirty level is shallow would otherwise stall the run-ahead)
      if (rc == 0 && R.B == 0 && L < E->acked) E->acked = L;
    }
    E->cv.notify_all();
    if (rc) {
      // later levels cannot run: mark them failed
      std::lock_guard<std::mutex> lk(E->m);
      for (int64_t L2 = L - 1; L2 >= E->lev_lo; --L2) {
        E->out[L2].rc = -1000;
        E->out[L2].ready = true;
      }
      E->cv.notify_all();
      return;
    }
  }
}

}  // namespace

extern "C" {

// arrays: {center, hw, nbr, lev, ix, iy, children, level_start, leaf(uint8)} (tree.py layout);
// store: {big, a_start, a_len, s_start, s_len, fill}; geo: {px, py, pos, nrm, w, cs} (pos/nrm/w device)
int skb_engine_start(const void* const* tree, int64_t depth, const double* root, double factor,
                     int64_t* const* store, int64_t cap, const double* const* geo, int64_t P,
                     double tol, void* stream, int64_t lev_lo, int64_t max_level_ints,
                     int32_t pde, int64_t* handle) {
  Engine* E = new Engine();
  E->pde = pde;
  E->center = (const double*)tree[0];
  E->hw = (const double*)tree[1];
  E->nbr = (const int64_t*)tree[2];
  E->lev = (const int64_t*)tree[3];
  E->ix = (const int64_t*)tree[4];
  E->iy = (const int64_t*)tree[5];
  E->children = (const int64_t*)tree[6];
  E->level_start = (const int64_t*)tree[7];
  E->leaf = (const uint8_t*)tree[8];
  E->depth = depth;
  memcpy(E->root, root, sizeof(E->root));
  E->factor = factor;
  E->big = store[0]; E->a_start = store[1]; E->a_len = store[2];
  E->s_start = store[3]; E->s_len = store[4]; E->fill = store[5];
  E->cap = cap;
  E->px = geo[0]; E->py = geo[1]; E->pos = geo[2]; E->nrm = geo[3]; E->w = geo[4]; E->cs = geo[5];
  E->P = P;
  E->tol = tol;
  E->s = (cudaStream_t)stream;
  const bool deferred = lev_lo <= 0;     // started later by skb_engine_go
  E->lev_lo = deferred ? 1 : lev_lo;
  cudaGetDevice(&E->dev);
  E->out.resize(depth + 1);
  for (int64_t L = E->lev_lo; L <= depth; ++L)
    SKB_RET(cudaEventCreateWithFlags(&E->out[L].ev, cudaEventDisableTiming));
  // pinned landing buffer for the per-level device->host copy: kept across
  // factorizations (cudaHostAlloc / cudaFreeHost would synchronise the device)
  {
    static char* g_pinned = nullptr;
    static size_t g_size = 0;
    static bool g_busy = false;
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    const size_t want = (size_t)(8 * max_level_ints + 1024);
    if (!g_busy) {
      if (g_size < want) {
        if (g_pinned) cudaFreeHost(g_pinned);
        SKB_RET(cudaHostAlloc((void**)&g_pinned, want, cudaHostAllocDefault));
        g_size = want;
      }
      g_busy = true;
      E->pinned = g_pinned;
      E->pinned_size = g_size;
      E->shared_pinned = &g_busy;
    } else {
      SKB_RET(cudaHostAlloc((void**)&E->pinned, want, cudaHostAllocDefault));
      E->pinned_size = want;
    }
  }
  {
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    PackBuf& g = g_pack();
    if (!g.busy) {
      g.busy = true;
      E->shared_pack = true;
      E->pack = g.p;
      E->pack_cap = g.cap;
    }
  }
  if (!deferred) E->th = std::thread(engine_main, E);
  *handle = (int64_t)E;
  return 0;
}

int skb_engine_go(int64_t handle) {
  Engine* E = (Engine*)handle;
  if (!E->th.joinable()) E->th = std::thread(engine_main, E);
  return 0;
}

// Update mode: compress only the boxes with todo[i] != 0; clean boxes take
// their skeleton from clean_off/clean_skel (CSR over all boxes).  Call right
// after skb_engine_start with lev_lo = depth + 1 (engine idle), then
// skb_engine_go to run.
int skb_engine_set_update(int64_t handle, const uint8_t* todo, const int64_t* clean_off,
                          const int64_t* clean_skel) {
  Engine* E = (Engine*)handle;
  E->todo = todo;
  E->clean_off = clean_off;
  E->clean_skel = clean_skel;
  return 0;
}

// Block until level L is compressed; sizes = {rc, B, na, box0, o_int, o_act, h2d, d2h}; ptrs =
// {act_off, act, rows, A, mq, perm(i32), k(i32), steps(i32), gap(f64), stack, dbuf, dup, event}
int skb_engine_wait(int64_t handle, int64_t L, int64_t* sizes, int64_t* ptrs) {
  Engine* E = (Engine*)handle;
  LevelOut& R = E->out[L];
  {
    std::unique_lock<std::mutex> lk(E->m);
    E->cv.wait(lk, [&] { return R.ready; });
  }
  sizes[0] = R.rc; sizes[1] = R.B; sizes[2] = R.na; sizes[3] = R.box0; sizes[4] = R.o_int;
  sizes[5] = R.o_act;
  sizes[6] = R.h2d;
  sizes[7] = R.d2h;
  ptrs[0] = (int64_t)R.act_off.data(); ptrs[1] = (int64_t)R.act.data(); ptrs[2] = (int64_t)R.rows.data();
  ptrs[3] = (int64_t)R.A.data(); ptrs[4] = (int64_t)R.mq.data(); ptrs[5] = (int64_t)R.perm.data();
  ptrs[6] = (int64_t)R.k.data(); ptrs[7] = (int64_t)R.steps.data(); ptrs[8] = (int64_t)R.gap.data();
  ptrs[9] = (int64_t)R.stack; ptrs[10] = (int64_t)R.dbuf; ptrs[11] = (int64_t)R.dup;
  ptrs[12] = (int64_t)R.ev;
  ptrs[13] = (int64_t)R.idx.data();
  return 0;
}

// The caller has enqueued level L's Schur stage (engine lead control).
int skb_engine_ack(int64_t handle, int64_t L) {
  Engine* E = (Engine*)handle;
  {
    std::lock_guard<std::mutex> lk(E->m);
    if (L < E->acked) E->acked = L;
  }
  E->cv.notify_all();
  return 0;
}

int skb_engine_set_lead(int64_t handle, int64_t lead) {
  Engine* E = (Engine*)handle;
  {
    std::lock_guard<std::mutex> lk(E->m);
    E->lead = lead;
  }
  E->cv.notify_all();
  return 0;
}

// Make `stream` wait for level L's compression (the Schur stage reads its stacks).
int skb_engine_stream_wait(int64_t handle, int64_t L, void* stream) {
  Engine* E = (Engine*)handle;
  SKB_RET(cudaStreamWaitEvent((cudaStream_t)stream, E->out[L].ev, 0));
  return 0;
}

// Release level L's device buffers, stream-ordered on `stream` (after the
// Schur stage that reads them has been enqueued there).
int skb_engine_release(int64_t handle, int64_t L, void* stream) {
  Engine* E = (Engine*)handle;
  LevelOut& R = E->out[L];
  cudaStream_t s = (cudaStream_t)stream;
  static const bool defer = getenv("SKB_ENGINE_DEFER_FREE") != nullptr;   // race hunt
  if (defer && !E->freeing) return 0;
  if (R.stack) { cudaFreeAsync(R.stack, s); R.stack = nullptr; }
  if (R.dbuf) { cudaFreeAsync(R.dbuf, s); R.dbuf = nullptr; }
  if (R.dup) { cudaFreeAsync(R.dup, s); R.dup = nullptr; }
  return 0;
}

// Ask the engine to stop after its current level and wait for the thread.
int skb_engine_stop(int64_t handle) {
  Engine* E = (Engine*)handle;
  {
    std::lock_guard<std::mutex> lk(E->m);
    E->stop.store(true);
  }
  E->cv.notify_all();
  if (E->th.joinable()) E->th.join();
  return 0;
}

// Debug: copy snapshot `which` (0 stack after assembly, 1 after the
// pre-reduction, 2 after QRCP) of the SKB_ENGINE_SNAP level to host; returns
// the element count (n_host = capacity of `host` in doubles).
int64_t skb_debug_snap(int32_t which, double* host, int64_t n_host) {
  Snap& S = g_snap();
  if (which < 0 || which > 2 || !S.buf[which]) return -1;
  if (host && n_host >= S.n)
    if (cudaMemcpy(host, S.buf[which], sizeof(double) * S.n, cudaMemcpyDeviceToHost) != cudaSuccess)
      return -2;
  return S.n;
}

int skb_engine_free(int64_t handle, void* stream) {
  Engine* E = (Engine*)handle;
  if (E->th.joinable()) E->th.join();
  E->freeing = true;
  if (getenv("SKB_ENGINE_DEFER_FREE")) cudaDeviceSynchronize();
  for (int64_t L = E->lev_lo; L <= E->depth; ++L) {
    skb_engine_release(handle, L, stream);
    if (E->out[L].ev) cudaEventDestroy(E->out[L].ev);
  }
  bool failed = false;
  for (int64_t L = E->lev_lo; L <= E->depth; ++L) failed |= E->out[L].rc != 0;
  if (failed) cudaStreamSynchronize(E->s);   // a level that stopped early may have a copy in flight
  if (E->shared_pinned) {
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    *E->shared_pinned = false;       // the engine thread has joined: no copy in flight
  } else if (E->pinned) {
    cudaFreeHost(E->pinned);
  }
  if (E->shared_pack) {
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    g_pack().busy = false;
  } else if (E->pack) {
    cudaFreeHost(E->pack);
  }
  delete E;
  return 0;
}

}  // extern "C"

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
  // ... or the previous factorization's level table (skb_engine_set_update_table)
  const int64_t* old_table = nullptr;
};

// One level of the previous factorization (update): arrays owned by the
// caller, addressed through a table of int64 [depth + 1][O_NF] (row = level,
// all zero when the level did not exist).  code = ix * 2^level + iy, ascending.
enum { O_B = 0, O_CODE, O_ACT_OFF, O_ACT, O_PERM, O_K, O_PTR0, O_IPIV = O_PTR0 + 6, O_INFO, O_RATIO,
       O_STASH, O_ST_US, O_ST_PS, O_ST_SP, O_GAP, O_STEPS, O_NF };
struct OldLevel {
  int64_t B = 0;
  const int64_t *code, *act_off, *act, *k, *info, *st_us, *st_ps, *st_sp, *steps;
  const int32_t* perm;
  const uint64_t* ptr[6];
  const uint64_t* ipiv;
  const double *ratio, *gap;
  uint64_t stash;
};
inline OldLevel old_level(const int64_t* table, int64_t lev) {
  const int64_t* t = table + lev * O_NF;
  OldLevel O;
  O.B = t[O_B];
  O.code = (const int64_t*)t[O_CODE]; O.act_off = (const int64_t*)t[O_ACT_OFF];
  O.act = (const int64_t*)t[O_ACT]; O.perm = (const int32_t*)t[O_PERM]; O.k = (const int64_t*)t[O_K];
  for (int f = 0; f < 6; ++f) O.ptr[f] = (const uint64_t*)t[O_PTR0 + f];
  O.ipiv = (const uint64_t*)t[O_IPIV]; O.info = (const int64_t*)t[O_INFO];
  O.ratio = (const double*)t[O_RATIO]; O.stash = (uint64_t)t[O_STASH];
  O.st_us = (const int64_t*)t[O_ST_US]; O.st_ps = (const int64_t*)t[O_ST_PS];
  O.st_sp = (const int64_t*)t[O_ST_SP]; O.gap = (const double*)t[O_GAP];
  O.steps = (const int64_t*)t[O_STEPS];
  return O;
}
inline int64_t find_code(const OldLevel& O, int64_t code) {
  int64_t lo = 0, hi = O.B;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (O.code[mid] < code) lo = mid + 1;
    else hi = mid;
  }
  return (lo < O.B && O.code[lo] == code) ? lo : -1;
}

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

// Blocks until the engine may enqueue level L's kernels (run-ahead control,
// skb_engine_ack / skb_engine_set_lead); false when the engine was stopped.
bool launch_gate(Engine& E, int64_t L) {
  std::unique_lock<std::mutex> lk(E.m);
  E.cv.wait(lk, [&] { return E.stop.load() || E.lead < 0 || E.acked <= L + 1 + E.lead || L + 1 + E.lead > E.depth; });
  return !E.stop.load();
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
  if (E.todo && E.old_table) {
    const OldLevel O = old_level(E.old_table, L);
    const int64_t side = (int64_t)1 << L;
    std::vector<int64_t> sk;
    for (int64_t i = b0; i < b0 + nall; ++i) {
      if (E.todo[i]) continue;
      const int64_t pos = O.B ? find_code(O, E.ix[i] * side + E.iy[i]) : -1;
      if (pos < 0) return 20;               // clean box without a twin: the caller re-runs
      const int64_t a0 = O.act_off[pos], nk = O.k[pos];
      sk.resize(nk);
      for (int64_t j = 0; j < nk; ++j) sk[j] = O.act[a0 + O.perm[a0 + j]];
      const int64_t o = append(E, sk.data(), nk);
      if (o < 0) return 7;
      E.s_start[i] = o;
      E.s_len[i] = nk;
    }
  } else if (E.todo) {
    for (int64_t i = b0; i < b0 + nall; ++i) {
      if (E.todo[i]) continue;
      const int64_t n0 = E.clean_off[i], nk = E.clean_off[i + 1] - n0;
      const int64_t o = append(E, E.clean_skel + n0, nk);
      if (o < 0) return 7;
      E.s_start[i] = o;
      E.s_len[i] = nk;
    }
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
  const int64_t npk = o_f + nfar;
  tm.tick("pack");
  // the host side of the level (active sets, far lists, proxy rings, packing)
  // is done; only the kernel launches wait for the run-ahead gate
  if (!launch_gate(E, L)) return -1000;
  tm.tick("gate");
  SKB_RET(malloc_async((void**)&R.stack, sizeof(double) * std::max<int64_t>(so, 1), s));
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

// The engine thread allocates from a stream-ordered pool of its own (never
// shrinks), so its allocations never share a pool with the caller's.
cudaMemPool_t engine_pool(int dev) {
  static cudaMemPool_t pool = nullptr;
  static std::mutex pm;
  std::lock_guard<std::mutex> lk(pm);
  if (!pool) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      if (getenv("SKB_POOL_STRICT")) pool_strict(pool);   // debug, see ring_stage
    } else {
      pool = nullptr;
    }
  }
  return pool;
}

void engine_main(Engine* E) {
  cudaSetDevice(E->dev);
  use_engine_side(true);
  use_engine_ring(true);          // descriptor uploads through the engine's own pinned ring
  if (!getenv("SKB_ENGINE_SHARED_POOL")) skb::tl_pool() = engine_pool(E->dev);
  for (int64_t L = E->depth; L >= E->lev_lo; --L) {
    LevelOut& R = E->out[L];
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
        // grown with slack: an update chain's trees gain and lose a few boxes,
        // and cudaFreeHost / cudaHostAlloc wait for the device (0.9 s on cfg3)
        if (g_pinned) cudaFreeHost(g_pinned);
        g_pinned = nullptr; g_size = 0;
        SKB_RET(cudaHostAlloc((void**)&g_pinned, want + want / 2, cudaHostAllocDefault));
        g_size = want + want / 2;
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

// ===========================================================================
// Native level driver: the consumer side of the level loop (reference
// run_level / compress_box (c) / _finish_top sweep, skel.py:316-361, 384-396)
// on the calling thread, one C call for all levels:
//
//   wait for the engine's level -> X_RR pivot check of the level below
//   (migration rule skel.py:317-330: reported, the caller re-runs on its slow
//   path) -> merge with the previous factorization's clean boxes (update,
//   skel.py:342-353) -> factor storage layout -> Schur stage (skb_level_schur)
//   -> acknowledge -> augmentation sweep of the level below -> skeleton /
//   redundant / hole-column lists of the level on the device.
//
// The caller (skel.py) only wraps the resulting arrays afterwards.
// ===========================================================================
extern "C" int skb_level_schur(int64_t nbox, const int64_t* nB, const int64_t* k,
                               const int64_t* act_off, const double* pos, const double* nrm,
                               const double* w, const double* kappa, const int64_t* act_off_dev,
                               const int64_t* act_dev, const int32_t* perm_dev, const int64_t* A,
                               const int64_t* lda, const int64_t* child_off,
                               const uint64_t* child_xss, const uint64_t* T, const uint64_t* Xrr,
                               const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                               const uint64_t* Xss, const uint64_t* ipiv, int32_t* info_dev,
                               double* ratio_dev, int32_t pde, void* stream);
extern "C" int skb_level_aug(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                             const int64_t* cols_off, const int64_t* cols, const int64_t* sd_off,
                             const int64_t* sd, const int64_t* rd_off, const int64_t* rd,
                             const int64_t* c_off, const int64_t* c, const uint64_t* T,
                             const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                             const uint64_t* ipiv, double* UH, double* PsiV, double* UH_div,
                             double* schur, double* stash, const int64_t* st_us,
                             const int64_t* st_ps, const int64_t* st_sp, int32_t acc, void* stream);
extern "C" int skb_level_aug_update(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                                    const int64_t* cols_off, const int64_t* cols,
                                    const int64_t* sd_off, const int64_t* sd, const int64_t* rd_off,
                                    const int64_t* rd, const uint8_t* dirty, const uint8_t* parent_dirty,
                                    const uint64_t* T, const uint64_t* LU, const uint64_t* Xsr,
                                    const uint64_t* Xrsdiv, const uint64_t* ipiv, const uint64_t* old_us,
                                    const uint64_t* old_ps, const uint64_t* old_sp, int64_t nqc,
                                    const int64_t* qc, const uint8_t* qmask_dev, double* UH, double* PsiV,
                                    double* UH_div, double* schur, double* stash, const int64_t* st_us,
                                    const int64_t* st_ps, const int64_t* st_sp, void* stream);
extern "C" int skb_dev_alloc(int64_t bytes, void* stream, uint64_t* out);
extern "C" int skb_prof_add(int32_t fam, double flops, double bytes);

namespace {

struct DrvLevel {
  int64_t lev = 0, B = 0, nnew = 0;
  std::vector<int64_t> idx, code, act_off, act, k, steps, clean_pos, info, new_pos;
  std::vector<int32_t> perm;
  std::vector<double> gap, ratio;
  std::vector<uint64_t> ptr[6], ipiv;
  std::vector<int64_t> sd_off, sd, rd_off, rd, cols_off, cols, st_us, st_ps, st_sp;
  uint64_t slab = 0, stash = 0, desc = 0;
  int64_t slab_bytes = 0, stash_bytes = 0, desc_bytes = 0;
  int64_t o_desc[6] = {0, 0, 0, 0, 0, 0};     // element offsets: sd_off | sd | rd_off | rd | c_off | c
  cudaEvent_t ready = nullptr;                // level stream: factors and lists of the level final
  cudaEvent_t pev = nullptr;                  // X_RR pivot info of the new boxes landed
  char* pin = nullptr;                        // pinned: ratio (f64 x nnew) | info (i32 x nnew)
  bool resolved = true, adopted = false, used = false;
};

struct DrvCfg {
  cudaStream_t S, AS;
  const double* kap;
  int64_t q;
  int64_t npairs;
  const int64_t *pair_box, *pair_curve, *parent;
  double *UH, *PsiV, *UH_div, *schur;
  int64_t update;
  const uint8_t* dmask;
  int64_t nqc;
  const int64_t* qc;
  const uint8_t* qmask_dev;
  const int64_t* old_table;
  int64_t inc;
  uint64_t* xss;
  double floor;
  // npairs < 0: (box, curve) membership computed here from the tree's node lists
  const int64_t *level_nodes = nullptr, *level_nodes_off = nullptr, *node_start = nullptr,
                *node_cnt = nullptr, *curve_off = nullptr;
  int64_t ncurves = 0;
};

struct Driver {
  Engine* E = nullptr;
  DrvCfg c;
  std::vector<DrvLevel> lv;
  DrvLevel* prev = nullptr;
  char* pinned = nullptr;
  size_t pinned_cap = 0, pinned_used = 0;
  bool shared_pinned = false;
  int64_t h2d = 0, d2h = 0;
  int64_t fail_level = -1;
  std::vector<std::vector<int32_t>> curves;   // per box: curves with nodes in the box (ascending)
};

// process-wide pinned landing buffer of the pivot info (one driver at a time)
struct DrvPinned {
  char* p = nullptr;
  size_t cap = 0;
  bool busy = false;
};
DrvPinned& g_drv_pinned() {
  static DrvPinned b;
  return b;
}

// X_RR pivot info of a level's new boxes: wait for the copy, apply the
// migration rule's trigger (skel.py:317-330).  100 = a box must migrate.
int drv_resolve(Driver& D, DrvLevel& L, bool block = true) {
  if (L.resolved) return 0;
  if (!block) {
    const cudaError_t q = cudaEventQuery(L.pev);
    if (q == cudaErrorNotReady) return 0;
    SKB_RET(q);
  }
  SKB_RET(cudaEventSynchronize(L.pev));
  const double* ratio = (const double*)L.pin;
  const int32_t* info = (const int32_t*)(L.pin + 8 * L.nnew);
  bool bad = false;
  for (int64_t j = 0; j < L.nnew; ++j) {
    const int64_t p = L.new_pos[j];
    L.ratio[p] = ratio[j];
    L.info[p] = info[j];
    const int64_t nB = L.act_off[p + 1] - L.act_off[p];
    if ((info[j] >= 0 || ratio[j] < D.c.floor) && L.k[p] < nB) bad = true;
  }
  L.resolved = true;
  return bad ? 100 : 0;
}

int drv_sweep(Driver& D, DrvLevel& L) {
  const DrvCfg& c = D.c;
  const int64_t B = L.B, q = c.q;
  if (q <= 0 || B <= 0) return 0;
  SKB_RET(cudaStreamWaitEvent(c.AS, L.ready, 0));
  // per-box storage of the sweep results (outgoing UH_S | PsiV_S | Schur part)
  std::vector<int64_t> r(B);
  L.st_us.assign(B, 0); L.st_ps.assign(B, 0); L.st_sp.assign(B, 0);
  int64_t a = 0;
  for (int64_t b = 0; b < B; ++b) { L.st_us[b] = a; a += L.k[b] * q; }
  for (int64_t b = 0; b < B; ++b) { L.st_ps[b] = a; a += L.k[b] * (L.cols_off[b + 1] - L.cols_off[b]); }
  for (int64_t b = 0; b < B; ++b) { L.st_sp[b] = a; a += (L.cols_off[b + 1] - L.cols_off[b]) * q; }
  L.stash_bytes = 8 * std::max<int64_t>(a, 1);
  int rc;
  if ((rc = skb_dev_alloc(L.stash_bytes, c.AS, &L.stash))) return rc;
  for (int64_t b = 0; b < B; ++b) r[b] = (L.act_off[b + 1] - L.act_off[b]) - L.k[b];
  const int64_t zero = 0;
  const int64_t* cols = L.cols.empty() ? &zero : L.cols.data();
  const int64_t* dd = (const int64_t*)L.desc;
  if (!c.inc)
    return skb_level_aug(B, L.k.data(), r.data(), q, L.cols_off.data(), cols, dd + L.o_desc[0],
                         dd + L.o_desc[1], dd + L.o_desc[2], dd + L.o_desc[3], dd + L.o_desc[4],
                         dd + L.o_desc[5], L.ptr[0].data(), L.ptr[2].data(), L.ptr[3].data(),
                         L.ptr[4].data(), L.ipiv.data(), c.UH, c.PsiV, c.UH_div, c.schur,
                         (double*)L.stash, L.st_us.data(), L.st_ps.data(), L.st_sp.data(), 1, c.AS);
  std::vector<uint8_t> dirty(B), pdirty(B);
  std::vector<uint64_t> ous(B, 0), ops(B, 0), osp(B, 0);
  const OldLevel O = old_level(c.old_table, L.lev);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t i = L.idx[b], par = c.parent[i];
    dirty[b] = c.dmask[i];
    pdirty[b] = (par >= 0 && c.dmask[par]) ? 1 : 0;
    if (!dirty[b]) {
      const int64_t pos = L.clean_pos[b];
      if (pos < 0 || !O.stash) return 103;
      ous[b] = O.stash + 8 * (uint64_t)O.st_us[pos];
      ops[b] = O.stash + 8 * (uint64_t)O.st_ps[pos];
      osp[b] = O.stash + 8 * (uint64_t)O.st_sp[pos];
    }
  }
  const int64_t* sd = L.sd.empty() ? &zero : L.sd.data();
  const int64_t* rd = L.rd.empty() ? &zero : L.rd.data();
  return skb_level_aug_update(B, L.k.data(), r.data(), q, L.cols_off.data(), cols, L.sd_off.data(), sd,
                              L.rd_off.data(), rd, dirty.data(), pdirty.data(), L.ptr[0].data(),
                              L.ptr[2].data(), L.ptr[3].data(), L.ptr[4].data(), L.ipiv.data(),
                              ous.data(), ops.data(), osp.data(), c.nqc, c.nqc ? c.qc : &zero,
                              c.qmask_dev, c.UH, c.PsiV, c.UH_div, c.schur, (double*)L.stash,
                              L.st_us.data(), L.st_ps.data(), L.st_sp.data(), c.AS);
}

int drv_level(Driver& D, int64_t lev) {
  Engine& E = *D.E;
  const DrvCfg& c = D.c;
  LevelOut& R = E.out[lev];
  ETimer tm;
  {
    std::unique_lock<std::mutex> lk(E.m);
    E.cv.wait(lk, [&] { return R.ready; });
  }
  tm.tick("WAIT");
  if (R.rc) return R.rc == 20 ? 101 : 200 + std::abs(R.rc) % 100;
  D.h2d += R.h2d;
  D.d2h += R.d2h;
  int rc;
  // X_RR pivot info of the levels below: checked as it arrives, never waited
  // for here (a migration aborts the whole run, so the check only has to
  // happen before the run returns; waiting would serialise the host with
  // every level's Schur stage on the device)
  // (update: the few dirty boxes' compression chain is latency bound and the
  // level below is awaited -- that keeps its Schur / sweep kernels from
  // crowding the chain's kernels; measured 22.2 vs 23.8 ms on cfg2 moves)
  for (int64_t l2 = lev + 1; l2 <= E.depth; ++l2)
    if (D.lv[l2].used && (rc = drv_resolve(D, D.lv[l2], c.update && l2 == lev + 1))) return rc;
  tm.tick("resolve");
  const int64_t b0 = E.level_start[lev], B = E.level_start[lev + 1] - b0;
  DrvLevel& L = D.lv[lev];
  L.lev = lev;
  L.B = B;
  L.used = true;
  L.idx.resize(B); L.code.resize(B); L.act_off.assign(B + 1, 0);
  const int64_t side = (int64_t)1 << lev;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t i = b0 + b;
    L.idx[b] = i;
    L.code[b] = E.ix[i] * side + E.iy[i];
    L.act_off[b + 1] = L.act_off[b] + E.a_len[i];
  }
  const int64_t na = L.act_off[B];
  L.act.resize(na); L.perm.assign(na, 0);
  for (int64_t b = 0; b < B; ++b)
    if (E.a_len[b0 + b])
      memcpy(L.act.data() + L.act_off[b], E.big + E.a_start[b0 + b], sizeof(int64_t) * E.a_len[b0 + b]);
  L.k.assign(B, 0); L.steps.assign(B, 0); L.gap.assign(B, 1.0); L.ratio.assign(B, 1.0);
  L.info.assign(B, -1); L.clean_pos.assign(B, -1);
  for (auto& v : L.ptr) v.assign(B, 0);
  L.ipiv.assign(B, 0);
  // recompressed boxes: QRCP results of the engine
  const int64_t Bn = R.B;
  L.nnew = Bn;
  L.new_pos.resize(Bn);
  std::vector<uint8_t> is_new(B, 0);
  std::vector<int64_t> nBn(Bn), kn(Bn);
  for (int64_t j = 0; j < Bn; ++j) {
    const int64_t p = R.idx[j] - b0;
    if (p < 0 || p >= B) return 104;
    L.new_pos[j] = p;
    is_new[p] = 1;
    const int64_t n = R.act_off[j + 1] - R.act_off[j];
    if (n != L.act_off[p + 1] - L.act_off[p]) return 104;
    memcpy(L.perm.data() + L.act_off[p], R.perm.data() + R.act_off[j], sizeof(int32_t) * n);
    L.k[p] = R.k[j];
    L.steps[p] = R.steps[j];
    L.gap[p] = R.gap[j];
    nBn[j] = n;
    kn[j] = R.k[j];
  }
  // factor storage of the new boxes: T | X_rr | LU | X_sr | X_rs_div | Xss_mod per box (f64),
  // then the LU pivots (i32), in ONE allocation ordered on the level stream
  if (Bn > 0) {
    int64_t tot = 0, rsum = 0;
    for (int64_t j = 0; j < Bn; ++j) {
      const int64_t kk = kn[j], rr = nBn[j] - kk;
      tot += 3 * kk * rr + 2 * rr * rr + kk * kk;
      rsum += rr;
    }
    const int64_t nf = std::max<int64_t>(tot, 1);
    L.slab_bytes = 8 * nf + 4 * std::max<int64_t>(rsum, 1);
    if ((rc = skb_dev_alloc(L.slab_bytes, c.S, &L.slab))) return rc;
    int64_t fo = 0, io = 0;
    for (int64_t j = 0; j < Bn; ++j) {
      const int64_t p = L.new_pos[j], kk = kn[j], rr = nBn[j] - kk;
      const int64_t sz[6] = {kk * rr, rr * rr, rr * rr, kk * rr, rr * kk, kk * kk};
      // field-major inside the slab as in the Python layout: box-major blocks
      int64_t o = fo;
      for (int f = 0; f < 6; ++f) { L.ptr[f][p] = L.slab + 8 * (uint64_t)o; o += sz[f]; }
      fo = o;
      L.ipiv[p] = L.slab + 8 * (uint64_t)nf + 4 * (uint64_t)io;
      io += rr;
    }
  }
  // clean boxes share the previous factorization's memory (skel.py:342-353)
  if (Bn < B) {
    if (!c.update || !c.old_table) return 104;
    const OldLevel O = old_level(c.old_table, lev);
    if (!O.B) return 101;
    for (int64_t p = 0; p < B; ++p) {
      if (is_new[p]) continue;
      const int64_t pos = find_code(O, L.code[p]);
      if (pos < 0) return 101;
      const int64_t a0 = O.act_off[pos], n = O.act_off[pos + 1] - a0;
      if (n != L.act_off[p + 1] - L.act_off[p] ||
          (n && memcmp(O.act + a0, L.act.data() + L.act_off[p], sizeof(int64_t) * n)))
        return 102;                           // clean box changed its active set
      memcpy(L.perm.data() + L.act_off[p], O.perm + a0, sizeof(int32_t) * n);
      L.k[p] = O.k[pos]; L.steps[p] = O.steps[pos]; L.gap[p] = O.gap[pos];
      L.info[p] = O.info[pos]; L.ratio[p] = O.ratio[pos];
      for (int f = 0; f < 6; ++f) L.ptr[f][p] = O.ptr[f][pos];
      L.ipiv[p] = O.ipiv[pos];
      L.clean_pos[p] = pos;
    }
  }
  tm.tick("merge");
  if (Bn > 0) {
    if (prof().on) {
      // algorithmic work: stack + self-block bytes written,
      // Householder 2 m n^2 - 2/3 n^3, QRCP 2mn + sum_i 4 (m-i)(n-i-1)
      double ab = 0, gf = 0, gb = 0, qf = 0, qb = 0;
      for (int64_t j = 0; j < Bn; ++j) {
        const double m = (double)R.rows[j], n = (double)nBn[j], mq = (double)R.mq[j];
        ab += m * n + n * n;
        if (R.rows[j] > 2 * nBn[j]) { gf += 2 * m * n * n - 2.0 / 3.0 * n * n * n; gb += m * n; }
        qf += 2.0 * mq * n;
        for (int64_t i = 0; i < R.steps[j]; ++i) qf += 4.0 * (mq - i) * (n - i - 1);
        qb += mq * n;
      }
      skb_prof_add(F_ASSEMBLE, 0.0, 8.0 * ab);
      skb_prof_add(F_GEQRF, gf, 8.0 * gb);
      skb_prof_add(F_QRCP, qf, 8.0 * qb);
    }
    // (c) Schur stage of the new boxes on the level stream
    SKB_RET(cudaStreamWaitEvent(c.S, R.ev, 0));
    std::vector<int64_t> co(5 * Bn);
    std::vector<uint64_t> cx(4 * Bn), pT(Bn), pXrr(Bn), pLU(Bn), pXsr(Bn), pDiv(Bn), pXss(Bn), pIp(Bn);
    for (int64_t j = 0; j < Bn; ++j) {
      const int64_t i = R.idx[j], p = L.new_pos[j];
      bool inner = false;
      int64_t cum = 0;
      for (int qd = 0; qd < 4; ++qd) {
        const int64_t ch = E.children[4 * i + qd];
        if (ch >= 0) {
          inner = true;
          cum += E.s_len[ch];
          co[5 * j + 1 + qd] = cum;
          cx[4 * j + qd] = c.xss[ch];
        } else {
          co[5 * j + 1 + qd] = -1;
          cx[4 * j + qd] = 0;
        }
      }
      co[5 * j] = inner ? 0 : -1;
      pT[j] = L.ptr[0][p]; pXrr[j] = L.ptr[1][p]; pLU[j] = L.ptr[2][p]; pXsr[j] = L.ptr[3][p];
      pDiv[j] = L.ptr[4][p]; pXss[j] = L.ptr[5][p]; pIp[j] = L.ipiv[p];
    }
    char* pbuf = nullptr;
    SKB_RET(malloc_async((void**)&pbuf, (size_t)(12 * Bn), c.S));
    if ((rc = skb_level_schur(Bn, nBn.data(), kn.data(), R.act_off.data(), E.pos, E.nrm, E.w, c.kap,
                              R.dup, R.dup + R.o_act, (const int32_t*)(R.dbuf + R.o_int), R.A.data(),
                              R.rows.data(), co.data(), cx.data(), pT.data(), pXrr.data(), pLU.data(),
                              pXsr.data(), pDiv.data(), pXss.data(), pIp.data(),
                              (int32_t*)(pbuf + 8 * Bn), (double*)pbuf, E.pde, c.S)))
      return rc;
    const size_t need = (size_t)(12 * Bn + 16);
    if (D.pinned_used + need > D.pinned_cap) return 105;
    L.pin = D.pinned + D.pinned_used;
    D.pinned_used += (need + 15) & ~(size_t)15;
    SKB_RET(cudaMemcpyAsync(L.pin, pbuf, (size_t)(12 * Bn), cudaMemcpyDeviceToHost, c.S));
    SKB_RET(cudaEventRecord(L.pev, c.S));
    L.resolved = false;
    D.d2h += 12 * Bn;
    cudaFreeAsync(pbuf, c.S);
    // the engine's level buffers (stacks, permutations, descriptors) are read
    // by the Schur stage only: released stream-ordered behind it
    if (R.stack) { cudaFreeAsync(R.stack, c.S); R.stack = nullptr; }
    if (R.dbuf) { cudaFreeAsync(R.dbuf, c.S); R.dbuf = nullptr; }
    if (R.dup) { cudaFreeAsync(R.dup, c.S); R.dup = nullptr; }
    {
      std::lock_guard<std::mutex> lk(E.m);
      if (lev < E.acked) E.acked = lev;
    }
    E.cv.notify_all();
  }
  tm.tick("schur");
  for (int64_t p = 0; p < B; ++p) c.xss[b0 + p] = L.ptr[5][p];
  // the level below is final now: its augmentation sweep goes to the sweep stream
  if (D.prev && (rc = drv_sweep(D, *D.prev))) return rc;
  tm.tick("sweep");
  // skeleton / redundant DOF lists and hole columns of the level, one upload
  L.sd_off.assign(B + 1, 0); L.rd_off.assign(B + 1, 0); L.cols_off.assign(B + 1, 0);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t n = L.act_off[b + 1] - L.act_off[b];
    L.sd_off[b + 1] = L.sd_off[b] + L.k[b];
    L.rd_off[b + 1] = L.rd_off[b] + (n - L.k[b]);
  }
  L.sd.resize(L.sd_off[B]); L.rd.resize(L.rd_off[B]);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t a0 = L.act_off[b], n = L.act_off[b + 1] - a0, kk = L.k[b];
    const int64_t* act = L.act.data() + a0;
    const int32_t* pm = L.perm.data() + a0;
    int64_t* sd = L.sd.data() + L.sd_off[b];
    int64_t* rd = L.rd.data() + L.rd_off[b];
    for (int64_t j = 0; j < kk; ++j) sd[j] = act[pm[j]];
    for (int64_t j = kk; j < n; ++j) rd[j - kk] = act[pm[j]];
  }
  L.cols.clear();
  if (c.npairs < 0) {
    // curve membership leaves -> root (tree.py hole_pairs): a leaf holds the
    // curves of its nodes, an internal box the union of its children's
    std::vector<int32_t> tmp;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t i = L.idx[b];
      std::vector<int32_t>& cv = D.curves[i];
      tmp.clear();
      if (E.leaf[i]) {
        const int64_t* nd = c.level_nodes + c.level_nodes_off[lev] + c.node_start[i];
        int32_t last = -1;
        for (int64_t t = 0; t < c.node_cnt[i]; ++t) {
          const int32_t cur = (int32_t)(std::upper_bound(c.curve_off, c.curve_off + c.ncurves + 1, nd[t]) -
                                        c.curve_off) - 1;
          if (cur != last) { tmp.push_back(cur); last = cur; }
        }
      } else {
        for (int qd = 0; qd < 4; ++qd) {
          const int64_t ch = E.children[4 * i + qd];
          if (ch >= 0) tmp.insert(tmp.end(), D.curves[ch].begin(), D.curves[ch].end());
        }
      }
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      cv = tmp;
      for (int32_t cur : cv)
        if (cur >= 1)
          for (int e = 0; e < 3; ++e) L.cols.push_back(3 * (int64_t)(cur - 1) + e);
      L.cols_off[b + 1] = (int64_t)L.cols.size();
    }
  } else if (c.npairs > 0) {
    for (int64_t b = 0; b < B; ++b) {
      const int64_t i = L.idx[b];
      const int64_t* lo = std::lower_bound(c.pair_box, c.pair_box + c.npairs, i);
      for (; lo < c.pair_box + c.npairs && *lo == i; ++lo) {
        const int64_t cur = c.pair_curve[lo - c.pair_box];
        if (cur >= 1)
          for (int e = 0; e < 3; ++e) L.cols.push_back(3 * (cur - 1) + e);
      }
      L.cols_off[b + 1] = (int64_t)L.cols.size();
    }
  }
  {
    auto al = [](int64_t o) { return (o + 1) & ~(int64_t)1; };
    const int64_t nsd = std::max<int64_t>((int64_t)L.sd.size(), 1), nrd = std::max<int64_t>((int64_t)L.rd.size(), 1);
    const int64_t ncl = std::max<int64_t>((int64_t)L.cols.size(), 1);
    L.o_desc[0] = 0;
    L.o_desc[1] = al(B + 1);
    L.o_desc[2] = al(L.o_desc[1] + nsd);
    L.o_desc[3] = al(L.o_desc[2] + B + 1);
    L.o_desc[4] = al(L.o_desc[3] + nrd);
    L.o_desc[5] = al(L.o_desc[4] + B + 1);
    const int64_t tot = al(L.o_desc[5] + ncl);
    std::vector<int64_t> h(tot, 0);
    memcpy(h.data() + L.o_desc[0], L.sd_off.data(), sizeof(int64_t) * (B + 1));
    if (!L.sd.empty()) memcpy(h.data() + L.o_desc[1], L.sd.data(), sizeof(int64_t) * L.sd.size());
    memcpy(h.data() + L.o_desc[2], L.rd_off.data(), sizeof(int64_t) * (B + 1));
    if (!L.rd.empty()) memcpy(h.data() + L.o_desc[3], L.rd.data(), sizeof(int64_t) * L.rd.size());
    memcpy(h.data() + L.o_desc[4], L.cols_off.data(), sizeof(int64_t) * (B + 1));
    if (!L.cols.empty()) memcpy(h.data() + L.o_desc[5], L.cols.data(), sizeof(int64_t) * L.cols.size());
    L.desc_bytes = 8 * tot;
    if ((rc = skb_dev_alloc(L.desc_bytes, c.S, &L.desc))) return rc;
    if ((rc = ring_stage(h.data(), (size_t)L.desc_bytes, c.S, (void*)L.desc))) return rc;
    D.h2d += L.desc_bytes;
  }
  SKB_RET(cudaEventRecord(L.ready, c.S));
  D.prev = &L;
  tm.tick("lists");
  if (ETimer::on()) fprintf(stderr, "driver level %lld (%lld boxes, %lld new):%s us\n", (long long)lev, (long long)B, (long long)Bn, tm.buf);
  return 0;
}

}  // namespace

extern "C" {

// Grow the engine's pool / the default stream-ordered pool to at least the
// given reserved sizes now (one allocation + free each), so that no level of
// a later factorization pays for pool growth -- a host-side stall of tens to
// hundreds of milliseconds in the middle of the level pipeline.
int skb_pool_prewarm(int64_t engine_bytes, int64_t default_bytes) {
  int dev = 0;
  SKB_RET(cudaGetDevice(&dev));
  cudaMemPool_t pools[2] = {getenv("SKB_ENGINE_SHARED_POOL") ? nullptr : engine_pool(dev), nullptr};
  SKB_RET(cudaDeviceGetDefaultMemPool(&pools[1], dev));
  const int64_t want[2] = {engine_bytes, default_bytes};
  for (int i = 0; i < 2; ++i) {
    if (!pools[i] || want[i] <= 0) continue;
    uint64_t thr = ~0ull, have = 0;
    SKB_RET(cudaMemPoolSetAttribute(pools[i], cudaMemPoolAttrReleaseThreshold, &thr));
    SKB_RET(cudaMemPoolGetAttribute(pools[i], cudaMemPoolAttrReservedMemCurrent, &have));
    if ((int64_t)have >= want[i]) continue;
    void* p = nullptr;
    if (cudaMallocFromPoolAsync(&p, (size_t)want[i], pools[i], 0) != cudaSuccess) {
      cudaGetLastError();                    // not enough memory: keep what is there
      continue;
    }
    SKB_RET(cudaFreeAsync(p, 0));
  }
  SKB_RET(cudaStreamSynchronize(0));
  return 0;
}

// Update mode with the previous factorization's level table (see OldLevel):
// clean boxes' skeletons are read from it by the engine itself.
int skb_engine_set_update_table(int64_t handle, const uint8_t* todo, const int64_t* old_table) {
  Engine* E = (Engine*)handle;
  E->todo = todo;
  E->old_table = old_table;
  return 0;
}

// Run the consumer side of every level on the calling thread (see above).
// cfg (int64 x 24; [20..23] = level_nodes, level_nodes_off, node_start, node_cnt and
// [5], [6] = curve offsets, curve count when npairs < 0): level stream, sweep stream, curvature (device), q, npairs,
// pair_box, pair_curve, parent, UH, PsiV, UH_div, schur, update, dmask, nqc, qc,
// qmask (device), old level table, incremental sweep, xss (uint64 per box).
// Returns 0, 100 (a box must migrate), 101/102 (clean box missing / changed)
// or a library error; the handle is valid either way (skb_drv_free).
int skb_drv_run(int64_t engine, const int64_t* cfg, double pivot_floor, int64_t* handle) {
  Engine* E = (Engine*)engine;
  Driver* D = new Driver();
  *handle = (int64_t)D;
  D->E = E;
  DrvCfg& c = D->c;
  c.S = (cudaStream_t)cfg[0]; c.AS = (cudaStream_t)cfg[1];
  c.kap = (const double*)cfg[2]; c.q = cfg[3]; c.npairs = cfg[4];
  c.pair_box = (const int64_t*)cfg[5]; c.pair_curve = (const int64_t*)cfg[6];
  c.parent = (const int64_t*)cfg[7];
  c.UH = (double*)cfg[8]; c.PsiV = (double*)cfg[9]; c.UH_div = (double*)cfg[10]; c.schur = (double*)cfg[11];
  c.update = cfg[12]; c.dmask = (const uint8_t*)cfg[13]; c.nqc = cfg[14]; c.qc = (const int64_t*)cfg[15];
  c.qmask_dev = (const uint8_t*)cfg[16]; c.old_table = (const int64_t*)cfg[17]; c.inc = cfg[18];
  c.xss = (uint64_t*)cfg[19];
  c.floor = pivot_floor;
  if (c.npairs < 0) {
    c.level_nodes = (const int64_t*)cfg[20]; c.level_nodes_off = (const int64_t*)cfg[21];
    c.node_start = (const int64_t*)cfg[22]; c.node_cnt = (const int64_t*)cfg[23];
    c.curve_off = (const int64_t*)cfg[5]; c.ncurves = cfg[6];
    D->curves.resize(E->level_start[E->depth + 1]);
  }
  D->lv.resize(E->depth + 1);
  const int64_t nbox = E->level_start[E->depth + 1];
  {
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    DrvPinned& g = g_drv_pinned();
    const size_t want = (size_t)(12 * nbox + 32 * (E->depth + 2) + 1024);
    if (!g.busy) {
      if (g.cap < want) {
        if (g.p) cudaFreeHost(g.p);
        g.p = nullptr; g.cap = 0;
        SKB_RET(cudaHostAlloc((void**)&g.p, want + want / 2, cudaHostAllocDefault));
        g.cap = want + want / 2;
      }
      g.busy = true;
      D->pinned = g.p; D->pinned_cap = g.cap; D->shared_pinned = true;
    } else {
      SKB_RET(cudaHostAlloc((void**)&D->pinned, want, cudaHostAllocDefault));
      D->pinned_cap = want;
    }
  }
  for (int64_t L = 1; L <= E->depth; ++L) {
    SKB_RET(cudaEventCreateWithFlags(&D->lv[L].ready, cudaEventDisableTiming));
    SKB_RET(cudaEventCreateWithFlags(&D->lv[L].pev, cudaEventDisableTiming));
  }
  for (int64_t L = E->depth; L >= 1; --L) {
    const int rc = drv_level(*D, L);
    if (rc) { D->fail_level = L; return rc; }
  }
  if (D->prev) {
    int rc;
    if ((rc = drv_sweep(*D, *D->prev))) { D->fail_level = D->prev->lev; return rc; }
  }
  // pivot info already landed is checked now; the rest by skb_drv_resolve (the
  // caller first enqueues its root block / corner LU behind the last level)
  for (int64_t L = E->depth; L >= 1; --L) {
    if (!D->lv[L].used) continue;
    const int rc = drv_resolve(*D, D->lv[L], false);
    if (rc) { D->fail_level = L; return rc; }
  }
  return 0;
}

// Wait for the X_RR pivot info of every level (the Schur stages on the
// device) and apply the migration trigger: 0, or 100 = a box must migrate.
int skb_drv_resolve(int64_t handle) {
  Driver* D = (Driver*)handle;
  for (int64_t L = (int64_t)D->lv.size() - 1; L >= 1; --L) {
    if (!D->lv[L].used) continue;
    const int rc = drv_resolve(*D, D->lv[L]);
    if (rc) { D->fail_level = L; return rc; }
  }
  return 0;
}

// Arrays of one level (valid until skb_drv_free).  sizes (int64 x 24): B, na, nnew, nsd,
// nrd, ncols, slab, slab_bytes, stash, stash_bytes, desc, desc_bytes, o_desc[6],
// total h2d, total d2h.  ptrs (int64 x 32): idx, code, act_off, act, perm(i32), k, steps,
// gap, info, ratio, clean_pos, ptr[6], ipiv, sd_off, sd, rd_off, rd, cols_off, cols,
// st_us, st_ps, st_sp, new_pos.  The device allocations become the caller's.
int skb_drv_level(int64_t handle, int64_t lev, int64_t* sizes, int64_t* ptrs) {
  Driver* D = (Driver*)handle;
  if (lev < 1 || lev >= (int64_t)D->lv.size()) return 1;
  DrvLevel& L = D->lv[lev];
  if (!L.used) return 2;
  L.adopted = true;
  int64_t* s = sizes;
  s[0] = L.B; s[1] = (int64_t)L.act.size(); s[2] = L.nnew; s[3] = (int64_t)L.sd.size();
  s[4] = (int64_t)L.rd.size(); s[5] = (int64_t)L.cols.size(); s[6] = (int64_t)L.slab; s[7] = L.slab_bytes;
  s[8] = (int64_t)L.stash; s[9] = L.stash_bytes; s[10] = (int64_t)L.desc; s[11] = L.desc_bytes;
  for (int i = 0; i < 6; ++i) s[12 + i] = L.o_desc[i];
  s[18] = D->h2d; s[19] = D->d2h;
  int64_t* p = ptrs;
  p[0] = (int64_t)L.idx.data(); p[1] = (int64_t)L.code.data(); p[2] = (int64_t)L.act_off.data();
  p[3] = (int64_t)L.act.data(); p[4] = (int64_t)L.perm.data(); p[5] = (int64_t)L.k.data();
  p[6] = (int64_t)L.steps.data(); p[7] = (int64_t)L.gap.data(); p[8] = (int64_t)L.info.data();
  p[9] = (int64_t)L.ratio.data(); p[10] = (int64_t)L.clean_pos.data();
  for (int f = 0; f < 6; ++f) p[11 + f] = (int64_t)L.ptr[f].data();
  p[17] = (int64_t)L.ipiv.data(); p[18] = (int64_t)L.sd_off.data(); p[19] = (int64_t)L.sd.data();
  p[20] = (int64_t)L.rd_off.data(); p[21] = (int64_t)L.rd.data(); p[22] = (int64_t)L.cols_off.data();
  p[23] = (int64_t)L.cols.data(); p[24] = (int64_t)L.st_us.data(); p[25] = (int64_t)L.st_ps.data();
  p[26] = (int64_t)L.st_sp.data(); p[27] = (int64_t)L.new_pos.data();
  return 0;
}

int skb_drv_free(int64_t handle) {
  Driver* D = (Driver*)handle;
  if (!D) return 0;
  bool orphan = false;
  for (auto& L : D->lv) orphan |= L.used && !L.adopted && (L.slab || L.stash || L.desc);
  if (orphan) {
    // an aborted run: nobody took over these allocations
    cudaStreamSynchronize(D->c.S);
    cudaStreamSynchronize(D->c.AS);
    for (auto& L : D->lv)
      if (L.used && !L.adopted) {
        if (L.slab) cudaFree((void*)L.slab);
        if (L.stash) cudaFree((void*)L.stash);
        if (L.desc) cudaFree((void*)L.desc);
      }
  }
  bool pending = false;
  for (auto& L : D->lv) pending |= !L.resolved;
  if (pending) cudaStreamSynchronize(D->c.S);     // a pivot-info copy may still be in flight
  for (auto& L : D->lv) {
    if (L.ready) cudaEventDestroy(L.ready);
    if (L.pev) cudaEventDestroy(L.pev);
  }
  if (D->shared_pinned) {
    std::lock_guard<std::recursive_mutex> lk(host_mutex());
    g_drv_pinned().busy = false;
  } else if (D->pinned) {
    cudaFreeHost(D->pinned);
  }
  delete D;
  return 0;
}

}  // extern "C"

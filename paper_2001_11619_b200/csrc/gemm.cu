// Grouped fp64 GEMM on the DMMA tensor path (mma.sync.m8n8k4.f64 -> SASS DMMA).
//
// One launch covers every (problem, output tile) pair of a ragged batch -- e.g.
// the Schur products of all boxes of a quadtree level (reference
// skel.py:321-334), the augmentation sweep (skel.py:384-396), the solve /
// apply sweeps (skel.py:126-221) or the trailing updates of a batched blocked
// QR / LU.
//
// sm_100a has no fp64 tcgen05 kind, so the tensor path is warp-level DMMA;
// the kernel is the Ampere-style multistage design that reaches the DMMA peak:
// operand tiles move global -> shared memory with cp.async (8-byte copies with
// zero fill at the ragged edges: row pointers of sub-blocks are only 8-byte
// aligned), STAGES deep, so the loads of k-tile t+2 overlap the DMMAs of t.
// Shared layouts follow op(A) / op(B)'s memory order (k-contiguous rows for
// A / B^T, m- / n-contiguous rows otherwise) with a stride = 4 mod 16 doubles:
// every fragment read (8x4 A / 4x8 B, one double per lane) and every cp.async
// write is bank-conflict free.
//
// Two tile shapes: 64 x 64 (4 warps of 32 x 32) for the many small problems of
// the lower levels, 128 x 128 (8 warps of 64 x 32) when the batch is made of
// large problems.  Each output element is produced by one thread with the same
// K order (k-tiles of 16 in increasing k, DMMA k-chunks of 4): results are
// deterministic, independent of the tile shape, of the batch composition and
// of the number of columns n (the update path relies on this).
#include "common.cuh"

namespace skb {

constexpr int BK = 16;
constexpr int KPAD = BK + 4;     // k-contiguous rows: 20 doubles (20 % 16 == 4)

__device__ __forceinline__ int find_problem(const SkbGemm* __restrict__ p, int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// BM x BN output tile, WM x WN warps (warp tile (BM/WM) x (BN/WN)), STAGES-deep pipeline.
template <int BM, int BN, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int NT = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN;      // warp tile
  static constexpr int MI = TM / 8, NI = TN / 8;        // DMMA tiles per warp
  static constexpr int A_ELEMS = (BM * KPAD > BK * (BM + 4)) ? BM * KPAD : BK * (BM + 4);
  static constexpr int B_ELEMS = (BN * KPAD > BK * (BN + 4)) ? BN * KPAD : BK * (BN + 4);
  static constexpr size_t SMEM = sizeof(double) * (size_t)STAGES * (A_ELEMS + B_ELEMS);
};

template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(WM * WN * 32)
k_gemm_grouped(const SkbGemm* __restrict__ probs, int nprob) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  constexpr int NT = C::NT, MI = C::MI, NI = C::NI;
  extern __shared__ double sm[];
  double* As = sm;                                    // [STAGES][A_ELEMS]
  double* Bs = sm + STAGES * C::A_ELEMS;              // [STAGES][B_ELEMS]
  const int64_t tile = blockIdx.x;
  const int pi = find_problem(probs, nprob, tile);
  const SkbGemm P = probs[pi];
  const int64_t local = tile - P.tile_begin;
  const int64_t ntn = (P.n + BN - 1) / BN;
  const int64_t m0 = (local / ntn) * BM;
  const int64_t n0 = (local % ntn) * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  // shared strides: element (row i of op(A), k p) at As[i * a_i + p * a_p]
  const bool ta = P.transA != 0, tb = P.transB != 0;
  const int a_i = ta ? 1 : KPAD, a_p = ta ? BM + 4 : 1;
  const int b_j = tb ? KPAD : 1, b_p = tb ? 1 : BN + 4;

  // Every thread copies a fixed column (k-contiguous layouts) or a fixed row
  // (m/n-contiguous layouts) of each operand tile: one base pointer and one
  // stride per operand, advanced per k-tile (keeps the register count low).
  static_assert(NT % BK == 0 && NT % BM == 0 && NT % BN == 0, "thread mapping");
  constexpr int A_IT = BM * BK / NT, B_IT = BN * BK / NT;
  int a_soff, a_sstep, b_soff, b_sstep;          // shared offset of copy 0 and per-copy step
  int64_t a_goff, a_gstep, b_goff, b_gstep;      // same in global memory (elements)
  int a_fix, a_var0, a_varstep, b_fix, b_var0, b_varstep;   // bounds: fixed / stepping coordinate
  if (ta) {      // op(A)[i][p] = A[p * lda + i]: thread = row i (coalesced over i), copies step p
    const int i = tid % BM, p0 = tid / BM;
    a_soff = i * a_i + p0 * a_p; a_sstep = (NT / BM) * a_p;
    a_goff = (int64_t)p0 * P.lda + m0 + i; a_gstep = (int64_t)(NT / BM) * P.lda;
    a_fix = i; a_var0 = p0; a_varstep = NT / BM;
  } else {       // op(A)[i][p] = A[i * lda + p]: thread = k column p, copies step i
    const int p = tid % BK, i0 = tid / BK;
    a_soff = i0 * a_i + p * a_p; a_sstep = (NT / BK) * a_i;
    a_goff = (m0 + i0) * P.lda + p; a_gstep = (int64_t)(NT / BK) * P.lda;
    a_fix = p; a_var0 = i0; a_varstep = NT / BK;
  }
  if (tb) {      // op(B)[p][j] = B[j * ldb + p]: thread = k column p, copies step j
    const int p = tid % BK, j0 = tid / BK;
    b_soff = j0 * b_j + p * b_p; b_sstep = (NT / BK) * b_j;
    b_goff = (n0 + j0) * P.ldb + p; b_gstep = (int64_t)(NT / BK) * P.ldb;
    b_fix = p; b_var0 = j0; b_varstep = NT / BK;
  } else {       // op(B)[p][j] = B[p * ldb + j]: thread = column j, copies step p
    const int j = tid % BN, p0 = tid / BN;
    b_soff = j * b_j + p0 * b_p; b_sstep = (NT / BN) * b_p;
    b_goff = (int64_t)p0 * P.ldb + n0 + j; b_gstep = (int64_t)(NT / BN) * P.ldb;
    b_fix = j; b_var0 = p0; b_varstep = NT / BN;
  }
  const int64_t a_kstep = ta ? (int64_t)BK * P.lda : BK;     // global advance per k-tile
  const int64_t b_kstep = tb ? BK : (int64_t)BK * P.ldb;

  auto load = [&](int64_t kt, int buf) {
    const int64_t k0 = kt * BK;
    double* as = As + buf * C::A_ELEMS + a_soff;
    double* bs = Bs + buf * C::B_ELEMS + b_soff;
    const double* ga = P.A + a_goff + kt * a_kstep;
    const double* gb = P.B + b_goff + kt * b_kstep;
    // in range: (row, k) of op(A) = ta ? (fix, k0 + var) : (m0 + var, k0 + fix)
    const int64_t alim_fix = ta ? P.m - m0 : P.k - k0, alim_var = ta ? P.k - k0 : P.m - m0;
    const int64_t blim_fix = tb ? P.k - k0 : P.n - n0, blim_var = tb ? P.n - n0 : P.k - k0;
    const bool afix = a_fix < alim_fix, bfix = b_fix < blim_fix;
#pragma unroll
    for (int it = 0; it < A_IT; ++it) {
      const bool ok = afix && (a_var0 + it * a_varstep) < alim_var;
      cp_async8(as + it * a_sstep, ok ? ga + it * a_gstep : P.A, ok);
    }
#pragma unroll
    for (int it = 0; it < B_IT; ++it) {
      const bool ok = bfix && (b_var0 + it * b_varstep) < blim_var;
      cp_async8(bs + it * b_sstep, ok ? gb + it * b_gstep : P.B, ok);
    }
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t nk = (P.k + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  const int ar = wm * C::TM + (lane >> 2), ac = lane & 3;     // fragment coordinates
  const int bc = wn * C::TN + (lane >> 2), br = lane & 3;
  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nt = kt + STAGES - 1;
      if (nt < nk) load(nt, (int)(nt % STAGES));
      cp_commit();
    }
    const double* as = As + (kt % STAGES) * C::A_ELEMS;
    const double* bs = Bs + (kt % STAGES) * C::B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[mi] = as[(ar + mi * 8) * a_i + (kk + ac) * a_p];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = bs[(bc + ni * 8) * b_j + (kk + br) * b_p];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
  cp_wait<0>();

  // epilogue: D = alpha*acc + beta*C
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t gi = m0 + wm * C::TM + mi * 8 + (lane >> 2);
    if (gi >= P.m) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = n0 + wn * C::TN + ni * 8 + (lane & 3) * 2 + h;
        if (gj >= P.n) continue;
        double v = P.alpha * acc[mi][ni][h];
        if (P.beta != 0.0) v += P.beta * P.C[gi * P.ldc + gj];
        P.D[gi * P.ldd + gj] = v;
      }
    }
  }
}

namespace {

template <int BM, int BN, int WM, int WN, int STAGES>
int launch_grouped(SkbGemm* probs, int64_t nprob, cudaStream_t s) {
  using Cfg = GemmCfg<BM, BN, WM, WN, STAGES>;
  int64_t tiles = 0;
  for (int64_t i = 0; i < nprob; ++i) {
    probs[i].tile_begin = tiles;
    if (probs[i].m > 0 && probs[i].n > 0)
      tiles += ((probs[i].m + BM - 1) / BM) * ((probs[i].n + BN - 1) / BN);
  }
  if (tiles == 0) return 0;
  if (tiles > 0x7fffffff) return 3;
  auto fn = k_gemm_grouped<BM, BN, WM, WN, STAGES>;
  SKB_RET(smem_optin((const void*)fn));
  SkbGemm* d = nullptr;
  int rc = upload(probs, nprob, s, &d);
  if (rc) return rc;
  fn<<<(unsigned)tiles, Cfg::NT, Cfg::SMEM, s>>>(d, (int)nprob);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(d, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // namespace

int gemm_grouped(SkbGemm* probs, int64_t nprob, cudaStream_t s) {
  if (nprob <= 0) return 0;
  double fl = 0.0, big = 0.0;
  for (int64_t i = 0; i < nprob; ++i) {
    const double f = 2.0 * (double)probs[i].m * (double)probs[i].n * (double)probs[i].k;
    fl += f;
    if (probs[i].m >= 96 && probs[i].n >= 96) big += f;
  }
  if (fl == 0.0) {
    // k == 0 problems still define D = beta * C
    bool any = false;
    for (int64_t i = 0; i < nprob; ++i) any |= probs[i].m > 0 && probs[i].n > 0;
    if (!any) return 0;
  }
  int rc;
  {
    ProfScope ps(F_GEMM, s);
    // batches dominated by large problems: 128 x 128 tiles; else 64 x 64
    // (SKB_GEMM_TILE=64|128 forces one: the tests check both give the same bits)
    static const int force = getenv("SKB_GEMM_TILE") ? atoi(getenv("SKB_GEMM_TILE")) : 0;
    int64_t tiles128 = 0;
    for (int64_t i = 0; i < nprob; ++i)
      if (probs[i].m > 0 && probs[i].n > 0) tiles128 += ((probs[i].m + 127) / 128) * ((probs[i].n + 127) / 128);
    // 128 x 128 tiles only when they still fill two waves of the 148 SMs
    const bool large = force ? force == 128 : (big >= 0.75 * fl && fl > 0.0 && tiles128 >= 296);
    if (large) rc = launch_grouped<128, 128, 2, 4, 3>(probs, nprob, s);
    else rc = launch_grouped<64, 64, 2, 2, 3>(probs, nprob, s);
  }
  if (prof().on) prof().flops[F_GEMM] += fl;
  return rc;
}

}  // namespace skb

extern "C" int skb_gemm_grouped(SkbGemm* probs, int64_t nprob, void* stream) {
  return skb::gemm_grouped(probs, nprob, (cudaStream_t)stream);
}

// Grouped fp64 GEMM on the DMMA tensor path (mma.sync.m8n8k4.f64 -> SASS DMMA).
//
// One launch covers every (problem, 64x64 output tile) pair of a ragged batch --
// e.g. the Schur products of all boxes of a quadtree level (reference
// skel.py:321-334) or the trailing updates of a batched blocked QR / LU.
// Each output element is produced by exactly one CTA with a fixed K order, so
// results are deterministic and independent of the rest of the batch.
#include "common.cuh"

namespace skb {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int GEMM_THREADS = 128;
constexpr int LDS = BM + 4;   // 68 doubles: conflict-free fragment reads (68 % 16 == 4)

__device__ __forceinline__ int find_problem(const SkbGemm* __restrict__ p, int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(GEMM_THREADS)
k_gemm_grouped(const SkbGemm* __restrict__ probs, int nprob) {
  __shared__ double As[2][BK][LDS];
  __shared__ double Bs[2][BK][LDS];
  const int64_t tile = blockIdx.x;
  const int pi = find_problem(probs, nprob, tile);
  const SkbGemm P = probs[pi];
  const int64_t local = tile - P.tile_begin;
  const int64_t ntn = (P.n + BN - 1) / BN;
  const int64_t m0 = (local / ntn) * BM;
  const int64_t n0 = (local % ntn) * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load_tiles = [&](int64_t k0) {
    // A tile: op(A)[m0:m0+64, k0:k0+16] -> ra (stored As[k][m])
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int e = tid + it * GEMM_THREADS;  // 0..1023
      int64_t i, p;
      if (P.transA) { i = e & 63; p = e >> 6; } else { p = e & 15; i = e >> 4; }
      int64_t gi = m0 + i, gp = k0 + p;
      double v = 0.0;
      if (gi < P.m && gp < P.k) v = P.transA ? P.A[gp * P.lda + gi] : P.A[gi * P.lda + gp];
      ra[it] = v;
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int e = tid + it * GEMM_THREADS;
      int64_t j, p;
      if (P.transB) { p = e & 15; j = e >> 4; } else { j = e & 63; p = e >> 6; }
      int64_t gj = n0 + j, gp = k0 + p;
      double v = 0.0;
      if (gj < P.n && gp < P.k) v = P.transB ? P.B[gj * P.ldb + gp] : P.B[gp * P.ldb + gj];
      rb[it] = v;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int e = tid + it * GEMM_THREADS;
      int i, p;
      if (P.transA) { i = e & 63; p = e >> 6; } else { p = e & 15; i = e >> 4; }
      As[buf][p][i] = ra[it];
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int e = tid + it * GEMM_THREADS;
      int j, p;
      if (P.transB) { p = e & 15; j = e >> 4; } else { j = e & 63; p = e >> 6; }
      Bs[buf][p][j] = rb[it];
    }
  };

  const int64_t nk = (P.k + BK - 1) / BK;
  if (nk > 0) {
    load_tiles(0);
    store_tiles(0);
    __syncthreads();
  }
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_tiles((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[buf][kk + (lane & 3)][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[buf][kk + (lane & 3)][wn * 32 + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    if (kt + 1 < nk) store_tiles(buf ^ 1);
    __syncthreads();
  }

  // epilogue: D = alpha*acc + beta*C
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    int64_t gi = m0 + wm * 32 + mi * 8 + (lane >> 2);
    if (gi >= P.m) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t gj = n0 + wn * 32 + ni * 8 + (lane & 3) * 2 + h;
        if (gj >= P.n) continue;
        double v = P.alpha * acc[mi][ni][h];
        if (P.beta != 0.0) v += P.beta * P.C[gi * P.ldc + gj];
        P.D[gi * P.ldd + gj] = v;
      }
    }
  }
}

int gemm_grouped(SkbGemm* probs, int64_t nprob, cudaStream_t s) {
  if (nprob <= 0) return 0;
  int64_t tiles = 0;
  double fl = 0.0;
  for (int64_t i = 0; i < nprob; ++i) {
    fl += 2.0 * (double)probs[i].m * (double)probs[i].n * (double)probs[i].k;
    probs[i].tile_begin = tiles;
    if (probs[i].m > 0 && probs[i].n > 0)
      tiles += ((probs[i].m + BM - 1) / BM) * ((probs[i].n + BN - 1) / BN);
  }
  if (tiles == 0) return 0;
  if (tiles > 0x7fffffff) return 3;
  SkbGemm* d = nullptr;
  int rc = upload(probs, nprob, s, &d);
  if (rc) return rc;
  {
    ProfScope ps(F_GEMM, s);
    k_gemm_grouped<<<(unsigned)tiles, GEMM_THREADS, 0, s>>>(d, (int)nprob);
  }
  if (prof().on) prof().flops[F_GEMM] += fl;
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(d, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // namespace skb

extern "C" int skb_gemm_grouped(SkbGemm* probs, int64_t nprob, void* stream) {
  return skb::gemm_grouped(probs, nprob, (cudaStream_t)stream);
}

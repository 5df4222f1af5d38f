// (c) Batched partially pivoted LU and LU solves (dgetrf / dgetrs semantics).
//
// Replaces the per-box PLU of reference dense.py:106-135 (sla.lu_factor /
// sla.lu_solve) for all X_RR blocks of a level at once, and the corner LU of
// _finish_top (skel.py:399-405).  Row-major storage; right-looking blocked
// algorithm, panel width 64: the panel (getf2) is one CTA per matrix, the
// U12 triangular solve is batched over (matrix, column chunk), the trailing
// update goes to the grouped DMMA GEMM.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace skb {

int gemm_grouped(SkbGemm* probs, int64_t nprob, cudaStream_t s);

constexpr int LB = 64;  // LU block width
#ifndef SKB_PANEL_NT
#define SKB_PANEL_NT 512    // threads of the panel CTA (1024: no gain at n=849)
#endif

struct LuPanel {
  double* A;
  int64_t n, ld, j0, jb;
  int32_t* ipiv;
  int32_t* info;
  int32_t* swp;   // [2*LB] destination rows (-1: skip), [2*LB] source rows, relative to j0
};

struct AbsMax {
  double v;
  int64_t idx;
};

__device__ __forceinline__ AbsMax absmax_merge(AbsMax a, AbsMax b) {
  return (b.v > a.v || (b.v == a.v && b.idx < a.idx)) ? b : a;
}

// Exact |max| with the lowest row index among ties, over a warp: max of the
// values, then the minimum index among the lanes holding it.
__device__ __forceinline__ void warp_absmax(double& v, int& idx) {
  double m = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  idx = __reduce_min_sync(0xffffffffu, v == m ? idx : INT_MAX);
  v = m;
}

// dgetf2 on the panel A[j0:n, j0:j0+jb], staged row-major in shared memory
// with an odd row length (pld = jb | 1: conflict-free 64-bit column scans and
// row sweeps).  A thread owns rows; it owns the same rows in the update of
// column c and the pivot search of column c+1, so a column costs two
// barriers.  The pivot row is copied to s_u with its entries at and left of
// column c zeroed, so the row update is one predicate-free sweep over 8-column
// groups (all loads of a group issue before its stores) followed by the
// multiplier store.  Then the panel's interchanges are composed into one
// permutation of the touched rows and applied to the columns outside the
// panel through a shared-memory stage (dlaswp with every load of a chunk in
// flight at once).
template <int NT>
__global__ void __launch_bounds__(NT) k_getf2_panel(const LuPanel* __restrict__ descs) {
  extern __shared__ __align__(16) double P[];
  constexpr int NW = NT / 32;
  __shared__ double red_v[NW];
  __shared__ int red_i[NW];
  __shared__ __align__(16) double s_u[LB + 8];
  __shared__ double s_pv;
  __shared__ int s_piv[LB];
  const LuPanel D = descs[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = (int)(D.n - D.j0);
  const int jb = (int)D.jb;
  const int pld = jb | 1;
  const int ng = (jb + 7) >> 3;                      // 8-column groups
  for (int t = threadIdx.x; t < LB + 8; t += NT) s_u[t] = 0.0;
  // global loads batched 8 rows deep per lane (one dependent round trip per batch)
  for (int cc = lane; cc < jb; cc += 32)
    for (int r0 = warp; r0 < rows; r0 += 8 * NW) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u * NW;
        if (r < rows) v[u] = D.A[(D.j0 + r) * D.ld + D.j0 + cc];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (r0 + u * NW < rows) P[(r0 + u * NW) * pld + cc] = v[u];
    }
  __syncthreads();
  int info = -1;
  for (int c = 0; c < jb; ++c) {
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = c + threadIdx.x; r < rows; r += NT) {
      const double v = fabs(P[r * pld + c]);
      if (v > bv) { bv = v; bi = r; }
    }
    warp_absmax(bv, bi);
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    double gv = lane < NW ? red_v[lane] : -1.0;
    int gi = lane < NW ? red_i[lane] : INT_MAX;
    warp_absmax(gv, gi);
    const int p = gi == INT_MAX ? c : gi;
    if (threadIdx.x == 0) {
      D.ipiv[D.j0 + c] = (int32_t)(D.j0 + p);
      s_piv[c] = p;
    }
    if (gv == 0.0) {       // |pivot| == 0: no interchange, no update
      if (info < 0) info = (int)(D.j0 + c);
      __syncthreads();     // red_* are rewritten by the next search
      continue;
    }
    if (threadIdx.x < jb) {   // pivot row -> s_u (left part zeroed), interchange rows c and p
      const int k = threadIdx.x;
      const double t = P[p * pld + k];
      s_u[k] = k > c ? t : 0.0;
      if (k == c) s_pv = t;
      if (p != c) {
        P[p * pld + k] = P[c * pld + k];
        P[c * pld + k] = t;
      }
    }
    __syncthreads();
    const double rinv = 1.0 / s_pv;
    const int g0 = c >> 3;
    for (int r = c + 1 + threadIdx.x; r < rows; r += NT) {
      double* pr = P + r * pld;
      const double l = pr[c] * rinv;
      for (int g = g0; g < ng; ++g) {
        double* q = pr + 8 * g;
        const double2* u2 = reinterpret_cast<const double2*>(s_u + 8 * g);
        double a[8];
        if (8 * g + 8 <= jb) {
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = q[k];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double2 u = u2[k];
            a[2 * k] = a[2 * k] - l * u.x;
            a[2 * k + 1] = a[2 * k + 1] - l * u.y;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) q[k] = a[k];
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) if (8 * g + k < jb) a[k] = q[k];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double2 u = u2[k];
            a[2 * k] = a[2 * k] - l * u.x;
            a[2 * k + 1] = a[2 * k + 1] - l * u.y;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) if (8 * g + k < jb) q[k] = a[k];
        }
      }
      pr[c] = l;
    }
  }
  __syncthreads();
  for (int r = warp; r < rows; r += NW) {
    double* dst = D.A + (D.j0 + r) * D.ld + D.j0;
    for (int cc = lane; cc < jb; cc += 32) dst[cc] = P[r * pld + cc];
  }
  if (threadIdx.x == 0 && info >= 0 && *D.info < 0) *D.info = info;
  // compose the interchanges (perm[d] = source row of destination d) into a
  // list of moved rows for k_laswp
  __syncthreads();
  int* perm = reinterpret_cast<int*>(P);
  for (int i = threadIdx.x; i < rows; i += NT) perm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int c = 0; c < jb; ++c) {
      const int q = s_piv[c];
      const int t = perm[c]; perm[c] = perm[q]; perm[q] = t;
    }
  __syncthreads();
  if (threadIdx.x < 2 * LB) {
    const int t = threadIdx.x;
    int d = -1, sr = 0;
    if (t < 2 * jb) {
      d = t < jb ? t : s_piv[t - jb];
      if ((t >= jb && d < jb) || perm[d] == d) d = -1;   // listed already / unmoved
      else sr = perm[d];
    }
    D.swp[t] = d;
    D.swp[2 * LB + t] = sr;
  }
}


// dgetf2 of one LB-wide panel on a thread-block cluster (large matrices: the
// tall panel does not fit one CTA's shared memory at LB columns).  Panel row r
// lives in CTA r % C (row-major, odd stride LB + 1).  Per column: local |max|
// search, cluster barrier, every CTA merges the C candidates (lowest row among
// equal maxima, as idamax) and pulls the pivot row (the owner of the pivot
// also pulls row c) through DSMEM, cluster barrier, then the owners write the
// interchange and every CTA scales / updates its rows (8 threads per row).
// Same per-row arithmetic as k_getf2_panel (l = a_rc * (1/piv),
// a_rk -= l u_k): results do not depend on which panel kernel ran.  Writes
// the moved-row lists for k_laswp like k_getf2_panel.  (A one-barrier variant
// publishing candidate rows in double-buffered slots measured 10-20 % slower:
// the column cost is instruction latency, not the second barrier.)
__global__ void __launch_bounds__(256) k_getf2_cl(const LuPanel* __restrict__ descs) {
  constexpr int NT = 256, NW = NT / 32, pld = LB + 1;
  extern __shared__ __align__(16) double P[];
  __shared__ double red_v[NW];
  __shared__ int red_i[NW];
  __shared__ double s_cand_v;
  __shared__ int s_cand_i;
  __shared__ double s_u[LB], s_rc[LB];
  __shared__ int s_piv[LB];
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
  const LuPanel D = descs[blockIdx.x / C];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = (int)(D.n - D.j0), jb = (int)D.jb;
  const int nloc = rows > me ? (rows - me + C - 1) / C : 0;     // my rows: me, me + C, ...
  for (int e = threadIdx.x; e < nloc * jb; e += NT) {
    const int lr = e / jb, k = e - lr * jb;
    P[lr * pld + k] = D.A[(D.j0 + (int64_t)lr * C + me) * D.ld + D.j0 + k];
  }
  __syncthreads();
  int info = -1;
  for (int c = 0; c < jb; ++c) {
    // local rows with global index >= c: lr >= ceil((c - me) / C)
    const int lr0 = c > me ? (c - me + C - 1) / C : 0;
    double bv = -1.0;
    int bi = INT_MAX;
    for (int lr = lr0 + threadIdx.x; lr < nloc; lr += NT) {
      const double v = fabs(P[lr * pld + c]);
      if (v > bv) { bv = v; bi = lr * C + me; }
    }
    warp_absmax(bv, bi);
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      double gv = lane < NW ? red_v[lane] : -1.0;
      int gi = lane < NW ? red_i[lane] : INT_MAX;
      warp_absmax(gv, gi);
      if (lane == 0) { s_cand_v = gv; s_cand_i = gi; }
    }
    cl.sync();                                             // candidates published
    double gv = -1.0;
    int gi = INT_MAX;
    if (lane < C) {
      gv = *cl.map_shared_rank(&s_cand_v, lane);
      gi = *cl.map_shared_rank(&s_cand_i, lane);
    }
    warp_absmax(gv, gi);                                   // every warp: the same merge
    const int p = gi == INT_MAX ? c : gi;
    const bool zero = !(gv > 0.0);
    if (me == 0 && threadIdx.x == 0) D.ipiv[D.j0 + c] = (int32_t)(D.j0 + p);
    if (threadIdx.x == 0) s_piv[c] = p;
    if (!zero && threadIdx.x < jb) {
      const int k = threadIdx.x;
      s_u[k] = cl.map_shared_rank(P, p % C)[(p / C) * pld + k];
      if (me == p % C && p != c) s_rc[k] = cl.map_shared_rank(P, c % C)[(c / C) * pld + k];
    }
    cl.sync();                                             // remote rows read
    if (zero) {
      if (info < 0) info = (int)(D.j0 + c);
      continue;
    }
    if (threadIdx.x < jb) {
      const int k = threadIdx.x;
      if (me == c % C) P[(c / C) * pld + k] = s_u[k];
      if (me == p % C && p != c) P[(p / C) * pld + k] = s_rc[k];
    }
    __syncthreads();
    const double rinv = 1.0 / s_u[c];
    const int lr1 = c + 1 > me ? (c + 1 - me + C - 1) / C : 0;   // rows > c
    for (int e = threadIdx.x; e < (nloc - lr1) * 8; e += NT) {
      // (row, 8-column group) work items, groups of one row on consecutive threads
      const int lr = lr1 + e / 8, g = e & 7;
      double* pr = P + lr * pld;
      const double l = pr[c] * rinv;
      for (int k = c + 1 + g; k < jb; k += 8) pr[k] = pr[k] - l * s_u[k];
    }
    __syncthreads();
    for (int lr = lr1 + threadIdx.x; lr < nloc; lr += NT) P[lr * pld + c] *= rinv;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nloc * jb; e += NT) {
    const int lr = e / jb, k = e - lr * jb;
    D.A[(D.j0 + (int64_t)lr * C + me) * D.ld + D.j0 + k] = P[lr * pld + k];
  }
  if (me == 0 && threadIdx.x == 0 && info >= 0 && *D.info < 0) *D.info = info;
  cl.sync();
  if (me != 0) return;
  // moved-row lists for k_laswp (rank 0), as k_getf2_panel
  __syncthreads();
  int* perm = reinterpret_cast<int*>(P);
  for (int i = threadIdx.x; i < rows; i += NT) perm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int c = 0; c < jb; ++c) {
      const int q = s_piv[c];
      const int t = perm[c]; perm[c] = perm[q]; perm[q] = t;
    }
  __syncthreads();
  if (threadIdx.x < 2 * LB) {
    const int t = threadIdx.x;
    int d = -1, sr = 0;
    if (t < 2 * jb) {
      d = t < jb ? t : s_piv[t - jb];
      if ((t >= jb && d < jb) || perm[d] == d) d = -1;
      else sr = perm[d];
    }
    D.swp[t] = d;
    D.swp[2 * LB + t] = sr;
  }
}

// dlaswp of one panel on the columns outside it: every CTA stages a 32-column
// tile of the moved rows (all loads in flight), then writes them to their
// destinations.  grid = (column tiles, matrices).
__global__ void __launch_bounds__(256) k_laswp(const LuPanel* __restrict__ descs) {
  const LuPanel D = descs[blockIdx.y];
  const int jb = (int)D.jb;
  const int ncol = (int)D.n - jb;
  const int k = blockIdx.x * 32 + (threadIdx.x & 31);
  if (blockIdx.x * 32 >= ncol) return;
  __shared__ int s_d[2 * LB], s_s[2 * LB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 2 * LB) {
    s_d[threadIdx.x] = D.swp[threadIdx.x];
    s_s[threadIdx.x] = D.swp[2 * LB + threadIdx.x];
  }
  __syncthreads();
  double* base = D.A + D.j0 * D.ld;
  const int g = k < D.j0 ? k : k + jb;
  const bool on = k < ncol;
  double v[2 * LB / 8];
#pragma unroll
  for (int u = 0; u < 2 * LB / 8; ++u) {
    const int t = warp + 8 * u;
    if (on && t < 2 * jb && s_d[t] >= 0) v[u] = base[(int64_t)s_s[t] * D.ld + g];
  }
  __syncthreads();   // every load of the tile precedes every store
#pragma unroll
  for (int u = 0; u < 2 * LB / 8; ++u) {
    const int t = warp + 8 * u;
    if (on && t < 2 * jb && s_d[t] >= 0) base[(int64_t)s_d[t] * D.ld + g] = v[u];
  }
  (void)lane;
}

// a / b from the reciprocal y = 1/b: one residual correction of a*y (the
// final step of the hardware-style division).  Keeps the upper solves free of
// the division slow-path call (which forced the x[] register block to spill);
// every upper solve uses it, so results do not depend on the kernel variant.
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q = a * y;
  return fma(fma(-b, q, a), y, q);
}

// In-place triangular solve of a jb-row block B (row-major, ldb) against the
// jb x jb diagonal block L (ldl) of an LU factor.  UPPER=false: unit lower,
// forward; UPPER=true: non-unit upper, backward.  One thread per column.
struct TrsmDesc {
  const double* L;
  int64_t ldl;
  double* B;
  int64_t ldb;
  int64_t jb, ncols;
};

template <bool UPPER, bool FULL>
__device__ __forceinline__ void trsm_col(const TrsmDesc& D, const double (*Ls)[LB + 1],
                                         const double* Linv, int jb, int64_t c) {
  double x[LB];
#pragma unroll
  for (int i = 0; i < LB; ++i)
    if (FULL || i < jb) x[i] = D.B[i * D.ldb + c];
  if (!UPPER) {
#pragma unroll
    for (int i = 1; i < LB; ++i) {
      if (!FULL && i >= jb) break;
      double s = x[i];
#pragma unroll
      for (int p = 0; p < LB; ++p)
        if (p < i) s -= Ls[i][p] * x[p];
      x[i] = s;
    }
  } else {
    // p descending: the same operation order as the warp-per-column variant
#pragma unroll
    for (int i = LB - 1; i >= 0; --i) {
      if (!FULL && i >= jb) continue;
      double s = x[i];
#pragma unroll
      for (int p = LB - 1; p > 0; --p)
        if (p > i && (FULL || p < jb)) s -= Ls[i][p] * x[p];
      x[i] = div_rcp(s, Ls[i][i], Linv[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < LB; ++i)
    if (FULL || i < jb) D.B[i * D.ldb + c] = x[i];
}

template <bool UPPER>
__global__ void __launch_bounds__(256) k_trsm_block(const TrsmDesc* __restrict__ descs) {
  __shared__ double Ls[LB][LB + 1];
  __shared__ double Linv[LB];
  const TrsmDesc D = descs[blockIdx.y];
  const int jb = (int)D.jb;
  for (int t = threadIdx.x; t < jb * jb; t += blockDim.x) {
    const int i = t / jb, p = t % jb;
    Ls[i][p] = D.L[i * D.ldl + p];
  }
  if (UPPER && threadIdx.x < jb) Linv[threadIdx.x] = 1.0 / D.L[threadIdx.x * D.ldl + threadIdx.x];
  __syncthreads();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= D.ncols) return;
  // full diagonal blocks (the common case) without the jb predicates
  if (jb == LB) trsm_col<UPPER, true>(D, Ls, Linv, LB, c);
  else trsm_col<UPPER, false>(D, Ls, Linv, jb, c);
}

// Narrow right-hand sides: one warp per column, lanes own rows (jb <= 64).
template <bool UPPER>
__global__ void __launch_bounds__(128) k_trsm_warp(const TrsmDesc* __restrict__ descs) {
  const TrsmDesc D = descs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (c >= D.ncols) return;
  const int jb = (int)D.jb;
  double x0 = lane < jb ? D.B[lane * D.ldb + c] : 0.0;
  double x1 = lane + 32 < jb ? D.B[(lane + 32) * D.ldb + c] : 0.0;
  if (!UPPER) {
    for (int p = 0; p < jb; ++p) {
      const double xp = __shfl_sync(0xffffffffu, p < 32 ? x0 : x1, p & 31);
      if (lane > p && lane < jb) x0 -= D.L[lane * D.ldl + p] * xp;
      if (lane + 32 > p && lane + 32 < jb) x1 -= D.L[(lane + 32) * D.ldl + p] * xp;
    }
  } else {
    for (int p = jb - 1; p >= 0; --p) {
      double xp = __shfl_sync(0xffffffffu, p < 32 ? x0 : x1, p & 31);
      const double d = D.L[p * D.ldl + p];
      xp = div_rcp(xp, d, 1.0 / d);
      if (lane == (p & 31)) { if (p < 32) x0 = xp; else x1 = xp; }
      if (lane < p) x0 -= D.L[lane * D.ldl + p] * xp;
      if (lane + 32 < p) x1 -= D.L[(lane + 32) * D.ldl + p] * xp;
    }
  }
  if (lane < jb) D.B[lane * D.ldb + c] = x0;
  if (lane + 32 < jb) D.B[(lane + 32) * D.ldb + c] = x1;
}

static int launch_trsm(std::vector<TrsmDesc>& td, bool upper, cudaStream_t s) {
  if (td.empty()) return 0;
  int64_t maxc = 0;
  for (auto& t : td) maxc = std::max(maxc, t.ncols);
  if (maxc == 0) return 0;
  TrsmDesc* d = nullptr;
  int rc = upload(td.data(), (int64_t)td.size(), s, &d);
  if (rc) return rc;
  ProfScope ps(F_TRSM, s);
  if (maxc <= 16) {
    for (int64_t b0 = 0; b0 < (int64_t)td.size(); b0 += 65535) {
      const int64_t nb = std::min<int64_t>(65535, (int64_t)td.size() - b0);
      dim3 grid((unsigned)((maxc + 3) / 4), (unsigned)nb);
      if (upper) k_trsm_warp<true><<<grid, 128, 0, s>>>(d + b0);
      else k_trsm_warp<false><<<grid, 128, 0, s>>>(d + b0);
    }
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(d, s);
    return e == cudaSuccess ? 0 : -(int)e;
  }
  for (int64_t b0 = 0; b0 < (int64_t)td.size(); b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, (int64_t)td.size() - b0);
    dim3 grid((unsigned)((maxc + 255) / 256), (unsigned)nb);
    if (upper) k_trsm_block<true><<<grid, 256, 0, s>>>(d + b0);
    else k_trsm_block<false><<<grid, 256, 0, s>>>(d + b0);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(d, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

struct RatioDesc {
  const double* A;
  int64_t n, ld;
};

__global__ void k_pivot_ratio(const RatioDesc* __restrict__ descs, double* __restrict__ out) {
  __shared__ double smin[256], smax[256];
  const RatioDesc D = descs[blockIdx.x];
  double mn = INFINITY, mx = 0.0;
  for (int64_t i = threadIdx.x; i < D.n; i += blockDim.x) {
    const double v = fabs(D.A[i * D.ld + i]);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + o]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = D.n == 0 ? 1.0 : smin[0] / smax[0];
}

// Whole-matrix LU in shared memory, one CTA per matrix (n <= kSmallLU):
// right-looking dgetf2 with the row swap applied to the full row.
constexpr int kSmallLU_ = 160;
static inline int64_t small_lu_max() {   // SKB_SMALL_LU: debug override of the one-CTA LU bound
  static const int64_t v = getenv("SKB_SMALL_LU") ? atoll(getenv("SKB_SMALL_LU")) : kSmallLU_;
  return v;
}
#define kSmallLU small_lu_max()

struct SmallLU {
  double* A;
  int64_t n, ld;
  int32_t* ipiv;
  int32_t* info;
};

template <int NT>
__global__ void __launch_bounds__(NT) k_getrf_small(const SmallLU* __restrict__ descs) {
  extern __shared__ double M[];
  __shared__ AbsMax red[NT / 32 + 1];
  const SmallLU D = descs[blockIdx.x];
  const int n = (int)D.n, L = n + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < n * n; t += NT) M[(t / n) * L + t % n] = D.A[(t / n) * D.ld + t % n];
  int info = -1;
  double prev_rinv = 0.0;   // multipliers of column j-1 are scaled lazily at step j
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    AbsMax loc{-1.0, INT64_MAX};
    for (int r = j + threadIdx.x; r < n; r += NT) {
      if (j > 0 && prev_rinv != 0.0) M[r * L + j - 1] *= prev_rinv;
      const double v = fabs(M[r * L + j]);
      if (v > loc.v) { loc.v = v; loc.idx = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      AbsMax y{__shfl_xor_sync(0xffffffffu, loc.v, o), __shfl_xor_sync(0xffffffffu, loc.idx, o)};
      loc = absmax_merge(loc, y);
    }
    if (lane == 0) red[warp] = loc;
    __syncthreads();
    AbsMax best = red[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) best = absmax_merge(best, red[w]);
    const int p = (int)best.idx;
    const double piv = M[p * L + j];
    if (threadIdx.x == 0) D.ipiv[j] = p;
    if (piv == 0.0) {
      if (info < 0) info = j;
      prev_rinv = 0.0;
      __syncthreads();
      continue;
    }
    // every thread has read the pivot before the row interchange moves it
    __syncthreads();
    if (p != j)
      for (int c = threadIdx.x; c < n; c += NT) {
        const double t = M[j * L + c]; M[j * L + c] = M[p * L + c]; M[p * L + c] = t;
      }
    __syncthreads();
    const double rinv = 1.0 / piv;
    prev_rinv = rinv;
    // rank-1 update of the trailing block, one thread per (row, 8-column chunk),
    // consecutive threads on consecutive rows (odd row stride: conflict-free);
    // the chunk's loads all issue before its stores.  Column j itself is only
    // read here and scaled at the next step
    const int rows = n - j - 1, cols = n - j - 1;
    const int cpr = cols > 0 ? (cols + 7) / 8 : 1;
    for (int e = threadIdx.x; e < rows * cpr; e += NT) {
      const int q = e / rows;
      const int r = j + 1 + (e - q * rows);
      const int c0 = j + 1 + q * 8;
      const double l = M[r * L + j] * rinv;
      double a[8], u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < n) { a[k] = M[r * L + c0 + k]; u[k] = M[j * L + c0 + k]; }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < n) M[r * L + c0 + k] = a[k] - l * u[k];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < n * n; t += NT) D.A[(t / n) * D.ld + t % n] = M[(t / n) * L + t % n];
  if (threadIdx.x == 0) *D.info = info;
}

int getrf_batched(int64_t nbox, const SkbMat* a, const int64_t* ipiv, int32_t* info_out,
                  double* ratio_out, cudaStream_t s) {
  if (nbox <= 0) return 0;
  SKB_RET(cudaMemsetAsync(info_out, 0xff, sizeof(int32_t) * nbox, s));
  int64_t max_n = 0, max_small = 0;
  std::vector<SmallLU> sl;
  for (int64_t b = 0; b < nbox; ++b) {
    if (a[b].rows <= 0) continue;
    if (a[b].rows <= kSmallLU) {
      sl.push_back(SmallLU{a[b].ptr, a[b].rows, a[b].ld, reinterpret_cast<int32_t*>(ipiv[b]),
                           info_out + b});
      max_small = std::max(max_small, a[b].rows);
    } else {
      max_n = std::max(max_n, a[b].rows);
    }
  }
  int rc = 0;
  if (!sl.empty()) {
    SmallLU* ds = nullptr;
    if ((rc = upload(sl.data(), (int64_t)sl.size(), s, &ds))) return rc;
    const size_t smem = sizeof(double) * (size_t)max_small * (max_small + 1);
    SKB_RET(smem_optin((const void*)k_getrf_small<256>));
    {
      ProfScope ps(F_GETRF, s);
      k_getrf_small<256><<<(unsigned)sl.size(), 256, smem, s>>>(ds);
    }
    SKB_LAUNCH_CHECK();
    cudaFreeAsync(ds, s);
  }
  std::vector<LuPanel> pd;
  std::vector<TrsmDesc> td;
  std::vector<SkbGemm> gd;
  // panel width: a function of each matrix's own order only (so results do not
  // depend on the batch composition): as wide as shared memory allows (<= 64)
  // (rows are stored with an odd stride PB + 1)
  // Panels taller than one CTA's shared memory at LB columns run on a
  // thread-block cluster (k_getf2_cl, identical per-row arithmetic); its size
  // is a function of n only.
  constexpr size_t kPanelSmem = 224 * 1024;
  auto one_cta = [&](int64_t n) { return (size_t)n * (LB / 2 + 1) * sizeof(double) <= kPanelSmem; };
  auto pbw = [&](int64_t n) {
    if (!one_cta(n)) return (int64_t)LB;
    return (size_t)n * (LB + 1) * sizeof(double) <= kPanelSmem ? (int64_t)LB : (int64_t)LB / 2;
  };
  static const int64_t lcmax = getenv("SKB_LU_CMAX") ? atoll(getenv("SKB_LU_CMAX")) : 16;
  auto csize = [&](int64_t n) {       // <= 100 KB of panel rows per CTA (200 KB at the cap)
    int64_t C = 2;
    while (C < lcmax && (size_t)((n + C - 1) / C) * (LB + 1) * sizeof(double) > 100 * 1024) C *= 2;
    return C;
  };
  int64_t rounds = 0;
  for (int64_t b = 0; b < nbox; ++b)
    if (a[b].rows > kSmallLU) rounds = std::max(rounds, (a[b].rows + pbw(a[b].rows) - 1) / pbw(a[b].rows));
  int32_t* swp = nullptr;   // moved-row lists of one round's panels (k_laswp)
  if (rounds > 0) {
    SKB_RET(smem_optin((const void*)k_getf2_panel<SKB_PANEL_NT>));
    SKB_RET(smem_optin((const void*)k_getf2_cl));
    SKB_RET(cudaFuncSetAttribute((const void*)k_getf2_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int64_t nbig = 0;
    for (int64_t b = 0; b < nbox; ++b) nbig += a[b].rows > kSmallLU;
    SKB_RET(cudaMallocAsync(reinterpret_cast<void**>(&swp), sizeof(int32_t) * 4 * LB * nbig, s));
  }
  // Look-ahead (SKB_LU_LOOKAHEAD=0 disables): the trailing update of each round
  // is split into the next panel's columns (main stream, so the next panel
  // starts right after them) and the rest (a side stream, overlapping the
  // next single-CTA panel); the next round's dlaswp joins the side stream.
  // Every element sees the same operations in the same order either way.
  static const bool lookahead = !getenv("SKB_LU_LOOKAHEAD") || atoi(getenv("SKB_LU_LOOKAHEAD")) != 0;
  std::vector<TrsmDesc> tdr;
  std::vector<SkbGemm> gdr;
  bool pending_rest = false;
  for (int64_t rd_ = 0; rd_ < rounds; ++rd_) {
    pd.clear(); td.clear(); gd.clear(); tdr.clear(); gdr.clear();
    size_t smem = 0;
    int64_t maxcol = 0;
    // panels: one-CTA ones first, then cluster ones grouped by cluster size
    std::vector<int64_t> order;
    for (int pass = 0; pass < 5; ++pass)
      for (int64_t b = 0; b < nbox; ++b) {
        const int64_t n = a[b].rows;
        if (n <= kSmallLU || rd_ * pbw(n) >= n) continue;
        const int grp = one_cta(n) ? 0 : (int)__builtin_ctzll((unsigned long long)csize(n));  // 1..4
        if (grp == pass) order.push_back(b);
      }
    int64_t ngrp[5] = {0, 0, 0, 0, 0};
    size_t csm[5] = {0, 0, 0, 0, 0};
    for (int64_t b : order) {
      const int64_t n = a[b].rows;
      const int64_t PB = pbw(n);
      const int64_t j0 = rd_ * PB;
      const int64_t jb = std::min<int64_t>(PB, n - j0), n2 = n - j0 - jb;
      const int grp = one_cta(n) ? 0 : (int)__builtin_ctzll((unsigned long long)csize(n));
      ngrp[grp]++;
      if (grp == 0) {
        smem = std::max(smem, sizeof(double) * (size_t)(n - j0) * (size_t)(PB + 1));
        smem = std::max(smem, sizeof(int) * (size_t)(n - j0));   // composed permutation
      } else {
        const int64_t C = csize(n);
        csm[grp] = std::max(csm[grp], sizeof(double) * (size_t)((n - j0 + C - 1) / C) * (LB + 1));
        csm[grp] = std::max(csm[grp], sizeof(int) * (size_t)(n - j0));
      }
      double* A = a[b].ptr;
      const int64_t ld = a[b].ld;
      pd.push_back(LuPanel{A, n, ld, j0, jb, reinterpret_cast<int32_t*>(ipiv[b]), info_out + b,
                           swp + (int64_t)pd.size() * 4 * LB});
      maxcol = std::max(maxcol, n - jb);
      if (n2 > 0) {
        // columns [j0+jb, j0+jb+w) on the main stream, the rest on the side stream
        // (only where the trailing update outweighs its extra launches: n >= 1536;
        // n = 2532: 27.1 -> 24.6 ms, n = 849: 3.02 -> 3.14 ms, so off there)
        const int64_t w = lookahead && n >= 1536 ? std::min<int64_t>(PB, n2) : n2;
        auto add = [&](int64_t c0, int64_t nc, std::vector<TrsmDesc>& T, std::vector<SkbGemm>& G) {
          T.push_back(TrsmDesc{A + j0 * ld + j0, ld, A + j0 * ld + c0, ld, jb, nc});
          SkbGemm g{};
          g.A = A + (j0 + jb) * ld + j0; g.lda = ld;           // L21: n2 x jb
          g.B = A + j0 * ld + c0; g.ldb = ld;                  // U12 columns: jb x nc
          g.C = A + (j0 + jb) * ld + c0; g.ldc = ld;           // A22 columns
          g.D = A + (j0 + jb) * ld + c0; g.ldd = ld;
          g.m = n2; g.n = nc; g.k = jb; g.alpha = -1.0; g.beta = 1.0;
          G.push_back(g);
        };
        add(j0 + jb, w, td, gd);
        if (n2 > w) add(j0 + jb + w, n2 - w, tdr, gdr);
      }
    }
    if (pd.empty()) continue;
    LuPanel* dp = nullptr;
    if ((rc = upload(pd.data(), (int64_t)pd.size(), s, &dp))) return rc;
    {
      ProfScope ps(F_GETRF, s);
      if (ngrp[0]) k_getf2_panel<SKB_PANEL_NT><<<(unsigned)ngrp[0], SKB_PANEL_NT, smem, s>>>(dp);
      SKB_LAUNCH_CHECK();
      int64_t off = ngrp[0];
      for (int g = 1; g < 5; ++g) {
        if (!ngrp[g]) continue;
        const int C = 1 << g;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(ngrp[g] * C));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = csm[g];
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SKB_RET(cudaLaunchKernelEx(&cfg, k_getf2_cl, (const LuPanel*)(dp + off)));
        off += ngrp[g];
      }
      // the interchanges touch the columns the side stream is still updating
      if (pending_rest) { SKB_RET((cudaError_t)(-join_n(s, 1))); pending_rest = false; }
      if (maxcol > 0) k_laswp<<<dim3((unsigned)((maxcol + 31) / 32), (unsigned)pd.size()), 256, 0, s>>>(dp);
    }
    SKB_LAUNCH_CHECK();
    cudaFreeAsync(dp, s);
    if (!tdr.empty()) {
      SKB_RET((cudaError_t)(-fork_n(s, 1)));
      cudaStream_t ss = side().st[0];
      if ((rc = launch_trsm(tdr, false, ss))) return rc;
      if ((rc = gemm_grouped(gdr.data(), (int64_t)gdr.size(), ss))) return rc;
      pending_rest = true;
    }
    if ((rc = launch_trsm(td, false, s))) return rc;
    if ((rc = gemm_grouped(gd.data(), (int64_t)gd.size(), s))) return rc;
  }
  if (pending_rest) SKB_RET((cudaError_t)(-join_n(s, 1)));
  if (swp) cudaFreeAsync(swp, s);
  std::vector<RatioDesc> rd(nbox);
  for (int64_t b = 0; b < nbox; ++b) rd[b] = RatioDesc{a[b].ptr, a[b].rows, a[b].ld};
  RatioDesc* dr = nullptr;
  if ((rc = upload(rd.data(), nbox, s, &dr))) return rc;
  k_pivot_ratio<<<(unsigned)nbox, 256, 0, s>>>(dr, ratio_out);
  SKB_LAUNCH_CHECK();
  cudaFreeAsync(dr, s);
  return 0;
}

struct SwapDesc {
  double* B;
  int64_t n, ld, ncols;
  const int32_t* ipiv;
};

// Narrow B: compose the interchanges into a permutation (one thread per
// matrix), then gather rows in parallel through a scratch copy.
__global__ void k_ipiv_perm(const SwapDesc* __restrict__ descs, int32_t* __restrict__ perm,
                            const int64_t* __restrict__ poff) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const SwapDesc D = descs[b];
  int32_t* p = perm + poff[b];
  for (int64_t i = 0; i < D.n; ++i) p[i] = (int32_t)i;
  for (int64_t i = 0; i < D.n; ++i) {
    const int64_t q = D.ipiv[i];
    if (q != i) { const int32_t t = p[i]; p[i] = p[q]; p[q] = t; }
  }
}

// The same composition with ipiv and the permutation in shared memory (one
// warp per matrix; lane 0 walks the interchanges): ~50 ns per interchange
// instead of a global-memory round trip (the 2532-row corner: 0.8 -> 0.15 ms).
__global__ void k_ipiv_perm_smem(const SwapDesc* __restrict__ descs, int32_t* __restrict__ perm,
                                 const int64_t* __restrict__ poff) {
  extern __shared__ int32_t sp[];
  const SwapDesc D = descs[blockIdx.x];
  const int n = (int)D.n;
  int32_t* piv = sp;
  int32_t* p = sp + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { piv[i] = D.ipiv[i]; p[i] = i; }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < n; ++i) {
      const int q = piv[i];
      if (q != i) { const int32_t t = p[i]; p[i] = p[q]; p[q] = t; }
    }
  __syncthreads();
  int32_t* out = perm + poff[blockIdx.x];
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = p[i];
}

// rows of a matrix over the blocks (x), consecutive threads on consecutive columns
__global__ void k_perm_rows(const SwapDesc* __restrict__ descs, const int32_t* __restrict__ perm,
                            const int64_t* __restrict__ poff, double* __restrict__ tmp,
                            const int64_t* __restrict__ toff, int phase) {
  const SwapDesc D = descs[blockIdx.y];
  const int32_t* p = perm + poff[blockIdx.y];
  double* t = tmp + toff[blockIdx.y];
  const int n = (int)D.n, nc = (int)D.ncols;
  const int tpr = nc > 128 ? 256 : (nc > 64 ? 128 : (nc > 32 ? 64 : 32)), rps = 256 / tpr;
  const int tr = threadIdx.x / tpr, tc = threadIdx.x - tr * tpr;
  for (int i = blockIdx.x * rps + tr; i < n; i += gridDim.x * rps) {
    const int src = p[i];
    if (src == i) continue;                       // unmoved row: nothing to do in either phase
    if (phase == 0) {
      const double* sp_ = D.B + (int64_t)src * D.ld;
      double* dp = t + (int64_t)i * nc;
      for (int c = tc; c < nc; c += tpr) dp[c] = sp_[c];
    } else {
      const double* sp_ = t + (int64_t)i * nc;
      double* dp = D.B + (int64_t)i * D.ld;
      for (int c = tc; c < nc; c += tpr) dp[c] = sp_[c];
    }
  }
}

__global__ void k_apply_ipiv(const SwapDesc* __restrict__ descs) {
  const SwapDesc D = descs[blockIdx.y];
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= D.ncols) return;
  for (int64_t i = 0; i < D.n; ++i) {
    const int64_t p = D.ipiv[i];
    if (p != i) {
      const double t = D.B[i * D.ld + c];
      D.B[i * D.ld + c] = D.B[p * D.ld + c];
      D.B[p * D.ld + c] = t;
    }
  }
}

// B <- L^-1 B (unit lower, forward) for a batch, blocked: diagonal blocks by
// substitution, off-diagonal blocks on the grouped GEMM.
int trsm_lower_unit_batched(int64_t nbox, const SkbMat* lu, const SkbMat* b, cudaStream_t s) {
  int64_t max_n = 0;
  for (int64_t i = 0; i < nbox; ++i)
    if (b[i].cols > 0) max_n = std::max(max_n, lu[i].rows);
  std::vector<TrsmDesc> td;
  std::vector<SkbGemm> gd;
  int rc = 0;
  for (int64_t j0 = 0; j0 < max_n; j0 += LB) {
    td.clear(); gd.clear();
    for (int64_t i = 0; i < nbox; ++i) {
      const int64_t n = lu[i].rows, nc = b[i].cols;
      if (j0 >= n || nc == 0) continue;
      const int64_t jb = std::min<int64_t>(LB, n - j0), n2 = n - j0 - jb;
      const double* L = lu[i].ptr;
      const int64_t ldl = lu[i].ld, ldb = b[i].ld;
      td.push_back(TrsmDesc{L + j0 * ldl + j0, ldl, b[i].ptr + j0 * ldb, ldb, jb, nc});
      if (n2 > 0) {
        SkbGemm g{};
        g.A = L + (j0 + jb) * ldl + j0; g.lda = ldl;
        g.B = b[i].ptr + j0 * ldb; g.ldb = ldb;
        g.C = b[i].ptr + (j0 + jb) * ldb; g.ldc = ldb;
        g.D = b[i].ptr + (j0 + jb) * ldb; g.ldd = ldb;
        g.m = n2; g.n = nc; g.k = jb; g.alpha = -1.0; g.beta = 1.0;
        gd.push_back(g);
      }
    }
    if ((rc = launch_trsm(td, false, s))) return rc;
    if ((rc = gemm_grouped(gd.data(), (int64_t)gd.size(), s))) return rc;
  }
  return 0;
}

// B <- U^-1 B (non-unit upper, backward), blocked.  Only the upper triangle of
// U is read.  Also computes T = R11^-1 R12 of the ID (dense.py:77).
int trsm_upper_batched(int64_t nbox, const SkbMat* u, const SkbMat* b, cudaStream_t s) {
  int64_t max_n = 0;
  for (int64_t i = 0; i < nbox; ++i)
    if (b[i].cols > 0) max_n = std::max(max_n, u[i].rows);
  if (max_n == 0) return 0;
  std::vector<TrsmDesc> td;
  std::vector<SkbGemm> gd;
  int rc = 0;
  for (int64_t j0 = ((max_n - 1) / LB) * LB; j0 >= 0; j0 -= LB) {
    td.clear(); gd.clear();
    for (int64_t i = 0; i < nbox; ++i) {
      const int64_t n = u[i].rows, nc = b[i].cols;
      if (j0 >= n || nc == 0) continue;
      const int64_t jb = std::min<int64_t>(LB, n - j0);
      const double* U = u[i].ptr;
      const int64_t ldu = u[i].ld, ldb = b[i].ld;
      td.push_back(TrsmDesc{U + j0 * ldu + j0, ldu, b[i].ptr + j0 * ldb, ldb, jb, nc});
      if (j0 > 0) {
        SkbGemm g{};
        g.A = U + j0; g.lda = ldu;                  // U[0:j0, j0:j0+jb]
        g.B = b[i].ptr + j0 * ldb; g.ldb = ldb;
        g.C = b[i].ptr; g.ldc = ldb;
        g.D = b[i].ptr; g.ldd = ldb;
        g.m = j0; g.n = nc; g.k = jb; g.alpha = -1.0; g.beta = 1.0;
        gd.push_back(g);
      }
    }
    if ((rc = launch_trsm(td, true, s))) return rc;
    if ((rc = gemm_grouped(gd.data(), (int64_t)gd.size(), s))) return rc;
  }
  return 0;
}

int getrs_batched(int64_t nbox, const SkbMat* lu, const int64_t* ipiv, const SkbMat* b,
                  cudaStream_t s) {
  if (nbox <= 0) return 0;
  int64_t max_c = 0;
  std::vector<SwapDesc> sd;
  for (int64_t i = 0; i < nbox; ++i) {
    if (lu[i].rows == 0 || b[i].cols == 0) continue;
    max_c = std::max(max_c, b[i].cols);
    sd.push_back(SwapDesc{b[i].ptr, lu[i].rows, b[i].ld, b[i].cols,
                          reinterpret_cast<const int32_t*>(ipiv[i])});
  }
  if (sd.empty()) return 0;
  int rc = 0;
  int64_t max_rows = 0;
  for (const SwapDesc& q : sd) max_rows = std::max(max_rows, q.n);
  // SKB_IPIV_PERM_MIN: tall matrices (the corner, top-level boxes) also go
  // through the composed permutation (pure data movement: same bits)
  static const int64_t perm_min = getenv("SKB_IPIV_PERM_MIN") ? atoll(getenv("SKB_IPIV_PERM_MIN")) : 512;
  const bool smem_perm = max_rows <= 5500;
  if (max_c <= 8 || (max_rows >= perm_min && smem_perm)) {
    // narrow or tall: permutation gather
    std::vector<int64_t> poff(sd.size()), toff(sd.size());
    int64_t pt = 0, tt = 0, maxe = 0;
    for (size_t i = 0; i < sd.size(); ++i) {
      poff[i] = pt; pt += sd[i].n;
      toff[i] = tt; tt += sd[i].n * sd[i].ncols;
      maxe = std::max(maxe, sd[i].n * sd[i].ncols);
    }
    SwapDesc* d = nullptr;
    int64_t *dpo = nullptr, *dto = nullptr;
    int32_t* perm = nullptr;
    double* tmp = nullptr;
    if ((rc = upload(sd.data(), (int64_t)sd.size(), s, &d))) return rc;
    if ((rc = upload(poff.data(), (int64_t)poff.size(), s, &dpo))) return rc;
    if ((rc = upload(toff.data(), (int64_t)toff.size(), s, &dto))) return rc;
    SKB_RET(malloc_async((void**)&perm, sizeof(int32_t) * std::max<int64_t>(pt, 1), s));
    SKB_RET(malloc_async((void**)&tmp, sizeof(double) * std::max<int64_t>(tt, 1), s));
    {
      ProfScope ps(F_TRSM, s);
      const int64_t nbx = (int64_t)sd.size();
      // one thread per matrix (exact multiple of the block via guard-free launch of 1-thread blocks)
      if (smem_perm && nbx <= 65535)
        k_ipiv_perm_smem<<<(unsigned)nbx, 128, sizeof(int32_t) * 2 * (size_t)max_rows, s>>>(d, perm, dpo);
      else
        k_ipiv_perm<<<(unsigned)nbx, 1, 0, s>>>(d, perm, dpo);
      for (int64_t b0 = 0; b0 < nbx; b0 += 65535) {
        const int64_t nb = std::min<int64_t>(65535, nbx - b0);
        dim3 grid(grid_cap(max_rows, nb > 64 ? 64 : 1024), (unsigned)nb);
        k_perm_rows<<<grid, 256, 0, s>>>(d + b0, perm, dpo + b0, tmp, dto + b0, 0);
        k_perm_rows<<<grid, 256, 0, s>>>(d + b0, perm, dpo + b0, tmp, dto + b0, 1);
      }
    }
    SKB_LAUNCH_CHECK();
    cudaFreeAsync(d, s);
    cudaFreeAsync(dpo, s);
    cudaFreeAsync(dto, s);
    cudaFreeAsync(perm, s);
    cudaFreeAsync(tmp, s);
  } else {
    SwapDesc* d = nullptr;
    if ((rc = upload(sd.data(), (int64_t)sd.size(), s, &d))) return rc;
    for (int64_t b0 = 0; b0 < (int64_t)sd.size(); b0 += 65535) {
      const int64_t nb = std::min<int64_t>(65535, (int64_t)sd.size() - b0);
      dim3 grid((unsigned)((max_c + 127) / 128), (unsigned)nb);
      ProfScope ps(F_TRSM, s);
      k_apply_ipiv<<<grid, 128, 0, s>>>(d + b0);
    }
    SKB_LAUNCH_CHECK();
    cudaFreeAsync(d, s);
  }
  if ((rc = trsm_lower_unit_batched(nbox, lu, b, s))) return rc;
  return trsm_upper_batched(nbox, lu, b, s);
}

}  // namespace skb

extern "C" int skb_getrf_batched(int64_t nbox, const SkbMat* a, const int64_t* ipiv,
                                 int32_t* info_out, double* ratio_out, void* stream) {
  return skb::getrf_batched(nbox, a, ipiv, info_out, ratio_out, (cudaStream_t)stream);
}

extern "C" int skb_getrs_batched(int64_t nbox, const SkbMat* lu, const int64_t* ipiv,
                                 const SkbMat* b, void* stream) {
  return skb::getrs_batched(nbox, lu, ipiv, b, (cudaStream_t)stream);
}

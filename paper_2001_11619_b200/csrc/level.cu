// Level-granular host orchestration: one C-ABI call per quadtree level for the
// Schur-complement stage (c) and for the augmentation sweep (d), replacing the
// per-box NumPy/LAPACK sequences of compress_box (skel.py:316-338) and
// _finish_top (skel.py:384-396).  The descriptor arithmetic (offsets, GEMM
// problem lists, the deterministic Schur accumulation order) runs here in C++;
// every floating-point operation runs in the batched kernels it enqueues.

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace skb {

int gemm_grouped(SkbGemm* probs, int64_t nprob, cudaStream_t s);

namespace {

inline SkbGemm G(const double* A, const double* B, const double* C, double* D, int64_t m, int64_t n,
                 int64_t k, int64_t lda, int64_t ldb, int64_t ldc, int64_t ldd, double alpha,
                 double beta, int transA = 0, int transB = 0) {
  SkbGemm g{};
  g.A = A; g.B = B; g.C = C; g.D = D;
  g.m = m; g.n = n; g.k = k;
  g.lda = lda; g.ldb = ldb; g.ldc = ldc; g.ldd = ldd;
  g.alpha = alpha; g.beta = beta;
  g.transA = transA; g.transB = transB;
  return g;
}

inline double* P(uint64_t a) { return reinterpret_cast<double*>(a); }

// one H2D upload of several int64 host arrays; returns device base, offsets in elements
struct Packed {
  std::vector<int64_t> host;
  std::vector<size_t> at;
  size_t add(const int64_t* a, size_t n) {
    const size_t o = host.size();
    host.insert(host.end(), a, a + n);
    at.push_back(o);
    return o;
  }
};

}  // namespace

}  // namespace skb

using namespace skb;

extern "C" int skb_level_schur(int64_t nbox, const int64_t* nB, const int64_t* k,
                               const int64_t* act_off, const double* pos, const double* nrm,
                               const double* w, const double* kappa, const int64_t* act_off_dev,
                               const int64_t* act_dev, const int32_t* perm_dev, const int64_t* A,
                               const int64_t* lda, const int64_t* child_off,
                               const uint64_t* child_xss, const uint64_t* T, const uint64_t* Xrr,
                               const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                               const uint64_t* Xss, const uint64_t* ipiv, int32_t* info_dev,
                               double* ratio_dev, int32_t pde, void* stream) {
  if (nbox <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = nbox;
  std::vector<int64_t> r(B), E_off(B + 1, 0), X_off(B + 1, 0), perm_ptr(B), ldE(B);
  int64_t maxn = 0;
  for (int64_t b = 0; b < B; ++b) {
    r[b] = nB[b] - k[b];
    E_off[b + 1] = E_off[b] + nB[b] * nB[b];
    X_off[b + 1] = X_off[b] + r[b] * k[b];
    perm_ptr[b] = (int64_t)(perm_dev + act_off[b]);
    ldE[b] = nB[b];
    maxn = std::max(maxn, nB[b]);
  }
  double* Ebuf = nullptr;
  double* Xrs = nullptr;
  SKB_RET(malloc_async((void**)&Ebuf, sizeof(double) * std::max<int64_t>(E_off[B], 1), s));
  SKB_RET(malloc_async((void**)&Xrs, sizeof(double) * std::max<int64_t>(X_off[B], 1), s));
  int rc;
  // T = R11^-1 R12 (dense.py:77)
  if ((rc = skb_id_T_batched(B, A, lda, k, nB, perm_ptr.data(), (const int64_t*)T, s))) return rc;
  // permuted self blocks with the children's Xss (skel.py:282-291, 316)
  Packed pk;
  pk.add(child_off, 5 * B);
  pk.add((const int64_t*)child_xss, 4 * B);   // four children per box
  pk.add(E_off.data(), B);
  pk.add(ldE.data(), B);
  int64_t* dpk = nullptr;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &dpk))) return rc;
  if ((rc = (pde == 1 ? skb_assemble_self_lap : skb_assemble_self)(
           pos, nrm, w, kappa, B, act_off_dev, act_dev, act_off_dev, perm_dev, dpk + pk.at[0],
           dpk + pk.at[1], Ebuf, dpk + pk.at[2], dpk + pk.at[3], maxn, s)))
    return rc;
  // X_sr = E_SR - E_SS T ; X_rs = E_RS - T^T E_SS ; X_rr = E_RR - E_RS T (skel.py:321-332)
  // problem order as in the Python restatement: [all X_sr | all X_rs | all X_rr]
  std::vector<SkbGemm> g1(3 * B), g2, g3;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t n = nB[b], kk = k[b], rr = r[b];
    double* E = Ebuf + E_off[b];
    double *Ess = E, *Esr = E + kk, *Ers = E + kk * n, *Err = Ers + kk;
    double* Xrsb = Xrs + X_off[b];
    g1[b] = G(Ess, P(T[b]), Esr, P(Xsr[b]), kk, rr, kk, n, rr, n, rr, -1.0, 1.0);
    g1[B + b] = G(P(T[b]), Ess, Ers, Xrsb, rr, kk, kk, rr, n, n, kk, -1.0, 1.0, 1);
    g1[2 * B + b] = G(Ers, P(T[b]), Err, P(Xrr[b]), rr, rr, kk, n, rr, n, rr, -1.0, 1.0);
    // X_rr -= T^T X_sr
    g2.push_back(G(P(T[b]), P(Xsr[b]), P(Xrr[b]), P(Xrr[b]), rr, rr, kk, rr, rr, rr, rr, -1.0, 1.0, 1));
    // Xss_mod = E_SS - X_sr X_rs_div (skel.py:334)
    g3.push_back(G(P(Xsr[b]), P(Xrsdiv[b]), Ess, P(Xss[b]), kk, kk, rr, rr, kk, n, kk, -1.0, 1.0));
  }
  if ((rc = gemm_grouped(g1.data(), (int64_t)g1.size(), s))) return rc;
  if ((rc = gemm_grouped(g2.data(), (int64_t)g2.size(), s))) return rc;
  // LU(X_rr) (skel.py:324) and X_rs_div = X_rr^-1 X_rs (skel.py:333)
  std::vector<SkbMat> mLU(B), mXrr(B), mDiv(B), mXrs(B);
  for (int64_t b = 0; b < B; ++b) {
    mLU[b] = SkbMat{P(LU[b]), r[b], r[b], r[b]};
    mXrr[b] = SkbMat{P(Xrr[b]), r[b], r[b], r[b]};
    mDiv[b] = SkbMat{P(Xrsdiv[b]), r[b], k[b], k[b]};
    mXrs[b] = SkbMat{Xrs + X_off[b], r[b], k[b], k[b]};
  }
  if ((rc = skb_copy2d_batched(B, mLU.data(), mXrr.data(), 0, s))) return rc;
  if ((rc = skb_getrf_batched(B, mLU.data(), (const int64_t*)ipiv, info_dev, ratio_dev, s))) return rc;
  if ((rc = skb_copy2d_batched(B, mDiv.data(), mXrs.data(), 0, s))) return rc;
  if ((rc = skb_getrs_batched(B, mLU.data(), (const int64_t*)ipiv, mDiv.data(), s))) return rc;
  if ((rc = gemm_grouped(g3.data(), (int64_t)g3.size(), s))) return rc;
  cudaFreeAsync(dpk, s);
  cudaFreeAsync(Ebuf, s);
  cudaFreeAsync(Xrs, s);
  return 0;
}

// Deterministic Schur accumulation of one level's parts (skel.py:396): rows
// of the q x q corner block in column order, box order kept within a row.
static int schur_acc_level(int64_t B, const int64_t* nc, const int64_t* cols_off, const int64_t* cols,
                           int64_t q, const double* part_base, const int64_t* part_off, double* schur,
                           cudaStream_t s) {
  const int64_t ncol = cols_off[B];
  if (ncol == 0) return 0;
  std::vector<int64_t> row_off(q + 1, 0), contrib(ncol);
  for (int64_t t = 0; t < ncol; ++t) row_off[cols[t] + 1]++;
  for (int64_t i = 0; i < q; ++i) row_off[i + 1] += row_off[i];
  std::vector<int64_t> fill(row_off.begin(), row_off.end() - 1);
  for (int64_t b = 0; b < B; ++b)
    for (int64_t j = 0; j < nc[b]; ++j) {
      const int64_t row = cols[cols_off[b] + j];
      contrib[fill[row]++] = part_off[b] + j * q;
    }
  Packed pk;
  pk.add(row_off.data(), q + 1);
  pk.add(contrib.data(), ncol);
  int64_t* d = nullptr;
  int rc;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &d))) return rc;
  rc = skb_schur_accumulate(q, d + pk.at[0], d + pk.at[1], part_base, schur, s);
  cudaFreeAsync(d, s);
  return rc;
}

// U sweep on H / V^T sweep on Psi for the boxes of one level (skel.py:384-396).
// stash (optional): per-box persistent storage of the box's outgoing skeleton
// rows UH_S (k x q at st_us[b]) and PsiV_S (k x nc at st_ps[b]) and of its
// Schur part PsiV_R^T w (nc x q at st_sp[b]) -- what a later update() needs
// to resume the sweep above clean boxes.  acc = 0 leaves the accumulation of
// the parts into schur to the caller (skb_level_schur_acc).
extern "C" int skb_level_aug(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                             const int64_t* cols_off, const int64_t* cols, const int64_t* sd_off,
                             const int64_t* sd, const int64_t* rd_off, const int64_t* rd,
                             const int64_t* c_off, const int64_t* c, const uint64_t* T,
                             const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                             const uint64_t* ipiv, double* UH, double* PsiV, double* UH_div,
                             double* schur, double* stash, const int64_t* st_us,
                             const int64_t* st_ps, const int64_t* st_sp, int32_t acc, void* stream) {
  if (nbox <= 0 || q <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = nbox;
  std::vector<int64_t> nc(B);
  for (int64_t b = 0; b < B; ++b) nc[b] = cols_off[b + 1] - cols_off[b];
  // scratch: Ur (r q) | w (r q) | Pr (r c) [| Us (k q) | Ps (k c) | Sp (c q) without a stash]
  std::vector<int64_t> oUs(B), oUr(B), oW(B), oPs(B), oPr(B), oSp(B), ldq(B, q);
  int64_t tUs = 0, tUr = 0, tPs = 0, tPr = 0, tSp = 0;
  int64_t mk = 0, mr = 0, mc = 0;
  for (int64_t b = 0; b < B; ++b) {
    oUs[b] = tUs; tUs += k[b] * q;
    oUr[b] = tUr; tUr += r[b] * q;
    oPs[b] = tPs; tPs += k[b] * nc[b];
    oPr[b] = tPr; tPr += r[b] * nc[b];
    oSp[b] = tSp; tSp += nc[b] * q;
    mk = std::max(mk, k[b]); mr = std::max(mr, r[b]); mc = std::max(mc, nc[b]);
  }
  const int64_t bUr = 0, bW = tUr, bPr = 2 * tUr, bUs = bPr + tPr, bPs = bUs + tUs, bSp = bPs + tPs;
  const int64_t total = stash ? bUs : bSp + tSp;
  for (int64_t b = 0; b < B; ++b) {
    oW[b] = oUr[b] + bW; oUr[b] += bUr; oPr[b] += bPr;
    if (stash) { oUs[b] = st_us[b]; oPs[b] = st_ps[b]; oSp[b] = st_sp[b]; }
    else { oUs[b] += bUs; oPs[b] += bPs; oSp[b] += bSp; }
  }
  double* buf = nullptr;
  SKB_RET(malloc_async((void**)&buf, sizeof(double) * std::max<int64_t>(total, 1), s));
  double* sbase = stash ? stash : buf;          // Us / Ps / Sp live here
  Packed pk;
  pk.add(oUs.data(), B); pk.add(oUr.data(), B); pk.add(oW.data(), B);
  pk.add(oPs.data(), B); pk.add(oPr.data(), B); pk.add(ldq.data(), B); pk.add(nc.data(), B);
  int64_t* d = nullptr;
  int rc;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &d))) return rc;
  const int64_t *dUs = d + pk.at[0], *dUr = d + pk.at[1], *dW = d + pk.at[2], *dPs = d + pk.at[3],
                *dPr = d + pk.at[4], *dldq = d + pk.at[5], *dldc = d + pk.at[6];
  // gathers (skel.py:385-392 row selections)
  if ((rc = skb_gather_rows(B, sd_off, sd, nullptr, nullptr, q, UH, q, sbase, dUs, dldq, mk, q, s))) return rc;
  if ((rc = skb_gather_rows(B, rd_off, rd, nullptr, nullptr, q, UH, q, buf, dUr, dldq, mr, q, s))) return rc;
  if (mc) {
    if ((rc = skb_gather_rows(B, sd_off, sd, c_off, c, 0, PsiV, q, sbase, dPs, dldc, mk, mc, s))) return rc;
    if ((rc = skb_gather_rows(B, rd_off, rd, c_off, c, 0, PsiV, q, buf, dPr, dldc, mr, mc, s))) return rc;
  }
  // UH_R -= T^T UH_S ; PsiV_R -= T^T PsiV_S
  std::vector<SkbGemm> g1(2 * B), g2(3 * B);
  std::vector<SkbMat> mW(B), mUr(B), mLU(B);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t kk = k[b], rr = r[b], cc = nc[b];
    double *Us = sbase + oUs[b], *Ur = buf + oUr[b], *Wb = buf + oW[b], *Ps = sbase + oPs[b],
           *Pr = buf + oPr[b], *Sp = sbase + oSp[b];
    g1[b] = G(P(T[b]), Us, Ur, Ur, rr, q, kk, rr, q, q, q, -1.0, 1.0, 1);
    g1[B + b] = G(P(T[b]), Ps, Pr, Pr, rr, cc, kk, rr, cc, cc, cc, -1.0, 1.0, 1);
    mW[b] = SkbMat{Wb, rr, q, q};
    mUr[b] = SkbMat{Ur, rr, q, q};
    mLU[b] = SkbMat{P(LU[b]), rr, rr, rr};
    // UH_S -= X_sr w ; PsiV_S -= X_rs_div^T PsiV_R ; schur part = PsiV_R^T w
    g2[b] = G(P(Xsr[b]), Wb, Us, Us, kk, q, rr, rr, q, q, q, -1.0, 1.0);
    g2[B + b] = G(P(Xrsdiv[b]), Pr, Ps, Ps, kk, cc, rr, kk, cc, cc, cc, -1.0, 1.0, 1);
    g2[2 * B + b] = G(Pr, Wb, nullptr, Sp, cc, q, rr, cc, q, 0, q, 1.0, 0.0, 1);
  }
  if ((rc = gemm_grouped(g1.data(), (int64_t)g1.size(), s))) return rc;
  // w = X_rr^-1 UH_R (skel.py:390)
  if ((rc = skb_copy2d_batched(B, mW.data(), mUr.data(), 0, s))) return rc;
  if ((rc = skb_getrs_batched(B, mLU.data(), (const int64_t*)ipiv, mW.data(), s))) return rc;
  if ((rc = gemm_grouped(g2.data(), (int64_t)g2.size(), s))) return rc;
  // scatters back (skel.py:391-395)
  if ((rc = skb_scatter_rows(B, rd_off, rd, nullptr, nullptr, q, buf, dUr, dldq, UH, q, 0, 1.0, mr, q, s))) return rc;
  if ((rc = skb_scatter_rows(B, sd_off, sd, nullptr, nullptr, q, sbase, dUs, dldq, UH, q, 0, 1.0, mk, q, s))) return rc;
  if ((rc = skb_scatter_rows(B, rd_off, rd, nullptr, nullptr, q, buf, dW, dldq, UH_div, q, 0, 1.0, mr, q, s))) return rc;
  if (mc) {
    if ((rc = skb_scatter_rows(B, rd_off, rd, c_off, c, 0, buf, dPr, dldc, PsiV, q, 0, 1.0, mr, mc, s))) return rc;
    if ((rc = skb_scatter_rows(B, sd_off, sd, c_off, c, 0, sbase, dPs, dldc, PsiV, q, 0, 1.0, mk, mc, s))) return rc;
    if (acc && (rc = schur_acc_level(B, nc.data(), cols_off, cols, q, sbase, oSp.data(), schur, s))) return rc;
  }
  cudaFreeAsync(d, s);
  cudaFreeAsync(buf, s);
  return 0;
}

// Accumulate one level's stored Schur parts into schur (skel.py:396), in the
// order skb_level_aug(acc = 1) uses.
extern "C" int skb_level_schur_acc(int64_t nbox, const int64_t* cols_off, const int64_t* cols,
                                   int64_t q, const double* stash, const int64_t* st_sp,
                                   double* schur, void* stream) {
  if (nbox <= 0 || q <= 0) return 0;
  std::vector<int64_t> nc(nbox);
  for (int64_t b = 0; b < nbox; ++b) nc[b] = cols_off[b + 1] - cols_off[b];
  return schur_acc_level(nbox, nc.data(), cols_off, cols, q, stash, st_sp, schur, (cudaStream_t)stream);
}

namespace skb_lvl {

// dst[dst_off[b] + i * ld + qc[j]] = src[src_off[b] + i * nqc + j], i < rows[b]
__global__ void k_put_cols(const int64_t* __restrict__ rows, const int64_t* __restrict__ src_off,
                           const int64_t* __restrict__ dst_off, const int64_t* __restrict__ qc,
                           int64_t nqc, int64_t ld, const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t b = blockIdx.y;
  const int64_t n = rows[b] * nqc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nqc, j = t - i * nqc;
    dst[dst_off[b] + i * ld + qc[j]] = src[src_off[b] + i * nqc + j];
  }
}

// UH[sd[i]][j] = us_b[i * q + j] for the columns with qmask[j] == 0 and
// PsiV[sd[i]][cols_b[t]] = ps_b[i * nc_b + t]: a clean box's outgoing
// skeleton rows, stored at its own sweep step, for a dirty parent.
__global__ void k_restore_rows(const int64_t* __restrict__ sd_off, const int64_t* __restrict__ sd,
                               const int64_t* __restrict__ c_off, const int64_t* __restrict__ c,
                               const uint64_t* __restrict__ us, const uint64_t* __restrict__ ps,
                               const uint8_t* __restrict__ qmask, int64_t q,
                               double* __restrict__ UH, double* __restrict__ PsiV) {
  const int64_t b = blockIdx.y;
  const int64_t i0 = sd_off[b], kk = sd_off[b + 1] - i0;
  const int64_t c0 = c_off[b], nc = c_off[b + 1] - c0;
  const double* u = reinterpret_cast<const double*>(us[b]);
  const double* pv = reinterpret_cast<const double*>(ps[b]);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < kk * q; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / q, j = t - i * q;
    if (!qmask[j]) UH[sd[i0 + i] * q + j] = u[i * q + j];
  }
  // the whole PsiV row: the box's hole columns from its stored rows, zero
  // elsewhere (the old parent's step mixed sibling holes into these rows)
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < kk * q; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / q, j = t - i * q;
    double val = 0.0;
    for (int64_t u = 0; u < nc; ++u)
      if (c[c0 + u] == j) val = pv[i * nc + u];
    PsiV[sd[i0 + i] * q + j] = val;
  }
}

__global__ void k_copy_rows(const int64_t* __restrict__ idx, int64_t n, int64_t ncols,
                            const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * ncols; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncols, j = t - i * ncols;
    dst[idx[i] * ncols + j] = src[idx[i] * ncols + j];
  }
}

__global__ void k_copy_cols(const int64_t* __restrict__ qc, int64_t nqc, int64_t nrows, int64_t ld,
                            const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows * nqc; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nqc, j = t - i * nqc;
    dst[i * ld + qc[j]] = src[i * ld + qc[j]];
  }
}

}  // namespace skb_lvl

using namespace skb_lvl;

// The augmentation sweep of a level restricted to the columns qc (3 per moved
// hole) for boxes whose factors did not change (update(), incremental
// _finish_top): UH / UH_div rows of the box at those columns, the stored
// outgoing UH_S at those columns and the Schur part's columns qc
// (PsiV_R = the box's final PsiV rows, unchanged).  The same kernels as
// skb_level_aug restricted to columns: bitwise the full sweep's values there.
extern "C" int skb_level_aug_narrow(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                                    int64_t nqc, const int64_t* qc, const int64_t* cols_off,
                                    const int64_t* sd_off, const int64_t* sd, const int64_t* rd_off,
                                    const int64_t* rd, const int64_t* c_off, const int64_t* c,
                                    const uint64_t* T, const uint64_t* LU, const uint64_t* Xsr,
                                    const uint64_t* ipiv, double* UH, const double* PsiV, double* UH_div,
                                    double* stash, const int64_t* st_us, const int64_t* st_sp,
                                    void* stream) {
  if (nbox <= 0 || q <= 0 || nqc <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = nbox;
  std::vector<int64_t> nc(B), oUs(B), oUr(B), oW(B), oPr(B), oSp(B), ldn(B, nqc), qoff(B + 1);
  int64_t t1 = 0, t2 = 0, t3 = 0, t4 = 0, mk = 0, mr = 0, mc = 0, tot_sp = 0;
  for (int64_t b = 0; b < B; ++b) {
    nc[b] = cols_off[b + 1] - cols_off[b];
    oUs[b] = t1; t1 += k[b] * nqc;
    oUr[b] = t2; t2 += r[b] * nqc;
    oPr[b] = t3; t3 += r[b] * nc[b];
    oSp[b] = t4; t4 += nc[b] * nqc;
    qoff[b] = b * nqc;
    mk = std::max(mk, k[b]); mr = std::max(mr, r[b]); mc = std::max(mc, nc[b]);
    tot_sp += nc[b];
  }
  qoff[B] = B * nqc;
  const int64_t bUs = 0, bUr = t1, bW = t1 + t2, bPr = t1 + 2 * t2, bSp = bPr + t3, total = bSp + t4;
  for (int64_t b = 0; b < B; ++b) {
    oW[b] = oUr[b] + bW; oUs[b] += bUs; oUr[b] += bUr; oPr[b] += bPr; oSp[b] += bSp;
  }
  double* buf = nullptr;
  SKB_RET(malloc_async((void**)&buf, sizeof(double) * std::max<int64_t>(total, 1), s));
  // per-box column lists = qc for every box
  std::vector<int64_t> qcl;
  qcl.reserve(B * nqc);
  for (int64_t b = 0; b < B; ++b) qcl.insert(qcl.end(), qc, qc + nqc);
  Packed pk;
  pk.add(oUs.data(), B); pk.add(oUr.data(), B); pk.add(oW.data(), B); pk.add(oPr.data(), B);
  pk.add(oSp.data(), B); pk.add(ldn.data(), B); pk.add(nc.data(), B); pk.add(qoff.data(), B + 1);
  pk.add(qcl.data(), (size_t)(B * nqc)); pk.add(k, B); pk.add(r, B); pk.add(st_us, B); pk.add(st_sp, B);
  int64_t* d = nullptr;
  int rc;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &d))) return rc;
  const int64_t *dUs = d + pk.at[0], *dUr = d + pk.at[1], *dW = d + pk.at[2], *dPr = d + pk.at[3],
                *dSp = d + pk.at[4], *dldn = d + pk.at[5], *dldc = d + pk.at[6], *dqoff = d + pk.at[7],
                *dqcl = d + pk.at[8], *dk = d + pk.at[9], *dr = d + pk.at[10], *dstus = d + pk.at[11],
                *dstsp = d + pk.at[12];
  if ((rc = skb_gather_rows(B, sd_off, sd, dqoff, dqcl, 0, UH, q, buf, dUs, dldn, mk, nqc, s))) return rc;
  if ((rc = skb_gather_rows(B, rd_off, rd, dqoff, dqcl, 0, UH, q, buf, dUr, dldn, mr, nqc, s))) return rc;
  if (mc && (rc = skb_gather_rows(B, rd_off, rd, c_off, c, 0, const_cast<double*>(PsiV), q, buf, dPr, dldc, mr, mc, s)))
    return rc;
  std::vector<SkbGemm> g1(B), g2(2 * B);
  std::vector<SkbMat> mW(B), mUr(B), mLU(B);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t kk = k[b], rr = r[b], cc = nc[b];
    double *Us = buf + oUs[b], *Ur = buf + oUr[b], *Wb = buf + oW[b], *Pr = buf + oPr[b], *Sp = buf + oSp[b];
    g1[b] = G(P(T[b]), Us, Ur, Ur, rr, nqc, kk, rr, nqc, nqc, nqc, -1.0, 1.0, 1);
    mW[b] = SkbMat{Wb, rr, nqc, nqc};
    mUr[b] = SkbMat{Ur, rr, nqc, nqc};
    mLU[b] = SkbMat{P(LU[b]), rr, rr, rr};
    g2[b] = G(P(Xsr[b]), Wb, Us, Us, kk, nqc, rr, rr, nqc, nqc, nqc, -1.0, 1.0);
    g2[B + b] = G(Pr, Wb, nullptr, Sp, cc, nqc, rr, cc, nqc, 0, nqc, 1.0, 0.0, 1);
  }
  if ((rc = gemm_grouped(g1.data(), (int64_t)g1.size(), s))) return rc;
  if ((rc = skb_copy2d_batched(B, mW.data(), mUr.data(), 0, s))) return rc;
  if ((rc = skb_getrs_batched(B, mLU.data(), (const int64_t*)ipiv, mW.data(), s))) return rc;
  if ((rc = gemm_grouped(g2.data(), (int64_t)g2.size(), s))) return rc;
  if ((rc = skb_scatter_rows(B, rd_off, rd, dqoff, dqcl, 0, buf, dUr, dldn, UH, q, 0, 1.0, mr, nqc, s))) return rc;
  if ((rc = skb_scatter_rows(B, sd_off, sd, dqoff, dqcl, 0, buf, dUs, dldn, UH, q, 0, 1.0, mk, nqc, s))) return rc;
  if ((rc = skb_scatter_rows(B, rd_off, rd, dqoff, dqcl, 0, buf, dW, dldn, UH_div, q, 0, 1.0, mr, nqc, s))) return rc;
  // stored outgoing UH_S and Schur parts, columns qc
  {
    dim3 grid(grid_cap((mk * nqc + 255) / 256, 256), (unsigned)B);
    k_put_cols<<<grid, 256, 0, s>>>(dk, dUs, dstus, dqcl, nqc, q, buf, stash);
    if (mc) {
      dim3 g2d(grid_cap((mc * nqc + 255) / 256, 256), (unsigned)B);
      k_put_cols<<<g2d, 256, 0, s>>>(dldc, dSp, dstsp, dqcl, nqc, q, buf, stash);
    }
  }
  cudaError_t e = cudaGetLastError();
  (void)dr; (void)tot_sp;
  cudaFreeAsync(d, s);
  cudaFreeAsync(buf, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

// Clean boxes with a dirty parent: their stored outgoing skeleton rows back
// into UH (columns with qmask 0) and PsiV (the box's hole columns).
extern "C" int skb_restore_rows(int64_t nbox, const int64_t* sd_off, const int64_t* sd, int64_t max_k,
                                const int64_t* c_off, const int64_t* c, const uint64_t* us,
                                const uint64_t* ps, const uint8_t* qmask_dev, int64_t q, double* UH,
                                double* PsiV, void* stream) {
  if (nbox <= 0 || q <= 0 || max_k <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t* d = nullptr;
  std::vector<uint64_t> pp(2 * nbox);
  for (int64_t b = 0; b < nbox; ++b) { pp[b] = us[b]; pp[nbox + b] = ps[b]; }
  int rc;
  if ((rc = upload(pp.data(), 2 * nbox, s, &d))) return rc;
  dim3 grid(grid_cap((max_k * q + 255) / 256, 256), (unsigned)nbox);
  k_restore_rows<<<grid, 256, 0, s>>>(sd_off, sd, c_off, c, d, d + nbox, qmask_dev, q, UH, PsiV);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(d, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

// dst[idx[i]][:] = src[idx[i]][:] (n rows of ncols), and dst[:, qc[j]] = src[:, qc[j]].
extern "C" int skb_copy_rows_cols(int64_t n, const int64_t* idx_dev, int64_t nqc, const int64_t* qc_dev,
                                  int64_t nrows, int64_t ncols, const double* src, double* dst,
                                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n > 0) k_copy_rows<<<grid_cap((n * ncols + 255) / 256, 4096), 256, 0, s>>>(idx_dev, n, ncols, src, dst);
  if (nqc > 0)
    k_copy_cols<<<grid_cap((nrows * nqc + 255) / 256, 4096), 256, 0, s>>>(qc_dev, nqc, nrows, ncols, src, dst);
  SKB_LAUNCH_CHECK();
  return 0;
}

// One level of the incremental augmentation sweep of update() in one call
// (SURVEY.md §8(f) row 3): the per-level work of _AugPipeUpdate without the
// Python bookkeeping.  Host inputs describe every box of the level (new tree
// order): sizes, hole columns, skeleton / redundant DOF lists, factor
// pointers, dirty[b], parent_dirty[b] and, for reused boxes, the addresses of
// their stored rows / parts in the previous factorization (old_us/ps/sp).
//   reused boxes: copy stored rows / parts -> narrow sweep on the moved
//                 columns qc -> (dirty parent) restore outgoing rows;
//   dirty boxes : full sweep into the new stash, no accumulation;
//   then the level's Schur parts are accumulated in the refactor's order.
extern "C" int skb_level_aug_update(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                                    const int64_t* cols_off, const int64_t* cols,
                                    const int64_t* sd_off, const int64_t* sd, const int64_t* rd_off,
                                    const int64_t* rd, const uint8_t* dirty, const uint8_t* parent_dirty,
                                    const uint64_t* T, const uint64_t* LU, const uint64_t* Xsr,
                                    const uint64_t* Xrsdiv, const uint64_t* ipiv, const uint64_t* old_us,
                                    const uint64_t* old_ps, const uint64_t* old_sp, int64_t nqc,
                                    const int64_t* qc, const uint8_t* qmask_dev, double* UH, double* PsiV,
                                    double* UH_div, double* schur, double* stash, const int64_t* st_us,
                                    const int64_t* st_ps, const int64_t* st_sp, void* stream) {
  if (nbox <= 0 || q <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = nbox;
  std::vector<int64_t> cl, dr, rs;
  for (int64_t b = 0; b < B; ++b) {
    if (dirty[b]) dr.push_back(b);
    else {
      cl.push_back(b);
      if (parent_dirty[b]) rs.push_back(b);
    }
  }
  // subset CSR lists (sd, rd, hole columns) of the three box sets, one upload
  struct Sub {
    std::vector<int64_t> sdo, sdv, rdo, rdv, co, cv;
    size_t a_sdo, a_sdv, a_rdo, a_rdv, a_co, a_cv;
  };
  auto build = [&](const std::vector<int64_t>& sel, Sub& S) {
    S.sdo.assign(1, 0); S.rdo.assign(1, 0); S.co.assign(1, 0);
    for (int64_t b : sel) {
      S.sdv.insert(S.sdv.end(), sd + sd_off[b], sd + sd_off[b + 1]);
      S.rdv.insert(S.rdv.end(), rd + rd_off[b], rd + rd_off[b + 1]);
      S.cv.insert(S.cv.end(), cols + cols_off[b], cols + cols_off[b + 1]);
      S.sdo.push_back((int64_t)S.sdv.size());
      S.rdo.push_back((int64_t)S.rdv.size());
      S.co.push_back((int64_t)S.cv.size());
    }
    if (S.sdv.empty()) S.sdv.push_back(0);
    if (S.rdv.empty()) S.rdv.push_back(0);
    if (S.cv.empty()) S.cv.push_back(0);
  };
  Sub Sc, Sd, Sr;
  build(cl, Sc); build(dr, Sd); build(rs, Sr);
  Packed pk;
  for (Sub* S : {&Sc, &Sd, &Sr}) {
    S->a_sdo = pk.add(S->sdo.data(), S->sdo.size()); S->a_sdv = pk.add(S->sdv.data(), S->sdv.size());
    S->a_rdo = pk.add(S->rdo.data(), S->rdo.size()); S->a_rdv = pk.add(S->rdv.data(), S->rdv.size());
    S->a_co = pk.add(S->co.data(), S->co.size()); S->a_cv = pk.add(S->cv.data(), S->cv.size());
  }
  int64_t* d = nullptr;
  int rc;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &d))) return rc;
  auto pick = [](const std::vector<int64_t>& sel, auto* arr) {
    std::vector<std::remove_const_t<std::remove_pointer_t<decltype(arr)>>> out(sel.size());
    for (size_t i = 0; i < sel.size(); ++i) out[i] = arr[sel[i]];
    return out;
  };
  if (!cl.empty()) {
    const int64_t C = (int64_t)cl.size();
    // copy the reused boxes' stored rows / parts into the new stash
    std::vector<SkbMat> dst, src;
    for (int64_t b : cl) {
      const int64_t nc = cols_off[b + 1] - cols_off[b];
      const int64_t n3[3] = {k[b] * q, k[b] * nc, nc * q};
      const int64_t so[3] = {st_us[b], st_ps[b], st_sp[b]};
      const uint64_t oo[3] = {old_us[b], old_ps[b], old_sp[b]};
      for (int w = 0; w < 3; ++w)
        if (n3[w] > 0) {
          dst.push_back(SkbMat{stash + so[w], 1, n3[w], n3[w]});
          src.push_back(SkbMat{reinterpret_cast<double*>(oo[w]), 1, n3[w], n3[w]});
        }
    }
    if (!dst.empty() && (rc = skb_copy2d_batched((int64_t)dst.size(), dst.data(), src.data(), 0, s))) return rc;
    if (nqc > 0) {
      auto kc = pick(cl, k), rc_ = pick(cl, r), stu = pick(cl, st_us), sts = pick(cl, st_sp);
      auto Tc = pick(cl, T), LUc = pick(cl, LU), Xc = pick(cl, Xsr), Ic = pick(cl, ipiv);
      if ((rc = skb_level_aug_narrow(C, kc.data(), rc_.data(), q, nqc, qc, Sc.co.data(), d + Sc.a_sdo,
                                     d + Sc.a_sdv, d + Sc.a_rdo, d + Sc.a_rdv, d + Sc.a_co, d + Sc.a_cv,
                                     Tc.data(), LUc.data(), Xc.data(), Ic.data(), UH, PsiV, UH_div, stash,
                                     stu.data(), sts.data(), s)))
        return rc;
    }
    if (!rs.empty()) {
      std::vector<uint64_t> us(rs.size()), ps(rs.size());
      int64_t mk = 0;
      for (size_t i = 0; i < rs.size(); ++i) {
        us[i] = (uint64_t)(stash + st_us[rs[i]]);
        ps[i] = (uint64_t)(stash + st_ps[rs[i]]);
        mk = std::max(mk, k[rs[i]]);
      }
      if ((rc = skb_restore_rows((int64_t)rs.size(), d + Sr.a_sdo, d + Sr.a_sdv, mk, d + Sr.a_co,
                                 d + Sr.a_cv, us.data(), ps.data(), qmask_dev, q, UH, PsiV, s)))
        return rc;
    }
  }
  if (!dr.empty()) {
    auto kd = pick(dr, k), rd_ = pick(dr, r), stu = pick(dr, st_us), stp = pick(dr, st_ps),
         sts = pick(dr, st_sp);
    auto Td = pick(dr, T), LUd = pick(dr, LU), Xd = pick(dr, Xsr), Vd = pick(dr, Xrsdiv), Id = pick(dr, ipiv);
    if ((rc = skb_level_aug((int64_t)dr.size(), kd.data(), rd_.data(), q, Sd.co.data(), Sd.cv.data(),
                            d + Sd.a_sdo, d + Sd.a_sdv, d + Sd.a_rdo, d + Sd.a_rdv, d + Sd.a_co,
                            d + Sd.a_cv, Td.data(), LUd.data(), Xd.data(), Vd.data(), Id.data(), UH, PsiV,
                            UH_div, schur, stash, stu.data(), stp.data(), sts.data(), 0, s)))
      return rc;
  }
  rc = skb_level_schur_acc(B, cols_off, cols, q, stash, st_sp, schur, s);
  cudaFreeAsync(d, s);
  return rc;
}

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
                               double* ratio_dev, void* stream) {
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
  pk.add((const int64_t*)child_xss, 5 * B);
  pk.add(E_off.data(), B);
  pk.add(ldE.data(), B);
  int64_t* dpk = nullptr;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &dpk))) return rc;
  if ((rc = skb_assemble_self(pos, nrm, w, kappa, B, act_off_dev, act_dev, act_off_dev, perm_dev,
                              dpk + pk.at[0], dpk + pk.at[1], Ebuf, dpk + pk.at[2], dpk + pk.at[3],
                              maxn, s)))
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

extern "C" int skb_level_aug(int64_t nbox, const int64_t* k, const int64_t* r, int64_t q,
                             const int64_t* cols_off, const int64_t* cols, const int64_t* sd_off,
                             const int64_t* sd, const int64_t* rd_off, const int64_t* rd,
                             const int64_t* c_off, const int64_t* c, const uint64_t* T,
                             const uint64_t* LU, const uint64_t* Xsr, const uint64_t* Xrsdiv,
                             const uint64_t* ipiv, double* UH, double* PsiV, double* UH_div,
                             double* schur, void* stream) {
  if (nbox <= 0 || q <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = nbox;
  std::vector<int64_t> nc(B);
  for (int64_t b = 0; b < B; ++b) nc[b] = cols_off[b + 1] - cols_off[b];
  // scratch regions: Us (k q) | Ur (r q) | w (r q) | Ps (k c) | Pr (r c) | Sp (c q)
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
  const int64_t bUs = 0, bUr = tUs, bW = bUr + tUr, bPs = bW + tUr, bPr = bPs + tPs, bSp = bPr + tPr;
  const int64_t total = bSp + tSp;
  for (int64_t b = 0; b < B; ++b) {
    oUs[b] += bUs; oUr[b] += bUr; oW[b] = oUr[b] - bUr + bW; oPs[b] += bPs; oPr[b] += bPr;
    oSp[b] += bSp;
  }
  double* buf = nullptr;
  SKB_RET(malloc_async((void**)&buf, sizeof(double) * std::max<int64_t>(total, 1), s));
  // deterministic schur accumulation order: contributions grouped by corner
  // row, box order kept (stable), skel.py:396
  const int64_t ncol = cols_off[B];
  std::vector<int64_t> row_off(q + 1, 0), contrib(ncol);
  for (int64_t t = 0; t < ncol; ++t) row_off[cols[t] + 1]++;
  for (int64_t i = 0; i < q; ++i) row_off[i + 1] += row_off[i];
  {
    std::vector<int64_t> fill(row_off.begin(), row_off.end() - 1);
    for (int64_t b = 0; b < B; ++b)
      for (int64_t j = 0; j < nc[b]; ++j) {
        const int64_t row = cols[cols_off[b] + j];
        contrib[fill[row]++] = oSp[b] + j * q;
      }
  }
  Packed pk;
  pk.add(oUs.data(), B); pk.add(oUr.data(), B); pk.add(oW.data(), B);
  pk.add(oPs.data(), B); pk.add(oPr.data(), B); pk.add(ldq.data(), B); pk.add(nc.data(), B);
  pk.add(row_off.data(), q + 1);
  if (ncol) pk.add(contrib.data(), ncol);
  int64_t* d = nullptr;
  int rc;
  if ((rc = upload(pk.host.data(), (int64_t)pk.host.size(), s, &d))) return rc;
  const int64_t *dUs = d + pk.at[0], *dUr = d + pk.at[1], *dW = d + pk.at[2], *dPs = d + pk.at[3],
                *dPr = d + pk.at[4], *dldq = d + pk.at[5], *dldc = d + pk.at[6],
                *drow = d + pk.at[7];
  const int64_t* dct = ncol ? d + pk.at[8] : nullptr;
  // gathers (skel.py:385-392 row selections)
  if ((rc = skb_gather_rows(B, sd_off, sd, nullptr, nullptr, q, UH, q, buf, dUs, dldq, mk, q, s))) return rc;
  if ((rc = skb_gather_rows(B, rd_off, rd, nullptr, nullptr, q, UH, q, buf, dUr, dldq, mr, q, s))) return rc;
  if (mc) {
    if ((rc = skb_gather_rows(B, sd_off, sd, c_off, c, 0, PsiV, q, buf, dPs, dldc, mk, mc, s))) return rc;
    if ((rc = skb_gather_rows(B, rd_off, rd, c_off, c, 0, PsiV, q, buf, dPr, dldc, mr, mc, s))) return rc;
  }
  // UH_R -= T^T UH_S ; PsiV_R -= T^T PsiV_S
  std::vector<SkbGemm> g1(2 * B), g2(3 * B);
  std::vector<SkbMat> mW(B), mUr(B), mLU(B);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t kk = k[b], rr = r[b], cc = nc[b];
    double *Us = buf + oUs[b], *Ur = buf + oUr[b], *Wb = buf + oW[b], *Ps = buf + oPs[b],
           *Pr = buf + oPr[b], *Sp = buf + oSp[b];
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
  if ((rc = skb_scatter_rows(B, sd_off, sd, nullptr, nullptr, q, buf, dUs, dldq, UH, q, 0, 1.0, mk, q, s))) return rc;
  if ((rc = skb_scatter_rows(B, rd_off, rd, nullptr, nullptr, q, buf, dW, dldq, UH_div, q, 0, 1.0, mr, q, s))) return rc;
  if (mc) {
    if ((rc = skb_scatter_rows(B, rd_off, rd, c_off, c, 0, buf, dPr, dldc, PsiV, q, 0, 1.0, mr, mc, s))) return rc;
    if ((rc = skb_scatter_rows(B, sd_off, sd, c_off, c, 0, buf, dPs, dldc, PsiV, q, 0, 1.0, mk, mc, s))) return rc;
    if ((rc = skb_schur_accumulate(q, drow, dct, buf, schur, s))) return rc;
  }
  cudaFreeAsync(d, s);
  cudaFreeAsync(buf, s);
  return 0;
}

// (a) Level-batched Stokes kernel-matrix assembly.
//
// Compiled with -fmad=false: every entry is evaluated with NumPy's operation
// order and per-operation rounding (reference kernels.py), so ID stacks and
// self blocks match the CPU reference bitwise except entries containing log()
// (Stokeslet proxy rows, H columns), which agree to ~1 ulp.
#include "common.cuh"

namespace skb {

#define SKB_PI 3.141592653589793  // np.pi

struct Geo {
  const double2* pos;
  const double2* nrm;
  const double* w;
};

__device__ __forceinline__ double comp(double2 v, int c) { return c == 0 ? v.x : v.y; }

// One thread per (box column j, item t); items: [0,nF) far pairs, [nF,nF+P)
// proxy points, nF+P the nullspace-capture rows.  Column-major output so the
// item index (fastest) walks down a column.
__global__ void k_assemble_stack(Geo g, const int64_t* __restrict__ act_off,
                                 const int64_t* __restrict__ act,
                                 const int64_t* __restrict__ far_off,
                                 const int64_t* __restrict__ far,
                                 const double2* __restrict__ ppts,
                                 const double2* __restrict__ pnrm,
                                 const double* __restrict__ pw, int P,
                                 const int64_t* __restrict__ stack_off,
                                 double* __restrict__ stack) {
  const int64_t b = blockIdx.y;
  const int64_t a0 = act_off[b], nB = act_off[b + 1] - a0;
  const int64_t f0 = far_off[b], nF = far_off[b + 1] - f0;
  const int64_t items = nF + P + 1;
  const int64_t rows = 2 * nF + 6 * (int64_t)P + 2;
  double* S = stack + stack_off[b];
  const double pwb = pw[b];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < items * nB;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / items, it = t - j * items;
    const int64_t bd = act[a0 + j];
    const int64_t nb = bd >> 1;
    const int cb = (int)(bd & 1);
    const double2 pb = g.pos[nb], nbv = g.nrm[nb];
    const double wb = g.w[nb];
    double* col = S + j * rows;
    if (it < nF) {
      const int64_t fd = far[f0 + it];
      const int64_t nf = fd >> 1;
      const int cf = (int)(fd & 1);
      const double2 pf = g.pos[nf], nfv = g.nrm[nf];
      const double rx = pf.x - pb.x, ry = pf.y - pb.y;
      const double r2 = rx * rx + ry * ry;
      const double rdn_b = rx * nbv.x + ry * nbv.y;
      const double rdn_f = rx * nfv.x + ry * nfv.y;
      const double ir4 = 1.0 / ((SKB_PI * r2) * r2);
      const double rr = (cf == 0 ? rx : ry) * (cb == 0 ? rx : ry);
      const double nsp = comp(nfv, cf) * comp(nbv, cb);
      col[it] = ((rdn_b * ir4) * rr + nsp) * wb;
      col[nF + 2 * P + 1 + it] = (((-rdn_f) * ir4) * rr + nsp) * g.w[nf];
    } else if (it < nF + P) {
      const int p = (int)(it - nF);
      const double2 pp = ppts[b * P + p];
      const double2 pn = pnrm[b * P + p];
      // incoming: proxy target, box source (stresslet, kernels.py:279-290,307-321)
      {
        const double rx = pp.x - pb.x, ry = pp.y - pb.y;
        const double r2 = rx * rx + ry * ry;
        const double coef = (rx * nbv.x + ry * nbv.y) / ((SKB_PI * r2) * r2);
        const double rs = cb == 0 ? rx : ry;
        col[nF + 2 * p] = ((coef * rx) * rs) * wb;
        col[nF + 2 * p + 1] = ((coef * ry) * rs) * wb;
      }
      // outgoing: box target, proxy source (kernels.py:328-346)
      {
        const double rx = pb.x - pp.x, ry = pb.y - pp.y;
        const double r2 = rx * rx + ry * ry;
        const double coef = (rx * pn.x + ry * pn.y) / ((SKB_PI * r2) * r2);
        const double rt = cb == 0 ? rx : ry;
        const int64_t base1 = 2 * nF + 2 * (int64_t)P + 1;
        col[base1 + 2 * p] = ((coef * rt) * rx) * pwb;
        col[base1 + 2 * p + 1] = ((coef * rt) * ry) * pwb;
        const double lg = -0.5 * log(r2);
        const double pref = 1.0 / (4.0 * SKB_PI);
        const int64_t base2 = base1 + 2 * (int64_t)P;
        double v0, v1;
        if (cb == 0) {
          v0 = pref * (lg + (rx * rx) / r2);
          v1 = pref * ((rx * ry) / r2);
        } else {
          v0 = pref * ((ry * rx) / r2);
          v1 = pref * (lg + (ry * ry) / r2);
        }
        col[base2 + 2 * p] = v0 * pwb;
        col[base2 + 2 * p + 1] = v1 * pwb;
      }
    } else {
      const double nc = comp(nbv, cb);
      col[nF + 2 * P] = wb * nc;
      col[rows - 1] = nc;
    }
  }
}

// Self block in permuted order with children's Xss blocks (skel.py:282-291).
__global__ void k_assemble_self(Geo g, const double* __restrict__ kappa,
                                const int64_t* __restrict__ act_off,
                                const int64_t* __restrict__ act,
                                const int64_t* __restrict__ perm_off,
                                const int32_t* __restrict__ perm,
                                const int64_t* __restrict__ child_off,
                                const int64_t* __restrict__ child_xss, double* __restrict__ E,
                                const int64_t* __restrict__ E_off,
                                const int64_t* __restrict__ E_ld) {
  const int64_t b = blockIdx.y;
  const int64_t a0 = act_off[b], n = act_off[b + 1] - a0;
  const int64_t* co = child_off + 5 * b;
  const int64_t ld = E_ld[b];
  double* Eb = E + E_off[b];
  const int32_t* pm = perm ? perm + perm_off[b] : nullptr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    const int64_t pi = pm ? pm[i] : i, pj = pm ? pm[j] : j;
    int ci = -1, cj = -1;
    if (co[0] >= 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (co[c + 1] < 0) break;
        if (pi >= co[c] && pi < co[c + 1]) ci = c;
        if (pj >= co[c] && pj < co[c + 1]) cj = c;
      }
    }
    double out;
    if (ci >= 0 && ci == cj) {
      const int64_t kc = co[ci + 1] - co[ci];
      const double* X = reinterpret_cast<const double*>(child_xss[4 * b + ci]);
      out = X[(pi - co[ci]) * kc + (pj - co[ci])];
    } else {
      const int64_t da = act[a0 + pi], db = act[a0 + pj];
      const int64_t na = da >> 1, nb = db >> 1;
      const int ca = (int)(da & 1), cb = (int)(db & 1);
      const double2 pa = g.pos[na], pb = g.pos[nb];
      const double2 nav = g.nrm[na], nbv = g.nrm[nb];
      const double rx = pa.x - pb.x, ry = pa.y - pb.y;
      double kern;
      if (na == nb) {
        // smooth-curve limit -(kappa/(2 pi)) tau_a tau_b, tau = (-n_y, n_x)
        const double ta = ca == 0 ? -nav.y : nav.x;
        const double tb = cb == 0 ? -nbv.y : nbv.x;
        kern = ((-(kappa[nb] / (2.0 * SKB_PI))) * ta) * tb;
      } else {
        const double r2 = rx * rx + ry * ry;
        const double rdn = rx * nbv.x + ry * nbv.y;
        const double coef = rdn / ((SKB_PI * r2) * r2);
        kern = (coef * (ca == 0 ? rx : ry)) * (cb == 0 ? rx : ry);
      }
      kern = kern + comp(nav, ca) * comp(nbv, cb);
      out = kern * g.w[nb];
      out = out + (da == db ? -0.5 : 0.0);
    }
    Eb[i * ld + j] = out;
  }
}


// ---- Laplace-Neumann branch (dof = node): reference kernels.py:119-125
// (self block), 161-168 (far pairs), 322-325 / 347-352 (proxy rows),
// 368-370 (nullspace rows); stack rows 2 nF + 2 P + 2, same order
// [k_in; P_in; n_in; k_out^T; P_out; n_out] (skel.py:306-314).
#define SKB_2PI (2.0 * SKB_PI)     // 2 * np.pi (exact doubling)
#define SKB_4PI (4.0 * SKB_PI)

__global__ void k_assemble_stack_lap(Geo g, const int64_t* __restrict__ act_off,
                                     const int64_t* __restrict__ act,
                                     const int64_t* __restrict__ far_off,
                                     const int64_t* __restrict__ far,
                                     const double2* __restrict__ ppts, const double* __restrict__ pw,
                                     int P, const int64_t* __restrict__ stack_off,
                                     double* __restrict__ stack) {
  const int64_t b = blockIdx.y;
  const int64_t a0 = act_off[b], nB = act_off[b + 1] - a0;
  const int64_t f0 = far_off[b], nF = far_off[b + 1] - f0;
  const int64_t items = nF + P + 1;
  const int64_t rows = 2 * nF + 2 * (int64_t)P + 2;
  double* S = stack + stack_off[b];
  const double pwb = pw[b];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < items * nB;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / items, it = t - j * items;
    const int64_t nb = act[a0 + j];
    const double2 pb = g.pos[nb], nbv = g.nrm[nb];
    const double wb = g.w[nb];
    double* col = S + j * rows;
    if (it < nF) {
      const int64_t nf = far[f0 + it];
      const double2 pf = g.pos[nf], nfv = g.nrm[nf];
      const double rx = pf.x - pb.x, ry = pf.y - pb.y;
      const double r2 = rx * rx + ry * ry;
      const double rdn_f = rx * nfv.x + ry * nfv.y;
      const double rdn_b = rx * nbv.x + ry * nbv.y;
      const double ir2 = 1.0 / (SKB_2PI * r2);
      col[it] = (rdn_f * ir2 + 1.0) * wb;
      col[nF + P + 1 + it] = ((-rdn_b) * ir2 + 1.0) * g.w[nf];
    } else if (it < nF + P) {
      const int p = (int)(it - nF);
      const double2 pp = ppts[b * P + p];
      {   // incoming: log potential of the box source at the proxy point
        const double rx = pp.x - pb.x, ry = pp.y - pb.y;
        const double r2 = rx * rx + ry * ry;
        col[nF + p] = ((-0.25 * log(r2)) / SKB_PI) * wb;
      }
      {   // outgoing: target-normal dipole of the proxy source at the box node
        const double rx = pb.x - pp.x, ry = pb.y - pp.y;
        const double r2 = rx * rx + ry * ry;
        const double blk = (rx * nbv.x + ry * nbv.y) / (SKB_2PI * r2);
        col[2 * nF + P + 1 + p] = blk * pwb;
      }
    } else {
      col[nF + P] = wb;
      col[rows - 1] = 1.0;
    }
  }
}

__global__ void k_assemble_self_lap(Geo g, const double* __restrict__ kappa,
                                    const int64_t* __restrict__ act_off,
                                    const int64_t* __restrict__ act,
                                    const int64_t* __restrict__ perm_off,
                                    const int32_t* __restrict__ perm,
                                    const int64_t* __restrict__ child_off,
                                    const int64_t* __restrict__ child_xss, double* __restrict__ E,
                                    const int64_t* __restrict__ E_off,
                                    const int64_t* __restrict__ E_ld) {
  const int64_t b = blockIdx.y;
  const int64_t a0 = act_off[b], n = act_off[b + 1] - a0;
  const int64_t* co = child_off + 5 * b;
  const int64_t ld = E_ld[b];
  double* Eb = E + E_off[b];
  const int32_t* pm = perm ? perm + perm_off[b] : nullptr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    const int64_t pi = pm ? pm[i] : i, pj = pm ? pm[j] : j;
    int ci = -1, cj = -1;
    if (co[0] >= 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (co[c + 1] < 0) break;
        if (pi >= co[c] && pi < co[c + 1]) ci = c;
        if (pj >= co[c] && pj < co[c + 1]) cj = c;
      }
    }
    double out;
    if (ci >= 0 && ci == cj) {
      const int64_t kc = co[ci + 1] - co[ci];
      const double* X = reinterpret_cast<const double*>(child_xss[4 * b + ci]);
      out = X[(pi - co[ci]) * kc + (pj - co[ci])];
    } else {
      const int64_t na = act[a0 + pi], nb = act[a0 + pj];
      double kern;
      if (na == nb) {
        kern = kappa[na] / SKB_4PI;                 // same-node limit kappa_row / (4 pi)
      } else {
        const double2 pa = g.pos[na], pb = g.pos[nb], nav = g.nrm[na];
        const double rx = pa.x - pb.x, ry = pa.y - pb.y;
        const double r2 = rx * rx + ry * ry;
        const double rdn = rx * nav.x + ry * nav.y;
        kern = rdn / (SKB_2PI * r2);
      }
      kern = kern + 1.0;
      out = kern * g.w[nb];
      out = out + (na == nb ? -0.5 : 0.0);
    }
    Eb[i * ld + j] = out;
  }
}

__global__ void k_assemble_H(const double2* __restrict__ pos, int64_t n,
                             const double2* __restrict__ ctr, int64_t p, double* __restrict__ H) {
  const int64_t q = 3 * p;
  const double pref = 1.0 / (4.0 * SKB_PI);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * p;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = t / p, h = t - node * p;
    const double2 x = pos[node], c = ctr[h];
    const double rx = x.x - c.x, ry = x.y - c.y;
    const double r2 = rx * rx + ry * ry;
    const double lg = -0.5 * log(r2);
    double* r0 = H + (2 * node) * q + 3 * h;
    double* r1 = r0 + q;
    r0[0] = pref * (lg + (rx * rx) / r2);
    r1[0] = pref * ((ry * rx) / r2);
    r0[1] = pref * ((rx * ry) / r2);
    r1[1] = pref * (lg + (ry * ry) / r2);
    r0[2] = (pref * (-ry)) / r2;
    r1[2] = (pref * rx) / r2;
  }
}

__global__ void k_assemble_Psi(const double2* __restrict__ pos, const double* __restrict__ w,
                               int64_t n, int64_t p, const int64_t* __restrict__ curve_off,
                               double* __restrict__ Psi) {
  const int64_t q = 3 * p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    double* r0 = Psi + (2 * t) * q;
    double* r1 = r0 + q;
    // curve index (outer = 0) of node t
    int64_t lo = 0, hi = p;  // curves 0..p; curve_off has p+2 entries
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) >> 1;
      if (curve_off[mid] <= t) lo = mid; else hi = mid - 1;
    }
    if (lo >= 1) {
      const int64_t h = lo - 1;
      const double wt = w[t];
      const double2 x = pos[t];
      r0[3 * h] = wt;
      r1[3 * h + 1] = wt;
      r0[3 * h + 2] = (-x.y) * wt;
      r1[3 * h + 2] = x.x * wt;
    }
  }
}

}  // namespace skb

using namespace skb;

extern "C" int skb_assemble_stack(const double* pos, const double* nrm, const double* w,
                                  int64_t nbox, const int64_t* act_off, const int64_t* act,
                                  const int64_t* far_off, const int64_t* far, const double* ppts,
                                  const double* pnrm, const double* pw, int32_t P,
                                  const int64_t* stack_off, double* stack, int64_t max_cols,
                                  int64_t max_items, void* stream) {
  if (nbox <= 0) return 0;
  if (nbox > 65535) return 2;
  Geo g{(const double2*)pos, (const double2*)nrm, w};
  int64_t work = max_cols * max_items;
  dim3 grid(grid_cap((work + 255) / 256, 4096), (unsigned)nbox);
  ProfScope ps(F_ASSEMBLE, (cudaStream_t)stream);
  k_assemble_stack<<<grid, 256, 0, (cudaStream_t)stream>>>(
      g, act_off, act, far_off, far, (const double2*)ppts, (const double2*)pnrm, pw, P, stack_off,
      stack);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_assemble_self(const double* pos, const double* nrm, const double* w,
                                 const double* kappa, int64_t nbox, const int64_t* act_off,
                                 const int64_t* act, const int64_t* perm_off, const int32_t* perm,
                                 const int64_t* child_off, const int64_t* child_xss, double* E,
                                 const int64_t* E_off, const int64_t* E_ld, int64_t max_n,
                                 void* stream) {
  if (nbox <= 0) return 0;
  if (nbox > 65535) return 2;
  Geo g{(const double2*)pos, (const double2*)nrm, w};
  dim3 grid(grid_cap((max_n * max_n + 255) / 256, 4096), (unsigned)nbox);
  ProfScope ps(F_ASSEMBLE, (cudaStream_t)stream);
  k_assemble_self<<<grid, 256, 0, (cudaStream_t)stream>>>(g, kappa, act_off, act, perm_off, perm,
                                                          child_off, child_xss, E, E_off, E_ld);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_assemble_aug(const double* pos, const double* w, int64_t n_nodes,
                                const double* hole_centers, int64_t n_holes,
                                const int64_t* curve_off_host, double* H, double* Psi,
                                void* stream) {
  if (n_holes <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* d_off = nullptr;
  int rc = upload(curve_off_host, n_holes + 2, s, &d_off);
  if (rc) return rc;
  k_assemble_H<<<grid_cap((n_nodes * n_holes + 255) / 256, 148 * 64), 256, 0, s>>>(
      (const double2*)pos, n_nodes, (const double2*)hole_centers, n_holes, H);
  cudaMemsetAsync(Psi, 0, sizeof(double) * 2 * n_nodes * 3 * n_holes, s);
  k_assemble_Psi<<<grid_cap((n_nodes + 255) / 256, 148 * 64), 256, 0, s>>>(
      (const double2*)pos, w, n_nodes, n_holes, d_off, Psi);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(d_off, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" int skb_assemble_stack_lap(const double* pos, const double* nrm, const double* w,
                                      int64_t nbox, const int64_t* act_off, const int64_t* act,
                                      const int64_t* far_off, const int64_t* far, const double* ppts,
                                      const double* pnrm, const double* pw, int32_t P,
                                      const int64_t* stack_off, double* stack, int64_t max_cols,
                                      int64_t max_items, void* stream) {
  (void)pnrm;
  if (nbox <= 0) return 0;
  if (nbox > 65535) return 2;
  Geo g{(const double2*)pos, (const double2*)nrm, w};
  int64_t work = max_cols * max_items;
  dim3 grid(grid_cap((work + 255) / 256, 4096), (unsigned)nbox);
  ProfScope ps(F_ASSEMBLE, (cudaStream_t)stream);
  k_assemble_stack_lap<<<grid, 256, 0, (cudaStream_t)stream>>>(
      g, act_off, act, far_off, far, (const double2*)ppts, pw, P, stack_off, stack);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_assemble_self_lap(const double* pos, const double* nrm, const double* w,
                                     const double* kappa, int64_t nbox, const int64_t* act_off,
                                     const int64_t* act, const int64_t* perm_off, const int32_t* perm,
                                     const int64_t* child_off, const int64_t* child_xss, double* E,
                                     const int64_t* E_off, const int64_t* E_ld, int64_t max_n,
                                     void* stream) {
  if (nbox <= 0) return 0;
  if (nbox > 65535) return 2;
  Geo g{(const double2*)pos, (const double2*)nrm, w};
  dim3 grid(grid_cap((max_n * max_n + 255) / 256, 4096), (unsigned)nbox);
  ProfScope ps(F_ASSEMBLE, (cudaStream_t)stream);
  k_assemble_self_lap<<<grid, 256, 0, (cudaStream_t)stream>>>(g, kappa, act_off, act, perm_off, perm,
                                                              child_off, child_xss, E, E_off, E_ld);
  SKB_LAUNCH_CHECK();
  return 0;
}

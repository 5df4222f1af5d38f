// Exact (uncompressed) augmented system product y = M x by direct summation --
// reference kernels.system_matvec (kernels.py:393-414) built on eval_block
// (kernels.py:89-130), stokeslet_rotlet_columns (kernels.py:201-223) and
// build_augmentation's Psi (kernels.py:226-246):
//   y[:nd] = (-1/2 I + D + N) mu + H lam,   y[nd:] = Psi^T mu - lam.
// The residual oracle for the large configs (cfg3/cfg5), where the CPU
// row-chunked product takes hours.  O(N^2) pairs, smem-tiled sources,
// one thread per target node, RHS processed in chunks of 4 columns.
#include "common.cuh"

namespace skb {

constexpr int MV_T = 128;   // targets per block / sources per tile
constexpr int MV_R = 4;     // RHS per pass
#define MV_PI 3.141592653589793

// s[h] = sum_j w_j n_j . mu_j over all nodes (the rank-one completion N)
__global__ void k_mv_ndot(const double2* __restrict__ nrm, const double* __restrict__ w,
                          int64_t n, const double* __restrict__ x, int64_t nr, int64_t r0,
                          int rc, double* __restrict__ out) {
  __shared__ double red[MV_R][MV_T];
  double acc[MV_R] = {0, 0, 0, 0};
  for (int64_t j = blockIdx.x * (int64_t)MV_T + threadIdx.x; j < n; j += (int64_t)gridDim.x * MV_T) {
    const double2 nj = nrm[j];
    const double wj = w[j];
    for (int q = 0; q < rc; ++q) {
      const double m0 = x[(2 * j) * nr + r0 + q], m1 = x[(2 * j + 1) * nr + r0 + q];
      acc[q] += wj * (nj.x * m0 + nj.y * m1);
    }
  }
  for (int q = 0; q < MV_R; ++q) red[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int o = MV_T / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int q = 0; q < MV_R; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < rc; ++q) out[blockIdx.x * MV_R + q] = red[q][0];
}

__global__ void __launch_bounds__(MV_T)
k_mv_direct(const double2* __restrict__ pos, const double2* __restrict__ nrm,
            const double* __restrict__ w, const double* __restrict__ kappa, int64_t n,
            const double2* __restrict__ ctr, int64_t p, const double* __restrict__ x, int64_t nr,
            int64_t r0, int rc, const double* __restrict__ ndot_parts, int nparts,
            double* __restrict__ y) {
  __shared__ double2 sp[MV_T], sn[MV_T];
  __shared__ double sw[MV_T];
  __shared__ double sx[MV_T][2 * MV_R];
  __shared__ double s_nd[MV_R];
  const int64_t i = blockIdx.x * (int64_t)MV_T + threadIdx.x;
  if (threadIdx.x < MV_R) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += ndot_parts[b * MV_R + threadIdx.x];
    s_nd[threadIdx.x] = s;
  }
  const bool act = i < n;
  const double2 pi = act ? pos[i] : make_double2(0, 0);
  const double2 ni = act ? nrm[i] : make_double2(0, 0);
  double a0[MV_R] = {0, 0, 0, 0}, a1[MV_R] = {0, 0, 0, 0};
  for (int64_t j0 = 0; j0 < n; j0 += MV_T) {
    __syncthreads();
    const int64_t j = j0 + threadIdx.x;
    if (j < n) {
      sp[threadIdx.x] = pos[j];
      sn[threadIdx.x] = nrm[j];
      sw[threadIdx.x] = w[j];
      for (int q = 0; q < rc; ++q) {
        sx[threadIdx.x][2 * q] = x[(2 * j) * nr + r0 + q];
        sx[threadIdx.x][2 * q + 1] = x[(2 * j + 1) * nr + r0 + q];
      }
    }
    __syncthreads();
    const int jn = (int)((n - j0) < MV_T ? (n - j0) : MV_T);
    if (!act) continue;
    for (int jj = 0; jj < jn; ++jj) {
      const int64_t jg = j0 + jj;
      const double2 pj = sp[jj], nj = sn[jj];
      const double wj = sw[jj];
      double k00, k01, k10, k11;
      if (jg == i) {
        // smooth-curve limit -(kappa/(2 pi)) tau tau^T, tau = (-n_y, n_x)
        const double c = -(kappa[i] / (2.0 * MV_PI)) * wj;
        const double t0 = -nj.y, t1 = nj.x;
        k00 = c * t0 * t0; k01 = c * t0 * t1; k10 = c * t1 * t0; k11 = c * t1 * t1;
      } else {
        const double rx = pi.x - pj.x, ry = pi.y - pj.y;
        const double r2 = rx * rx + ry * ry;
        const double c = (rx * nj.x + ry * nj.y) / (MV_PI * r2 * r2) * wj;
        k00 = c * rx * rx; k01 = c * rx * ry; k10 = k01; k11 = c * ry * ry;
      }
      for (int q = 0; q < MV_R; ++q) {
        if (q >= rc) break;
        const double m0 = sx[jj][2 * q], m1 = sx[jj][2 * q + 1];
        a0[q] += k00 * m0 + k01 * m1;
        a1[q] += k10 * m0 + k11 * m1;
      }
    }
  }
  if (!act) return;
  for (int q = 0; q < rc; ++q) {
    const double mu0 = x[(2 * i) * nr + r0 + q], mu1 = x[(2 * i + 1) * nr + r0 + q];
    double y0 = a0[q] + ni.x * s_nd[q] - 0.5 * mu0;
    double y1 = a1[q] + ni.y * s_nd[q] - 0.5 * mu1;
    // H lam: Stokeslet (2 columns) + rotlet per hole centre
    const double pref = 1.0 / (4.0 * MV_PI);
    for (int64_t h = 0; h < p; ++h) {
      const double2 c = ctr[h];
      const double rx = pi.x - c.x, ry = pi.y - c.y;
      const double r2 = rx * rx + ry * ry;
      const double lg = -0.5 * log(r2);
      const double l0 = x[(2 * n + 3 * h) * nr + r0 + q];
      const double l1 = x[(2 * n + 3 * h + 1) * nr + r0 + q];
      const double l2 = x[(2 * n + 3 * h + 2) * nr + r0 + q];
      y0 += pref * (lg + rx * rx / r2) * l0 + pref * (rx * ry / r2) * l1 + pref * (-ry) / r2 * l2;
      y1 += pref * (ry * rx / r2) * l0 + pref * (lg + ry * ry / r2) * l1 + pref * rx / r2 * l2;
    }
    y[(2 * i) * nr + r0 + q] = y0;
    y[(2 * i + 1) * nr + r0 + q] = y1;
  }
}

// y[nd + 3h + t] = sum over hole-h nodes of Psi rows . mu  - lam  (one block per hole)
__global__ void k_mv_psi(const double2* __restrict__ pos, const double* __restrict__ w,
                         const int64_t* __restrict__ curve_off, int64_t n,
                         const double* __restrict__ x, int64_t nr, int64_t r0, int rc,
                         double* __restrict__ y) {
  __shared__ double red[3][MV_T];
  const int64_t h = blockIdx.x;
  const int64_t a = curve_off[h + 1], b = curve_off[h + 2];
  for (int q = 0; q < rc; ++q) {
    double s0 = 0, s1 = 0, s2 = 0;
    for (int64_t j = a + threadIdx.x; j < b; j += MV_T) {
      const double m0 = x[(2 * j) * nr + r0 + q], m1 = x[(2 * j + 1) * nr + r0 + q];
      const double wj = w[j];
      const double2 pj = pos[j];
      s0 += wj * m0;
      s1 += wj * m1;
      s2 += (-pj.y) * wj * m0 + pj.x * wj * m1;
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    red[2][threadIdx.x] = s2;
    __syncthreads();
    for (int o = MV_T / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o)
        for (int t = 0; t < 3; ++t) red[t][threadIdx.x] += red[t][threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x < 3) {
      const int64_t row = 2 * n + 3 * h + threadIdx.x;
      y[row * nr + r0 + q] = red[threadIdx.x][0] - x[row * nr + r0 + q];
    }
    __syncthreads();
  }
}


// Interior evaluation u(t) = D mu + H lam at targets off the boundary --
// reference evaluate_interior (skel.py:537-564) with eval_forward_block
// (kernels.py:171-198, Stokes: no jump, no completion term) and
// stokeslet_rotlet_columns (kernels.py:201-223).  One thread per target,
// sources tiled through shared memory, summed in node order.
__global__ void __launch_bounds__(MV_T)
k_eval_interior(const double2* __restrict__ pos, const double2* __restrict__ nrm,
                const double* __restrict__ w, int64_t n, const double2* __restrict__ ctr,
                int64_t p, const double* __restrict__ x, int64_t nr, int64_t r0, int rc,
                const double2* __restrict__ tgt, int64_t m, double* __restrict__ out) {
  __shared__ double2 sp[MV_T], sn[MV_T];
  __shared__ double sw[MV_T];
  __shared__ double sx[MV_T][2 * MV_R];
  const int64_t i = blockIdx.x * (int64_t)MV_T + threadIdx.x;
  const bool act = i < m;
  const double2 ti = act ? tgt[i] : make_double2(0, 0);
  double a0[MV_R] = {0, 0, 0, 0}, a1[MV_R] = {0, 0, 0, 0};
  for (int64_t j0 = 0; j0 < n; j0 += MV_T) {
    __syncthreads();
    const int64_t j = j0 + threadIdx.x;
    if (j < n) {
      sp[threadIdx.x] = pos[j];
      sn[threadIdx.x] = nrm[j];
      sw[threadIdx.x] = w[j];
      for (int q = 0; q < rc; ++q) {
        sx[threadIdx.x][2 * q] = x[(2 * j) * nr + r0 + q];
        sx[threadIdx.x][2 * q + 1] = x[(2 * j + 1) * nr + r0 + q];
      }
    }
    __syncthreads();
    const int jn = (int)((n - j0) < MV_T ? (n - j0) : MV_T);
    if (!act) continue;
    for (int jj = 0; jj < jn; ++jj) {
      const double2 pj = sp[jj], nj = sn[jj];
      const double rx = ti.x - pj.x, ry = ti.y - pj.y;
      const double r2 = rx * rx + ry * ry;
      const double c = (rx * nj.x + ry * nj.y) / (MV_PI * r2 * r2) * sw[jj];
      for (int q = 0; q < MV_R; ++q) {
        if (q >= rc) break;
        const double proj = rx * sx[jj][2 * q] + ry * sx[jj][2 * q + 1];
        a0[q] += c * rx * proj;
        a1[q] += c * ry * proj;
      }
    }
  }
  if (!act) return;
  const double pref = 1.0 / (4.0 * MV_PI);
  for (int q = 0; q < rc; ++q) {
    double y0 = a0[q], y1 = a1[q];
    for (int64_t h = 0; h < p; ++h) {
      const double2 c = ctr[h];
      const double rx = ti.x - c.x, ry = ti.y - c.y;
      const double r2 = rx * rx + ry * ry;
      const double lg = -0.5 * log(r2);
      const double l0 = x[(2 * n + 3 * h) * nr + r0 + q];
      const double l1 = x[(2 * n + 3 * h + 1) * nr + r0 + q];
      const double l2 = x[(2 * n + 3 * h + 2) * nr + r0 + q];
      y0 += pref * (lg + rx * rx / r2) * l0 + pref * (rx * ry / r2) * l1 + pref * (-ry) / r2 * l2;
      y1 += pref * (ry * rx / r2) * l0 + pref * (lg + ry * ry / r2) * l1 + pref * rx / r2 * l2;
    }
    out[(2 * i) * nr + r0 + q] = y0;
    out[(2 * i + 1) * nr + r0 + q] = y1;
  }
}

// Boundary.point_in_domain (reference geometry.py:179-192, _winding
// geometry.py:221-233): winding number of every curve's node polyline around
// each target (inside the outer curve, outside every hole) and nearest-node
// distance > 1e-12.  One warp per target; per-curve angle sums in node order
// per lane, then a fixed-order warp reduction.
__global__ void k_point_in_domain(const double2* __restrict__ pos, const int64_t* __restrict__ off,
                                  int64_t ncurves, const double2* __restrict__ tgt, int64_t m,
                                  uint8_t* __restrict__ inside) {
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= m) return;
  const double2 q = tgt[t];
  bool ok = true;
  double dmin2 = 1e300;
  for (int64_t c = 0; c < ncurves; ++c) {
    const int64_t a = off[c], b = off[c + 1];
    double ang = 0.0;
    for (int64_t j = a + lane; j < b; j += 32) {
      const double2 p0 = pos[j], p1 = pos[j + 1 < b ? j + 1 : a];
      const double ax = p0.x - q.x, ay = p0.y - q.y, bx = p1.x - q.x, by = p1.y - q.y;
      ang += atan2(ax * by - ay * bx, ax * bx + ay * by);
      dmin2 = fmin(dmin2, ax * ax + ay * ay);
    }
    ang = warp_sum(ang);
    const double wn = rint(ang / (2.0 * MV_PI));
    ok = ok && (c == 0 ? wn != 0.0 : wn == 0.0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmin2 = fmin(dmin2, __shfl_xor_sync(0xffffffffu, dmin2, o));
  if (lane == 0) inside[t] = (ok && sqrt(dmin2) > 1e-12) ? 1 : 0;
}


// ---- Laplace-Neumann (one DOF per node) -----------------------------------
// s = sum_j w_j mu_j (the +1 completion of kernels.py:125), per RHS
__global__ void k_mv_wdot(const double* __restrict__ w, int64_t n, const double* __restrict__ x,
                          int64_t nr, int64_t r0, int rc, double* __restrict__ out) {
  __shared__ double red[MV_R][MV_T];
  double acc[MV_R] = {0, 0, 0, 0};
  for (int64_t j = blockIdx.x * (int64_t)MV_T + threadIdx.x; j < n; j += (int64_t)gridDim.x * MV_T)
    for (int q = 0; q < rc; ++q) acc[q] += w[j] * x[j * nr + r0 + q];
  for (int q = 0; q < MV_R; ++q) red[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int o = MV_T / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int q = 0; q < MV_R; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < rc; ++q) out[blockIdx.x * MV_R + q] = red[q][0];
}

// y_a = -1/2 mu_a + sum_b K'_ab w_b mu_b + sum_b w_b mu_b, K'_ab = (x_a - x_b).n_a / (2 pi r^2),
// K'_aa = kappa_a / (4 pi)  (kernels.py:119-125)
__global__ void __launch_bounds__(MV_T)
k_mv_direct_lap(const double2* __restrict__ pos, const double2* __restrict__ nrm,
                const double* __restrict__ w, const double* __restrict__ kappa, int64_t n,
                const double* __restrict__ x, int64_t nr, int64_t r0, int rc,
                const double* __restrict__ parts, int nparts, double* __restrict__ y) {
  __shared__ double2 sp[MV_T];
  __shared__ double swx[MV_T][MV_R];
  __shared__ double s_w[MV_R];
  const int64_t i = blockIdx.x * (int64_t)MV_T + threadIdx.x;
  if (threadIdx.x < MV_R) {
    double sm = 0.0;
    for (int b = 0; b < nparts; ++b) sm += parts[b * MV_R + threadIdx.x];
    s_w[threadIdx.x] = sm;
  }
  const bool act = i < n;
  const double2 pi = act ? pos[i] : make_double2(0, 0);
  const double2 ni = act ? nrm[i] : make_double2(0, 0);
  double a[MV_R] = {0, 0, 0, 0};
  for (int64_t j0 = 0; j0 < n; j0 += MV_T) {
    __syncthreads();
    const int64_t j = j0 + threadIdx.x;
    if (j < n) {
      sp[threadIdx.x] = pos[j];
      for (int q = 0; q < rc; ++q) swx[threadIdx.x][q] = w[j] * x[j * nr + r0 + q];
    }
    __syncthreads();
    const int jn = (int)((n - j0) < MV_T ? (n - j0) : MV_T);
    if (!act) continue;
    for (int jj = 0; jj < jn; ++jj) {
      const int64_t jg = j0 + jj;
      double k;
      if (jg == i) {
        k = kappa[i] / (4.0 * MV_PI);
      } else {
        const double2 pj = sp[jj];
        const double rx = pi.x - pj.x, ry = pi.y - pj.y;
        k = (rx * ni.x + ry * ni.y) / ((2.0 * MV_PI) * (rx * rx + ry * ry));
      }
      for (int q = 0; q < MV_R; ++q) {
        if (q >= rc) break;
        a[q] += k * swx[jj][q];
      }
    }
  }
  if (!act) return;
  for (int q = 0; q < rc; ++q) y[i * nr + r0 + q] = a[q] + s_w[q] - 0.5 * x[i * nr + r0 + q];
}

// u(t) = sum_j (1/2 log r^2 / (2 pi)) w_j mu_j  (kernels.py:193-194; u = -S mu)
__global__ void __launch_bounds__(MV_T)
k_eval_interior_lap(const double2* __restrict__ pos, const double* __restrict__ w, int64_t n,
                    const double* __restrict__ x, int64_t nr, int64_t r0, int rc,
                    const double2* __restrict__ tgt, int64_t m, double* __restrict__ out) {
  __shared__ double2 sp[MV_T];
  __shared__ double swx[MV_T][MV_R];
  const int64_t i = blockIdx.x * (int64_t)MV_T + threadIdx.x;
  const bool act = i < m;
  const double2 ti = act ? tgt[i] : make_double2(0, 0);
  double a[MV_R] = {0, 0, 0, 0};
  for (int64_t j0 = 0; j0 < n; j0 += MV_T) {
    __syncthreads();
    const int64_t j = j0 + threadIdx.x;
    if (j < n) {
      sp[threadIdx.x] = pos[j];
      for (int q = 0; q < rc; ++q) swx[threadIdx.x][q] = w[j] * x[j * nr + r0 + q];
    }
    __syncthreads();
    const int jn = (int)((n - j0) < MV_T ? (n - j0) : MV_T);
    if (!act) continue;
    for (int jj = 0; jj < jn; ++jj) {
      const double2 pj = sp[jj];
      const double rx = ti.x - pj.x, ry = ti.y - pj.y;
      const double g = (0.5 * log(rx * rx + ry * ry)) / (2.0 * MV_PI);
      for (int q = 0; q < MV_R; ++q) {
        if (q >= rc) break;
        a[q] += g * swx[jj][q];
      }
    }
  }
  if (!act) return;
  for (int q = 0; q < rc; ++q) out[i * nr + r0 + q] = a[q];
}

}  // namespace skb

using namespace skb;

extern "C" int skb_system_matvec(const double* pos, const double* nrm, const double* w,
                                 const double* kappa, int64_t n_nodes, const double* hole_centers,
                                 int64_t n_holes, const int64_t* curve_off_dev, const double* x,
                                 int64_t nrhs, double* y, void* stream) {
  if (n_nodes <= 0 || nrhs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int nparts = 148;
  double* parts = nullptr;
  SKB_RET(malloc_async((void**)&parts, sizeof(double) * nparts * MV_R, s));
  for (int64_t r0 = 0; r0 < nrhs; r0 += MV_R) {
    const int rc = (int)((nrhs - r0) < MV_R ? (nrhs - r0) : MV_R);
    k_mv_ndot<<<nparts, MV_T, 0, s>>>((const double2*)nrm, w, n_nodes, x, nrhs, r0, rc, parts);
    k_mv_direct<<<(unsigned)((n_nodes + MV_T - 1) / MV_T), MV_T, 0, s>>>(
        (const double2*)pos, (const double2*)nrm, w, kappa, n_nodes, (const double2*)hole_centers,
        n_holes, x, nrhs, r0, rc, parts, nparts, y);
    if (n_holes > 0)
      k_mv_psi<<<(unsigned)n_holes, MV_T, 0, s>>>((const double2*)pos, w, curve_off_dev, n_nodes,
                                                   x, nrhs, r0, rc, y);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(parts, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" int skb_eval_interior(const double* pos, const double* nrm, const double* w,
                                 int64_t n_nodes, const double* hole_centers, int64_t n_holes,
                                 const double* x, int64_t nrhs, const double* targets, int64_t m,
                                 double* out, void* stream) {
  if (m <= 0 || nrhs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t r0 = 0; r0 < nrhs; r0 += MV_R) {
    const int rc = (int)((nrhs - r0) < MV_R ? (nrhs - r0) : MV_R);
    k_eval_interior<<<(unsigned)((m + MV_T - 1) / MV_T), MV_T, 0, s>>>(
        (const double2*)pos, (const double2*)nrm, w, n_nodes, (const double2*)hole_centers, n_holes,
        x, nrhs, r0, rc, (const double2*)targets, m, out);
  }
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_point_in_domain(const double* pos, const int64_t* curve_off_dev, int64_t ncurves,
                                   const double* targets, int64_t m, uint8_t* inside, void* stream) {
  if (m <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  k_point_in_domain<<<(unsigned)((m * 32 + 255) / 256), 256, 0, s>>>(
      (const double2*)pos, curve_off_dev, ncurves, (const double2*)targets, m, inside);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_system_matvec_lap(const double* pos, const double* nrm, const double* w,
                                     const double* kappa, int64_t n_nodes, const double* x,
                                     int64_t nrhs, double* y, void* stream) {
  if (n_nodes <= 0 || nrhs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int nparts = 148;
  double* parts = nullptr;
  SKB_RET(malloc_async((void**)&parts, sizeof(double) * nparts * MV_R, s));
  for (int64_t r0 = 0; r0 < nrhs; r0 += MV_R) {
    const int rc = (int)((nrhs - r0) < MV_R ? (nrhs - r0) : MV_R);
    k_mv_wdot<<<nparts, MV_T, 0, s>>>(w, n_nodes, x, nrhs, r0, rc, parts);
    k_mv_direct_lap<<<(unsigned)((n_nodes + MV_T - 1) / MV_T), MV_T, 0, s>>>(
        (const double2*)pos, (const double2*)nrm, w, kappa, n_nodes, x, nrhs, r0, rc, parts, nparts, y);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(parts, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" int skb_eval_interior_lap(const double* pos, const double* w, int64_t n_nodes,
                                     const double* x, int64_t nrhs, const double* targets, int64_t m,
                                     double* out, void* stream) {
  if (m <= 0 || nrhs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t r0 = 0; r0 < nrhs; r0 += MV_R) {
    const int rc = (int)((nrhs - r0) < MV_R ? (nrhs - r0) : MV_R);
    k_eval_interior_lap<<<(unsigned)((m + MV_T - 1) / MV_T), MV_T, 0, s>>>(
        (const double2*)pos, w, n_nodes, x, nrhs, r0, rc, (const double2*)targets, m, out);
  }
  SKB_LAUNCH_CHECK();
  return 0;
}

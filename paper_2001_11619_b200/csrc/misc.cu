// Data-movement kernels of the level pipeline: DOF-list row gathers/scatters
// (the NumPy fancy indexing x[dofs] of reference skel.py:140-221, 384-396),
// batched 2-D copies, the deterministic Schur accumulation (skel.py:396) and
// the corner's -I - schur block (skel.py:404).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace skb {

// Batched 2-D copies / row gathers / row scatters.  Pure data movement (HBM /
// L2 bound): consecutive threads walk consecutive columns of a row, rows are
// dealt to warps (narrow rows) or to whole blocks (wide rows), all index
// arithmetic in 32 bits without divisions; compact blocks copy as double2.
__global__ void k_copy2d(const SkbMat* __restrict__ dst, const SkbMat* __restrict__ src,
                         int trans) {
  const SkbMat D = dst[blockIdx.y], S = src[blockIdx.y];
  const int rows = (int)D.rows, cols = (int)D.cols;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
  if (trans) {                                     // D[i][j] = S[j][i] (one small call per factorization)
    const unsigned tot = (unsigned)rows * (unsigned)cols;
    for (unsigned t = gtid; t < tot; t += nthr) {
      const unsigned j = t / (unsigned)rows, i = t - j * (unsigned)rows;   // walk src rows contiguously
      D.ptr[(int64_t)i * D.ld + j] = S.ptr[(int64_t)j * S.ld + i];
    }
    return;
  }
  if (D.ld == cols && S.ld == cols) {              // compact block: flat copy
    const int64_t tot = (int64_t)rows * cols;
    if ((((uintptr_t)D.ptr | (uintptr_t)S.ptr) & 15) == 0) {
      const int64_t n2 = tot >> 1;
      double2* d2 = reinterpret_cast<double2*>(D.ptr);
      const double2* s2 = reinterpret_cast<const double2*>(S.ptr);
      for (int64_t t = gtid; t < n2; t += nthr) d2[t] = s2[t];
      if ((tot & 1) && gtid == 0) D.ptr[tot - 1] = S.ptr[tot - 1];
    } else {
      for (int64_t t = gtid; t < tot; t += nthr) D.ptr[t] = S.ptr[t];
    }
    return;
  }
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5), nw = gridDim.x * wpb;
  for (int i = gw; i < rows; i += nw) {
    const double* sp = S.ptr + (int64_t)i * S.ld;
    double* dp = D.ptr + (int64_t)i * D.ld;
    for (int j = lane; j < cols; j += 32) dp[j] = sp[j];
  }
}

// rows per step and threads per row for a row length nc: 256 threads cover
// 256 / tpr rows at a time, tpr = 32 .. 256 consecutive threads on one row
__device__ __forceinline__ int row_tpr(int nc) { return nc > 128 ? 256 : (nc > 64 ? 128 : (nc > 32 ? 64 : 32)); }

__global__ void k_gather_rows(const int64_t* __restrict__ idx_off, const int64_t* __restrict__ idx,
                              const int64_t* __restrict__ col_off,
                              const int64_t* __restrict__ col, int64_t ncols,
                              const double* __restrict__ src, int64_t src_ld,
                              double* __restrict__ dst, const int64_t* __restrict__ dst_off,
                              const int64_t* __restrict__ dst_ld) {
  const int64_t b = blockIdx.y;
  const int64_t i0 = idx_off[b];
  const int nr = (int)(idx_off[b + 1] - i0);
  const int64_t c0 = col ? col_off[b] : 0;
  const int nc = (int)(col ? col_off[b + 1] - c0 : ncols);
  double* d = dst + dst_off[b];
  const int64_t ld = dst_ld[b];
  const int tpr = row_tpr(nc), rps = 256 / tpr;
  const int tr = threadIdx.x / tpr, tc = threadIdx.x - tr * tpr;
  if (!col && tpr == 256 && !(nc & 1) && !(src_ld & 1) && !(ld & 1) && !(dst_off[b] & 1) &&
      ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0)) {
    const int n2 = nc >> 1;
    for (int i = blockIdx.x; i < nr; i += gridDim.x) {
      const double2* sp = reinterpret_cast<const double2*>(src + idx[i0 + i] * src_ld);
      double2* dp = reinterpret_cast<double2*>(d + (int64_t)i * ld);
      for (int c = tc; c < n2; c += 256) dp[c] = sp[c];
    }
    return;
  }
  for (int i = blockIdx.x * rps + tr; i < nr; i += gridDim.x * rps) {
    const double* sp = src + idx[i0 + i] * src_ld;
    double* dp = d + (int64_t)i * ld;
    if (col)
      for (int c = tc; c < nc; c += tpr) dp[c] = sp[col[c0 + c]];
    else
      for (int c = tc; c < nc; c += tpr) dp[c] = sp[c];
  }
}

__global__ void k_scatter_rows(const int64_t* __restrict__ idx_off,
                               const int64_t* __restrict__ idx,
                               const int64_t* __restrict__ col_off,
                               const int64_t* __restrict__ col, int64_t ncols,
                               const double* __restrict__ src,
                               const int64_t* __restrict__ src_off,
                               const int64_t* __restrict__ src_ld, double* __restrict__ dst,
                               int64_t dst_ld, int accumulate, double alpha) {
  const int64_t b = blockIdx.y;
  const int64_t i0 = idx_off[b];
  const int nr = (int)(idx_off[b + 1] - i0);
  const int64_t c0 = col ? col_off[b] : 0;
  const int nc = (int)(col ? col_off[b + 1] - c0 : ncols);
  const double* s = src + src_off[b];
  const int64_t ld = src_ld[b];
  const int tpr = row_tpr(nc), rps = 256 / tpr;
  const int tr = threadIdx.x / tpr, tc = threadIdx.x - tr * tpr;
  if (!col && !accumulate && tpr == 256 && !(nc & 1) && !(dst_ld & 1) && !(ld & 1) &&
      !(src_off[b] & 1) && ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0)) {
    const int n2 = nc >> 1;
    for (int i = blockIdx.x; i < nr; i += gridDim.x) {
      const double2* sp = reinterpret_cast<const double2*>(s + (int64_t)i * ld);
      double2* dp = reinterpret_cast<double2*>(dst + idx[i0 + i] * dst_ld);
      for (int c = tc; c < n2; c += 256) dp[c] = sp[c];
    }
    return;
  }
  for (int i = blockIdx.x * rps + tr; i < nr; i += gridDim.x * rps) {
    const double* sp = s + (int64_t)i * ld;
    double* dp = dst + idx[i0 + i] * dst_ld;
    for (int c = tc; c < nc; c += tpr) {
      double* o = dp + (col ? col[c0 + c] : c);
      const double v = sp[c];
      if (accumulate) *o += alpha * v;
      else *o = v;
    }
  }
}

__global__ void k_schur_acc(int64_t q, const int64_t* __restrict__ row_off,
                            const int64_t* __restrict__ contrib, const double* __restrict__ part,
                            double* __restrict__ schur) {
  const int64_t row = blockIdx.y;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= q) return;
  double v = schur[row * q + c];
  for (int64_t t = row_off[row]; t < row_off[row + 1]; ++t) v += part[contrib[t] + c];
  schur[row * q + c] = v;
}

__global__ void k_diag_fill(int64_t n, double* dst, int64_t ld, double dv, const double* src,
                            int64_t sld, double scale) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    double v = (i == j) ? dv : 0.0;
    if (src) v = v + scale * src[i * sld + j];
    dst[i * ld + j] = v;
  }
}

__global__ void k_fill_rows(const int64_t* __restrict__ idx, int64_t nidx, double* dst,
                            int64_t ld, int64_t ncols, double v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nidx * ncols;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncols, c = t - i * ncols;
    dst[idx[i] * ld + c] = v;
  }
}

__global__ void k_sum_parts(int64_t count, int nparts, const double* __restrict__ parts,
                            int64_t stride, const double* C, double alpha, double* D) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += parts[p * stride + e];
    D[e] = (C ? C[e] : 0.0) + alpha * acc;
  }
}

// Error-free transformations (Knuth TwoSum, FMA TwoProduct) for the
// compensated Psi^T z reductions.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// out[c][j] = C[c][j] + alpha * sum_{t in col c} psi[rows[t]*ldp + c] * z[rows[t]*ldz + j],
// summed in list order with double-double (Dot2) accuracy.
__global__ void k_psi_dot(const int64_t* __restrict__ col_off, const int64_t* __restrict__ rows,
                          const double* __restrict__ psi, int64_t ldp,
                          const double* __restrict__ z, int64_t ldz, int64_t nrhs,
                          const double* C, int64_t ldc, double alpha, double* out, int64_t ldo) {
  const int64_t c = blockIdx.x;
  const int64_t t0 = col_off[c], t1 = col_off[c + 1];
  for (int64_t j = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; j < nrhs;
       j += (int64_t)gridDim.y * blockDim.x) {
    double s = 0.0, e = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t i = rows[t];
      const double a = psi[i * ldp + c], b = z[i * ldz + j];
      const double p = a * b;
      const double pe = fma(a, b, -p);
      double s2, se;
      two_sum(s, p, s2, se);
      s = s2;
      e += se + pe;
    }
    const double v = s + e;
    out[c * ldo + j] = (C ? C[c * ldc + j] : 0.0) + alpha * v;
  }
}

}  // namespace skb

using namespace skb;

extern "C" int skb_psi_dot(int64_t q, const int64_t* col_off, const int64_t* rows, const double* psi,
                           int64_t ldp, const double* z, int64_t ldz, int64_t nrhs, const double* C,
                           int64_t ldc, double alpha, double* out, int64_t ldo, void* stream) {
  if (q <= 0 || nrhs <= 0) return 0;
  const int nt = nrhs >= 128 ? 128 : (nrhs >= 32 ? 32 : 32);
  dim3 grid((unsigned)q, (unsigned)((nrhs + nt - 1) / nt));
  k_psi_dot<<<grid, nt, 0, (cudaStream_t)stream>>>(col_off, rows, psi, ldp, z, ldz, nrhs, C, ldc, alpha,
                                                    out, ldo);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_sum_partials(int64_t count, int32_t nparts, const double* parts, int64_t stride,
                                const double* C, double alpha, double* D, void* stream) {
  if (count <= 0) return 0;
  k_sum_parts<<<grid_cap((count + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(
      count, nparts, parts, stride, C, alpha, D);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_fill_rows(int64_t nidx, const int64_t* idx, double* dst, int64_t ld,
                             const void* unused, int64_t ncols, double value, void* stream) {
  (void)unused;
  if (nidx <= 0 || ncols <= 0) return 0;
  k_fill_rows<<<grid_cap((nidx * ncols + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(
      idx, nidx, dst, ld, ncols, value);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_copy2d_batched(int64_t nbox, const SkbMat* dst, const SkbMat* src,
                                  int32_t trans, void* stream) {
  if (nbox <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t maxe = 0;
  for (int64_t b = 0; b < nbox; ++b) maxe = std::max(maxe, dst[b].rows * dst[b].cols);
  if (maxe == 0) return 0;
  SkbMat *dd = nullptr, *ds = nullptr;
  int rc = upload(dst, nbox, s, &dd);
  if (rc) return rc;
  if ((rc = upload(src, nbox, s, &ds))) return rc;
  ProfScope ps(F_MOVE, s);
  for (int64_t b0 = 0; b0 < nbox; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, nbox - b0);
    // 2 doubles x 4 passes per thread on the flat path
    dim3 grid(grid_cap((maxe + 2047) / 2048, nb > 64 ? 32 : 1024), (unsigned)nb);
    k_copy2d<<<grid, 256, 0, s>>>(dd + b0, ds + b0, trans);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(dd, s);
  cudaFreeAsync(ds, s);
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" int skb_gather_rows(int64_t nbox, const int64_t* idx_off, const int64_t* idx,
                               const int64_t* col_off, const int64_t* col, int64_t ncols,
                               const double* src, int64_t src_ld, double* dst,
                               const int64_t* dst_off, const int64_t* dst_ld, int64_t max_rows,
                               int64_t max_cols, void* stream) {
  if (nbox <= 0 || max_rows <= 0 || max_cols <= 0) return 0;
  if (nbox > 65535) return 2;
  // one row per 32..256 threads (row_tpr): blocks walk the rows of a box
  const int64_t rps_g = max_cols > 128 ? 1 : (max_cols > 64 ? 2 : (max_cols > 32 ? 4 : 8));
  dim3 grid(grid_cap((max_rows + rps_g - 1) / rps_g, nbox > 64 ? 64 : 1024), (unsigned)nbox);
  ProfScope ps(F_MOVE, (cudaStream_t)stream);
  k_gather_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(idx_off, idx, col_off, col, ncols, src,
                                                        src_ld, dst, dst_off, dst_ld);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_scatter_rows(int64_t nbox, const int64_t* idx_off, const int64_t* idx,
                                const int64_t* col_off, const int64_t* col, int64_t ncols,
                                const double* src, const int64_t* src_off,
                                const int64_t* src_ld, double* dst, int64_t dst_ld,
                                int32_t accumulate, double alpha, int64_t max_rows,
                                int64_t max_cols, void* stream) {
  if (nbox <= 0 || max_rows <= 0 || max_cols <= 0) return 0;
  if (nbox > 65535) return 2;
  const int64_t rps_s = max_cols > 128 ? 1 : (max_cols > 64 ? 2 : (max_cols > 32 ? 4 : 8));
  dim3 grid(grid_cap((max_rows + rps_s - 1) / rps_s, nbox > 64 ? 64 : 1024), (unsigned)nbox);
  ProfScope ps(F_MOVE, (cudaStream_t)stream);
  k_scatter_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(idx_off, idx, col_off, col, ncols, src,
                                                         src_off, src_ld, dst, dst_ld, accumulate,
                                                         alpha);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_schur_accumulate(int64_t q, const int64_t* row_off, const int64_t* contrib,
                                    const double* part, double* schur, void* stream) {
  if (q <= 0) return 0;
  dim3 grid((unsigned)((q + 127) / 128), (unsigned)q);
  k_schur_acc<<<grid, 128, 0, (cudaStream_t)stream>>>(q, row_off, contrib, part, schur);
  SKB_LAUNCH_CHECK();
  return 0;
}

extern "C" int skb_diag_fill(int64_t n, double* dst, int64_t ld, double diag_val,
                             const double* src, int64_t src_ld, double scale, void* stream) {
  if (n <= 0) return 0;
  k_diag_fill<<<grid_cap((n * n + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(
      n, dst, ld, diag_val, src, src_ld, scale);
  SKB_LAUNCH_CHECK();
  return 0;
}

namespace skb {
Prof& prof() {
  static Prof p;
  return p;
}
// The native level engine thread has its own side streams: its size classes
// neither serialise behind the Python thread's Schur / sweep classes nor share
// their fork/join events.
thread_local bool t_engine_side = false;
SideStreams& side() {
  static SideStreams s;
  static SideStreams se;
  return t_engine_side ? se : s;
}
void use_engine_side(bool on) { t_engine_side = on; }
CaptureSession& capture() {
  static CaptureSession c;
  return c;
}
thread_local bool t_engine_ring = false;
PinnedRing& ring() {
  static PinnedRing r;
  static PinnedRing re;        // the native level engine thread's own ring
  return t_engine_ring ? re : r;
}
void use_engine_ring(bool on) { t_engine_ring = on; }
cudaMemPool_t& tl_pool() {
  thread_local cudaMemPool_t p = nullptr;
  return p;
}
std::recursive_mutex& host_mutex() {
  static std::recursive_mutex m;
  return m;
}
static std::vector<std::vector<void*>> g_sessions;
}  // namespace skb

extern "C" int skb_version(void) { return 1; }

// Factor storage (per-level factor slabs, sweep stashes): a process-wide
// stream-ordered pool that never shrinks.  Torch's caching allocator falls
// back to cudaMalloc -- which waits for the device -- whenever an update's
// slab sizes do not fit its cached blocks (10-25 ms stalls in update chains).
static cudaMemPool_t factor_pool() {
  static cudaMemPool_t pool = nullptr;
  static std::mutex m;
  std::lock_guard<std::mutex> lk(m);
  if (!pool) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pool;
}

extern "C" int skb_dev_alloc(int64_t bytes, void* stream, uint64_t* out) {
  cudaMemPool_t pool = factor_pool();
  if (!pool) return 11;
  // Sizes of 1 MB and more are rounded up to eight steps per octave: the slabs
  // and sweep stashes of successive updates differ by a few percent, and an
  // exact-size request that no freed block fits makes the pool map new
  // physical memory (a 0.3 s stall for a 700 MB stash on cfg3 update chains).
  size_t want = (size_t)(bytes > 0 ? bytes : 8);
  if (want >= ((size_t)1 << 20)) {
    int lg = 63 - __builtin_clzll((unsigned long long)want);
    const size_t gran = (size_t)1 << (lg - 3);
    want = (want + gran - 1) & ~(gran - 1);
  }
  void* p = nullptr;
  SKB_RET(cudaMallocFromPoolAsync(&p, want, pool, (cudaStream_t)stream));
  *out = (uint64_t)p;
  return 0;
}

extern "C" int skb_dev_free(uint64_t ptr, void* stream) {
  if (!ptr) return 0;
  SKB_RET(cudaFreeAsync((void*)ptr, (cudaStream_t)stream));
  return 0;
}

// Synchronous device -> host copy of raw bytes (factor inspection: BoxFactors.lu pivots).
extern "C" int skb_d2h(void* host, const void* dev, int64_t bytes) {
  if (bytes <= 0) return 0;
  SKB_RET(cudaMemcpy(host, dev, (size_t)bytes, cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int skb_capture_begin(int64_t arena_bytes) {
  auto& C = skb::capture();
  C.pinned.clear();
  C.size = (size_t)(arena_bytes > 0 ? arena_bytes : (16 << 20));
  C.used = 0;
  void* h = nullptr;
  cudaError_t e = cudaHostAlloc(&h, C.size, cudaHostAllocDefault);
  if (e != cudaSuccess) return -(int)e;
  C.arena = (char*)h;
  C.pinned.push_back(h);
  C.on = true;
  return 0;
}

extern "C" int skb_h2d(const void* host, int64_t bytes, void* dev, void* stream) {
  if (bytes <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  auto& C = skb::capture();
  if (C.on) {
    const size_t off = (C.used + 255) & ~(size_t)255;
    if (off + (size_t)bytes > C.size) return 5;        // arena exhausted
    memcpy(C.arena + off, host, (size_t)bytes);
    C.used = off + (size_t)bytes;
    SKB_RET(cudaMemcpyAsync(dev, C.arena + off, (size_t)bytes, cudaMemcpyHostToDevice, s));
    return 0;
  }
  return skb::ring_stage(host, (size_t)bytes, s, dev);
}

extern "C" int skb_capture_end(void) {
  skb::capture().on = false;
  skb::g_sessions.push_back(skb::capture().pinned);
  skb::capture().pinned.clear();
  return (int)skb::g_sessions.size();          // session id (1-based)
}

extern "C" int skb_capture_release(int32_t session) {
  if (session < 1 || session > (int)skb::g_sessions.size()) return 1;
  for (void* h : skb::g_sessions[session - 1]) cudaFreeHost(h);
  skb::g_sessions[session - 1].clear();
  return 0;
}

extern "C" int skb_prof_enable(int32_t on) {
  skb::prof().on = on != 0;
  return 0;
}

extern "C" int skb_prof_add(int32_t fam, double flops, double bytes) {
  if (fam < 0 || fam >= skb::F_NFAM) return 1;
  skb::prof().flops[fam] += flops;
  skb::prof().bytes[fam] += bytes;
  return 0;
}

extern "C" int skb_prof_read(double* ms_out, int64_t* count_out, double* flops_out,
                             double* bytes_out, int32_t reset) {
  auto& P = skb::prof();
  for (int f = 0; f < skb::F_NFAM; ++f) {
    double ms = 0.0;
    for (auto& e : P.ev[f]) {
      float t = 0.f;
      cudaEventSynchronize(e.second);
      cudaEventElapsedTime(&t, e.first, e.second);
      ms += t;
    }
    ms_out[f] = ms;
    count_out[f] = (int64_t)P.ev[f].size();
    flops_out[f] = P.flops[f];
    bytes_out[f] = P.bytes[f];
    if (reset) {
      for (auto& e : P.ev[f]) { P.pool.push_back(e.first); P.pool.push_back(e.second); }
      P.ev[f].clear();
      P.flops[f] = 0.0;
      P.bytes[f] = 0.0;
    }
  }
  return 0;
}

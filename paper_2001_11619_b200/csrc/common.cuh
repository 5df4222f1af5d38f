// Shared helpers for the sm_100a skeletonization kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <utility>
#include <vector>

#include "../../include/skelb200.h"

#define SKB_RET(expr)                                              \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return -(int)_e;                        \
  } while (0)

#define SKB_LAUNCH_CHECK() SKB_RET(cudaGetLastError())

namespace skb {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fp64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  SASS: DMMA.
// Fragment ownership (PTX ISA, m8n8k4 .f64): A[lane>>2][lane&3],
// B[lane&3][lane>>2], C/D[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// CUDA-graph capture support: while a capture session is open, descriptor
// uploads are staged through pinned host blocks that live as long as the
// session (the captured memcpy nodes read them at every replay).
struct CaptureSession {
  bool on = false;
  char* arena = nullptr;       // pinned, allocated before the capture starts
  size_t size = 0, used = 0;
  std::vector<void*> pinned;   // arenas owned by this session
};
CaptureSession& capture();

// Pinned staging ring for descriptor uploads (asynchronous H2D copies).  The
// ring is split into slots; a slot is rewritten (one lap later) only after
// every copy that read it has completed.  Copies are issued on several streams
// (compression, level, sweep streams) that progress independently, so each
// slot keeps one event per stream that copied from it in the current lap.
struct PinnedRing {
  static constexpr size_t kSize = 64u << 20, kSlot = 1u << 20, kSlots = kSize / kSlot;
  static constexpr int kPerSlot = 8;
  struct Slot {
    uint64_t lap = 0;
    int n = 0;
    cudaStream_t st[kPerSlot];
    cudaEvent_t ev[kPerSlot];
  };
  char* base = nullptr;
  size_t head = 0;
  uint64_t lap = 1;
  Slot slot[kSlots];
  std::vector<cudaEvent_t> pool;
  std::mutex mu;                 // per ring: a wait on a lap wrap never blocks the other thread's ring
};
PinnedRing& ring();
// host-side state shared by the Python thread and the native level engine
// thread (pinned ring, shared-memory opt-in table, profiling timers)
std::recursive_mutex& host_mutex();

inline int pool_strict(cudaMemPool_t pool) {
  int zero = 0;
  SKB_RET(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &zero));
  SKB_RET(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &zero));
  return 0;
}

inline int ring_stage(const void* host, size_t bytes, cudaStream_t s, void* dev) {
  PinnedRing& R = ring();
  std::lock_guard<std::mutex> lk(R.mu);
  if (!R.base) {
    // keep stream-ordered allocations cached in the pool across synchronisations
    int dev = 0;
    cudaMemPool_t pool;
    SKB_RET(cudaGetDevice(&dev));
    SKB_RET(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~0ull;
    SKB_RET(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // SKB_POOL_STRICT=1 (debug): cross-stream reuse only through explicit event
    // dependencies (no opportunistic reuse, no inserted waits)
    if (getenv("SKB_POOL_STRICT")) {
      const int prc = pool_strict(pool);
      if (prc) return prc;
    }
    SKB_RET(cudaHostAlloc((void**)&R.base, PinnedRing::kSize, cudaHostAllocDefault));
  }
  if (bytes > PinnedRing::kSize / 2) {      // oversized: plain (pageable) copy
    SKB_RET(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
    return 0;
  }
  size_t off = (R.head + 255) & ~(size_t)255;
  if (off + bytes > PinnedRing::kSize) { off = 0; ++R.lap; }
  const size_t s0 = off / PinnedRing::kSlot, s1 = (off + bytes - 1) / PinnedRing::kSlot;
  // data written in a previous lap may still be in flight in this region
  for (size_t k = s0; k <= s1; ++k) {
    PinnedRing::Slot& S = R.slot[k];
    if (S.lap != R.lap) {
      for (int i = 0; i < S.n; ++i) {
        SKB_RET(cudaEventSynchronize(S.ev[i]));
        R.pool.push_back(S.ev[i]);
      }
      S.n = 0;
      S.lap = R.lap;
    }
  }
  memcpy(R.base + off, host, bytes);
  SKB_RET(cudaMemcpyAsync(dev, R.base + off, bytes, cudaMemcpyHostToDevice, s));
  for (size_t k = s0; k <= s1; ++k) {
    PinnedRing::Slot& S = R.slot[k];
    int i = 0;
    while (i < S.n && S.st[i] != s) ++i;
    if (i == S.n) {
      if (S.n == PinnedRing::kPerSlot) {
        // too many streams on one slot: drain the oldest entries now
        for (int j = 0; j < S.n; ++j) SKB_RET(cudaEventSynchronize(S.ev[j]));
        for (int j = 0; j < S.n; ++j) R.pool.push_back(S.ev[j]);
        S.n = 0;
        i = 0;
      }
      cudaEvent_t e;
      if (R.pool.empty()) {
        SKB_RET(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      } else {
        e = R.pool.back();
        R.pool.pop_back();
      }
      S.st[i] = s;
      S.ev[i] = e;
      S.n = i + 1;
    }
    SKB_RET(cudaEventRecord(S.ev[i], s));     // latest copy of stream s from this slot
  }
  R.head = off + bytes;
  return 0;
}

// Opt a kernel into the largest dynamic shared memory once (changing the
// attribute between launches can serialise the device).
inline cudaError_t smem_optin(const void* fn) {
  std::lock_guard<std::recursive_mutex> lk(host_mutex());
  static std::vector<const void*> done;
  for (const void* f : done)
    if (f == fn) return cudaSuccess;
  int dev = 0, mx = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.push_back(fn);
  return e;
}

// Stream-ordered allocation from the calling thread's pool: the native level
// engine thread allocates from a pool of its own, so its allocations never
// share a pool with the Python thread's (cross-stream reuse stays per thread).
cudaMemPool_t& tl_pool();
inline cudaError_t malloc_async(void** p, size_t n, cudaStream_t s) {
  cudaMemPool_t pl = tl_pool();
  return pl ? cudaMallocFromPoolAsync(p, n, pl, s) : cudaMallocAsync(p, n, s);
}

// Copy host descriptors to a stream-ordered device buffer (freed async by caller).
template <typename T>
inline int upload(const T* host, int64_t n, cudaStream_t s, T** dev) {
  *dev = nullptr;
  if (n <= 0) return 0;
  SKB_RET(malloc_async((void**)dev, sizeof(T) * n, s));
  if (capture().on) {
    CaptureSession& C = capture();
    const size_t off = (C.used + 255) & ~(size_t)255;
    if (off + sizeof(T) * n > C.size) return 5;         // arena exhausted
    void* h = C.arena + off;
    C.used = off + sizeof(T) * n;
    memcpy(h, host, sizeof(T) * n);
    SKB_RET(cudaMemcpyAsync(*dev, h, sizeof(T) * n, cudaMemcpyHostToDevice, s));
  } else {
    const int rc = ring_stage(host, sizeof(T) * n, s, *dev);
    if (rc) return rc;
  }
  return 0;
}

inline int grid_cap(int64_t want, int64_t cap) {
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// ---- live per-kernel-family timing (CUDA events on the launching stream) ----
enum Family { F_ASSEMBLE = 0, F_GEQRF, F_QRCP, F_IDT, F_GEMM, F_GETRF, F_TRSM, F_MOVE, F_NFAM };

struct Prof {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[F_NFAM];
  std::vector<cudaEvent_t> pool;
  double flops[F_NFAM] = {0};
  double bytes[F_NFAM] = {0};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
  }
};
Prof& prof();

struct ProfScope {
  int fam;
  cudaStream_t s;
  cudaEvent_t a{}, b{};
  ProfScope(int f, cudaStream_t st) : fam(f), s(st) {
    if (prof().on) {
      std::lock_guard<std::recursive_mutex> lk(host_mutex());
      a = prof().get(); b = prof().get(); cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (prof().on) {
      std::lock_guard<std::recursive_mutex> lk(host_mutex());
      cudaEventRecord(b, s); prof().ev[fam].push_back({a, b});
    }
  }
};

// Side streams for running independent size classes of a batch concurrently
// (different dynamic shared memory footprints -> different CTAs per SM).
struct SideStreams {
  static constexpr int kN = 8;
  bool init = false;
  cudaStream_t st[kN];
  cudaEvent_t fork_ev, join_ev[kN];
};
SideStreams& side();
void use_engine_side(bool on);

inline int side_init() {
  SideStreams& S = side();
  if (!S.init) {
    // the size classes of the QR / QRCP are the factorization's critical path:
    // highest stream priority, so they win the SMs over the Schur / sweep work
    int least = 0, greatest = 0;
    SKB_RET(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    for (int i = 0; i < SideStreams::kN; ++i) {
      SKB_RET(cudaStreamCreateWithPriority(&S.st[i], cudaStreamNonBlocking, greatest));
      SKB_RET(cudaEventCreateWithFlags(&S.join_ev[i], cudaEventDisableTiming));
    }
    SKB_RET(cudaEventCreateWithFlags(&S.fork_ev, cudaEventDisableTiming));
    S.init = true;
  }
  return 0;
}

// side streams 0..n-1 wait for everything enqueued on s so far.  Record and
// waits are one critical section: the events are shared by every caller of
// this thread's stream set (an interleaved re-record would let a side stream
// wait on the wrong point of another stream -- a run-to-run race).
inline int fork_n(cudaStream_t s, int n) {
  std::lock_guard<std::recursive_mutex> lk(host_mutex());
  SKB_RET((cudaError_t)(-side_init()));
  SideStreams& S = side();
  SKB_RET(cudaEventRecord(S.fork_ev, s));
  for (int i = 0; i < n; ++i) SKB_RET(cudaStreamWaitEvent(S.st[i], S.fork_ev, 0));
  return 0;
}

// s waits for everything enqueued on side streams 0..n-1
inline int join_n(cudaStream_t s, int n) {
  std::lock_guard<std::recursive_mutex> lk(host_mutex());
  SideStreams& S = side();
  for (int i = 0; i < n; ++i) {
    SKB_RET(cudaEventRecord(S.join_ev[i], S.st[i]));
    SKB_RET(cudaStreamWaitEvent(s, S.join_ev[i], 0));
  }
  return 0;
}

inline int fork3(cudaStream_t s) { return fork_n(s, 3); }
inline int join3(cudaStream_t s) { return join_n(s, 3); }
inline int fork2(cudaStream_t s) { return fork_n(s, 2); }
inline int join2(cudaStream_t s) { return join_n(s, 2); }

}  // namespace skb

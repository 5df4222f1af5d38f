// clock64 breakdown of the cluster QR k_geqrf_cl (box 0): per panel step and
// cluster rank -- step start (after the cluster barrier), look-ahead apply,
// panel factorisation, remaining trailing update.
//   nvcc -DSKB_QR_TIMING -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     scripts/native/qrcl_timing.cu build_obj/{gemm,lu,misc}.o -o qrcl_timing
#include "../../paper_2001_11619_b200/csrc/qr.cu"
#include <cstdio>
#include <vector>
#include <random>

int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 912, n = argc > 2 ? atoi(argv[2]) : 464;
  int B = argc > 3 ? atoi(argv[3]) : 4;
  std::vector<double> h((size_t)m * n * B);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(g);
  double* d;
  cudaMalloc(&d, h.size() * 8);
  std::vector<int64_t> mm(B, m), nn(B, n), A(B);
  for (int b = 0; b < B; ++b) A[b] = (int64_t)(d + (size_t)b * m * n);
  float ms = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 4; ++it) {
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    skb::geqrf_batched(B, mm.data(), nn.data(), mm.data(), A.data(), 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
  }
  long long t[4096];
  cudaMemcpyFromSymbol(t, skb::g_qr_t, sizeof(t));
  printf("m %d n %d B %d: %.3f ms  err %s\n", m, n, B, ms, cudaGetErrorString(cudaGetLastError()));
  const int P = m <= 1024 ? 16 : 8, np_ = (n + P - 1) / P;
  const int CL = np_ <= 8 ? 2 : (np_ <= 16 ? 4 : 8);
  long long t0 = t[0];
  for (int p = 0; p < np_ && p < 128; ++p) {
    const int own = (p + 1) % CL;
    long long* q = t + own * 512 + p * 4;
    long long* o = t + (p % CL) * 512 + p * 4;
    printf("step %2d: at %7lld  next-owner r%d: copy %6lld apply %6lld panel %6lld | r%d total %6lld\n", p,
           q[0] - t0, own, q[1] - q[0], q[2] - q[1], q[3] - q[2], p % CL, o[3] - o[0]);
  }
  return 0;
}

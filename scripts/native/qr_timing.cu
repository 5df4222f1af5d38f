// clock64 breakdown of the fused per-box QR (block 0): build with
//   nvcc -DSKB_QR_TIMING ... scripts/native/qr_timing.cu + the library objects
#include "../../paper_2001_11619_b200/csrc/qr.cu"
#include <cstdio>
#include <vector>
#include <random>

int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 512, n = argc > 2 ? atoi(argv[2]) : 96;
  int B = argc > 3 ? atoi(argv[3]) : 1;
  std::vector<double> h((size_t)m * n * B);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(g);
  double* d;
  cudaMalloc(&d, h.size() * 8);
  std::vector<int64_t> mm(B, m), nn(B, n), A(B);
  for (int b = 0; b < B; ++b) A[b] = (int64_t)(d + (size_t)b * m * n);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    skb::geqrf_batched(B, mm.data(), nn.data(), mm.data(), A.data(), 0);
    cudaDeviceSynchronize();
  }
  long long t[4096];
  cudaMemcpyFromSymbol(t, skb::g_qr_t, sizeof(t));
  printf("m %d n %d B %d err %s\n", m, n, B, cudaGetErrorString(cudaGetLastError()));
  const char* nm[7] = {"load", "cols", "RV", "gram", "T", "trail", ""};
  long long t0 = t[0];
  for (int p = 0; p * 16 < n && p < 64; ++p) {
    printf("panel %2d:", p);
    for (int k = 0; k < 6; ++k) printf(" %s %6lld", nm[k], t[p * 8 + k + 1] - t[p * 8 + k]);
    printf("  (at %lld)\n", t[p * 8] - t0);
  }
  for (int c = 0; c < 16; ++c)
    printf("col %2d: part+bfly %5lld bar1 %5lld sum+bar2.. %5lld  update+next %5lld\n", c,
           t[2048 + c * 4 + 1] - t[2048 + c * 4], t[2048 + c * 4 + 2] - t[2048 + c * 4 + 1],
           t[2048 + c * 4 + 3] - t[2048 + c * 4 + 2],
           c < 15 ? t[2048 + (c + 1) * 4] - t[2048 + c * 4 + 3] : 0);
  return 0;
}

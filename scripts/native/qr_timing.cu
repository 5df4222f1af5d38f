// clock64 breakdown of the fused per-box QR (block 0): build with
//   nvcc -DSKB_QR_TIMING ... scripts/native/qr_timing.cu + the library objects
#include "../../paper_2001_11619_b200/csrc/qr.cu"
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>

int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 512, n = argc > 2 ? atoi(argv[2]) : 96;
  int B = argc > 3 ? atoi(argv[3]) : 1;
  const bool qrcp = argc > 4 && argv[4][0] == 'q';
  std::vector<double> h((size_t)m * n * B);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(g);
  double* d;
  cudaMalloc(&d, h.size() * 8);
  std::vector<int64_t> mm(B, m), nn(B, n), A(B);
  for (int b = 0; b < B; ++b) A[b] = (int64_t)(d + (size_t)b * m * n);
  // QRCP input: a numerically rank-deficient matrix (column scales 10^(-20 j/n))
  if (qrcp)
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < n; ++j)
        for (int r = 0; r < m; ++r) h[(size_t)b * m * n + (size_t)j * m + r] *= pow(10.0, -20.0 * j / n) * (1.0 + 0.1 * r / m);
  int32_t *perm, *ko;
  double *diag, *gap;
  cudaMalloc(&perm, 4 * n * B); cudaMalloc(&ko, 8 * B); cudaMalloc(&diag, 8 * n * B); cudaMalloc(&gap, 8 * B);
  std::vector<int64_t> kmin(B, 0), poff(B + 1);
  for (int b = 0; b <= B; ++b) poff[b] = (int64_t)b * n;
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    if (qrcp)
      skb::qrcp_batched(B, mm.data(), nn.data(), mm.data(), A.data(), kmin.data(), 1e-10, poff.data(),
                        perm, diag, ko, ko + B, gap, 0);
    else
      skb::geqrf_batched(B, mm.data(), nn.data(), mm.data(), A.data(), 0);
    cudaDeviceSynchronize();
  }
  long long t[4096];
  cudaMemcpyFromSymbol(t, skb::g_qr_t, sizeof(t));
  printf("m %d n %d B %d err %s\n", m, n, B, cudaGetErrorString(cudaGetLastError()));
  const char* nm[7] = {"load", "cols", "RV", "gram", "T", "trail", ""};
  if (qrcp) {
    for (int i = 0; i < 40; ++i) {
      long long* q = t + 3000 + i * 8;
      printf("step %3d: cand %5lld bar %5lld merge %5lld hh %5lld upd %5lld down %5lld recomp %5lld\n", i,
             q[1] - q[0], q[2] - q[1], q[3] - q[2], q[4] - q[3], q[5] - q[4], q[6] - q[5], q[8] - q[6]);
    }
    return 0;
  }
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

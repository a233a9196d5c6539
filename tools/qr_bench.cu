// Blocked Householder QR (dense.cu householder_qr, the low-rank basis
// rebuild) on an m x n random matrix: ms per call (Q formed), max |Q^T Q - I|
// on a few columns.  Build like tools/lu_bench.cu; run: tools/qr_bench m n [reps]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "dense.cuh"

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

__global__ void fill(long long n, unsigned long long seed, double* a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    a[i] = (double)(z >> 11) * 0x1.0p-53 - 0.5;
  }
}

int main(int argc, char** argv) {
  const long long m = argc > 1 ? std::atoll(argv[1]) : 1048576;
  const int n = argc > 2 ? std::atoi(argv[2]) : 600;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 2;
  double *a, *a0, *q, *r, *tau, *work;
  const size_t wd = rtlr::cuda::householder_qr_work(m, n);
  CK(cudaMalloc(&a, m * n * 8));
  CK(cudaMalloc(&a0, m * n * 8));
  CK(cudaMalloc(&q, m * n * 8));
  CK(cudaMalloc(&r, (size_t)n * n * 8));
  CK(cudaMalloc(&tau, n * 8));
  CK(cudaMalloc(&work, wd * 8));
  fill<<<1184, 256>>>(m * n, 7, a0);
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  auto run = [&] {
    CK(cudaMemcpyAsync(a, a0, m * n * 8, cudaMemcpyDeviceToDevice, s));
    rtlr::cuda::householder_qr(m, n, a, m, tau, q, m, r, work, wd, s);
  };
  run();
  CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) run();
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  std::vector<double> h(m * 2);
  CK(cudaMemcpy(h.data(), q, m * 2 * 8, cudaMemcpyDeviceToHost));
  double d00 = 0, d01 = 0;
  for (long long i = 0; i < m; ++i) d00 += h[i] * h[i], d01 += h[i] * h[m + i];
  std::printf("m %lld n %d: %.2f ms per QR (incl. a %.1f GB device copy), |q0|^2-1 %.1e, q0.q1 %.1e\n", m, n,
              ms / reps, m * n * 8e-9, d00 - 1, d01);
  return 0;
}

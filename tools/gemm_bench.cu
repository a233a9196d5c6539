// A^T B timing (dense.cu gemm_tn) for the low-rank shapes: M = r, N columns,
// K = N_x; with "nn" as the fifth argument A B (gemm_nn: X C, M = N_x rows,
// K = r).  Build like tools/lu_bench.cu; run: tools/gemm_bench M N K [reps] [nn].
// Prints ms per call, TFLOP/s (2 M N K) and the max |C - C_ref| / max|C_ref|
// against a host evaluation of a few columns.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
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

int main(int argc, char** argv) {
  const int M = argc > 1 ? std::atoi(argv[1]) : 600;
  const int N = argc > 2 ? std::atoi(argv[2]) : 40;
  const long long K = argc > 3 ? std::atoll(argv[3]) : 1048576;
  const int reps = argc > 4 ? std::atoi(argv[4]) : 10;
  const bool nn = argc > 5 && std::string(argv[5]) == "nn";
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> A(static_cast<size_t>(K) * M), B(static_cast<size_t>(K) * N);
  for (auto& v : A) v = u(g);
  for (auto& v : B) v = u(g);
  double *dA, *dB, *dC, *dw;
  const size_t wd = rtlr::cuda::gemm_tn_work(M, N, K);
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMalloc(&dB, B.size() * 8));
  CK(cudaMalloc(&dC, static_cast<size_t>(M) * N * 8));
  CK(cudaMalloc(&dw, std::max<size_t>(wd, 1) * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  // tn: A is K x M (ld K), B K x N (ld K); nn: A is M x K (ld M), B K x N (ld K)
  auto run = [&] {
    if (nn)
      rtlr::cuda::gemm_nn(M, N, static_cast<int>(K), dA, M, dB, K, dC, M, s);
    else
      rtlr::cuda::gemm_tn(M, N, K, dA, K, dB, K, dC, M, dw, wd, s);
  };
  run();
  CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < reps; ++i) run();
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= reps;
  std::vector<double> C(static_cast<size_t>(M) * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost));
  double err = 0.0, big = 0.0;
  for (int n = 0; n < N; n += std::max(1, N / 4))
    for (int m = 0; m < M; m += std::max(1, M / 16)) {
      double acc = 0.0;
      for (long long k = 0; k < K; ++k)
        acc += (nn ? A[m + static_cast<size_t>(k) * M] : A[k + static_cast<size_t>(m) * K]) * B[k + static_cast<size_t>(n) * K];
      err = std::max(err, std::fabs(C[m + static_cast<size_t>(n) * M] - acc));
      big = std::max(big, std::fabs(acc));
    }
  std::printf("M %d N %d K %lld: %.3f ms, %.2f TFLOP/s, rel err %.2e\n", M, N, K, ms, 2.0 * M * N * K / (ms * 1e-3) * 1e-12,
              err / big);
  return err / big < 1e-12 ? 0 : 1;
}

// fp64 tensor-pipe (DMMA) peak on this GPU, the denominator of the low-rank
// contractions' roofline fractions: (1) a register-only loop of independent
// mma.sync.m8n8k4.f64 per warp (no memory traffic), (2) cuBLAS DGEMM at
// 8192^3 (the library's reachable fp64 throughput).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dmma_peak.cu -o tools/dmma_peak -lcublas
// Run:   tools/dmma_peak   (one JSON line)
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

constexpr int kChains = 8;  // independent accumulators per warp (hides DMMA latency)

__global__ void dmma_loop(int iters, double* out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
  double c[kChains][2];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // DMMA loop: sms x 4 CTAs x 8 warps
  double best = 0.0;
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    const int blocks = sms * 4;
    dmma_loop<<<blocks, warps * 32>>>(iters, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dmma_loop<<<blocks, warps * 32>>>(iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 512.0 * kChains * iters * static_cast<double>(blocks) * warps;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  // cuBLAS DGEMM 8192^3
  const int n = 8192;
  double *A, *B, *C;
  CK(cudaMalloc(&A, sizeof(double) * n * n));
  CK(cudaMalloc(&B, sizeof(double) * n * n));
  CK(cudaMalloc(&C, sizeof(double) * n * n));
  CK(cudaMemset(A, 0, sizeof(double) * n * n));
  CK(cudaMemset(B, 0, sizeof(double) * n * n));
  cublasHandle_t h;
  cublasCreate(&h);
  const double one = 1.0, zero = 0.0;
  for (int i = 0; i < 2; ++i) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double dgemm = 2.0 * n * n * static_cast<double>(n) * reps / (ms * 1e-3) / 1e12;
  std::printf("{\"dmma_loop_tflops\": %.2f, \"cublas_dgemm_8192_tflops\": %.2f, \"sms\": %d}\n", best, dgemm, sms);
  return 0;
}

// Latency probe for the small-batch LU panel: what does one CTA of 256
// threads per system (16 CTAs) pay per column step?  Variants:
//  0 empty kernel; 1 32 x __syncthreads; 2 32 x (warp argmax + barrier);
//  3 = 2 + the 31-FMA row update from shared memory; 4 = 3 + a 600 x 32
//  panel load/store from global memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/panel_probe.cu -o tools/panel_probe
#include <cuda_runtime.h>
#include <cstdio>

__global__ void probe(int variant, double* g, int rows) {
  __shared__ double sh[2][8];
  __shared__ double urow[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double a[32];
  double* A = g + static_cast<size_t>(blockIdx.x) * rows * 32;
  if (variant == 4) {
    for (int c = 0; c < 32; ++c) a[c] = tid < rows ? A[tid + c * rows] : 0.0;
  } else {
    for (int c = 0; c < 32; ++c) a[c] = 1.0 + 1e-3 * (tid + c);
  }
  if (variant == 0) return;
  for (int j = 0; j < 32; ++j) {
    if (variant >= 2) {
      double v = fabs(a[0]);
      int idx = tid;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
          v = ov;
          idx = oi;
        }
      }
      if (lane == 0) sh[j & 1][wid] = v;
      if (tid == 0) urow[j] = a[0];
    }
    __syncthreads();
    if (variant >= 3) {
      double best = sh[j & 1][0];
      for (int w = 1; w < 8; ++w) best = fmax(best, sh[j & 1][w]);
      const double l = a[0] / (best + 1.0);
      if (variant == 5) {
#pragma unroll
        for (int c = 1; c < 32; ++c) a[c] -= l * 0.001 * c;
      } else {
#pragma unroll
        for (int c = 1; c < 32; ++c) a[c] -= l * urow[c];
      }
#pragma unroll
      for (int c = 0; c + 1 < 32; ++c) a[c] = a[c + 1];
      a[31] = 0.0;
    }
  }
  double s = 0.0;
  for (int c = 0; c < 32; ++c) s += a[c];
  if (variant == 4) {
    for (int c = 0; c < 32; ++c)
      if (tid < rows) A[tid + c * rows] = a[c];
  } else if (s == 12345.0) {
    g[0] = s;
  }
}

int main() {
  double* g;
  const int rows = 256, m = 16;
  cudaMalloc(&g, sizeof(double) * rows * 32 * m);
  cudaMemset(g, 0, sizeof(double) * rows * 32 * m);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v <= 5; ++v) {
    probe<<<m, 256>>>(v, g, rows);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int it = 0; it < 200; ++it) probe<<<m, 256>>>(v, g, rows);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("variant %d: %.2f us per launch\n", v, ms * 1e3 / 200);
  }
  return 0;
}

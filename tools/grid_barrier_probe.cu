// Cost of a grid-wide barrier for a cooperative launch of G CTAs x 256
// threads: cooperative_groups grid.sync() against a monotonic-counter
// barrier (one atomicAdd per CTA, acquire spin).  nvcc -arch=sm_100a -rdc=true
// is not needed: cg grid sync works in whole-program mode with
// cudaLaunchCooperativeKernel.  Usage: grid_barrier_probe [ctas] [iters]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void counter_barrier(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (static_cast<int>(v - epoch) < 0);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 2) probe(int mode, int iters, unsigned* bar, double* sink) {
  cg::grid_group grid = cg::this_grid();
  unsigned epoch = 0;
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    if (mode == 0)
      grid.sync();
    else
      counter_barrier(bar, epoch);
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
  int ctas = argc > 1 ? atoi(argv[1]) : 296, iters = argc > 2 ? atoi(argv[2]) : 2000;
  unsigned* bar;
  double* sink;
  cudaMalloc(&bar, 4);
  cudaMalloc(&sink, 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bar, 0, 4);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      void* args[] = {&mode, &iters, &bar, &sink};
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(probe), dim3(ctas), dim3(256), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s ctas %d: %.3f us per barrier (%s)\n", mode == 0 ? "cg grid.sync      " : "counter + acquire ", ctas,
             1e3 * ms / iters, cudaGetErrorString(e));
    }
  return 0;
}

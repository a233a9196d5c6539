// Dense fp64 kernels of the low-rank path (see dense.cuh).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <stdexcept>
#include <vector>

#include <cooperative_groups.h>

#include "dense.cuh"

namespace rtlr {
namespace cuda {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024); result valid in all threads.
__device__ __forceinline__ double block_sum_all(double v, double* sh) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += sh[i];  // fixed order
  __syncthreads();
  return s;
}

// ------------------------------------------------------------ GEMM A^T B
// C = sum over the split-K partials.  Few outputs with many splits (the
// CGS GEMVs): one warp per output, lanes stride the splits, fixed shuffle
// tree; many outputs: one thread per output, splits in order.  Both orders
// are fixed, so results are bitwise reproducible.
__global__ void splitk_reduce(int M, int N, int splits, const double* __restrict__ part, double* __restrict__ C,
                              long long ldc) {
  const long long total = static_cast<long long>(M) * N;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * total + e];
    const int m = static_cast<int>(e % M), n = static_cast<int>(e / M);
    C[m + n * ldc] = s;
  }
}

__global__ void splitk_reduce_warp(int M, int N, int splits, const double* __restrict__ part, double* __restrict__ C,
                                   long long ldc) {
  const long long total = static_cast<long long>(M) * N;
  const int lane = threadIdx.x & 31;
  for (long long e = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; e < total;
       e += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    double s = 0.0;
    for (int z = lane; z < splits; z += 32) s += part[z * total + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int m = static_cast<int>(e % M), n = static_cast<int>(e / M);
      C[m + n * ldc] = s;
    }
  }
}

int grid1d(long long n);

void launch_splitk_reduce(int M, int N, int splits, const double* part, double* C, long long ldc, cudaStream_t s) {
  const long long total = static_cast<long long>(M) * N;
  if (splits >= 64 && total <= 4096)
    splitk_reduce_warp<<<static_cast<unsigned>((total * 32 + 255) / 256), 256, 0, s>>>(M, N, splits, part, C, ldc);
  else
    splitk_reduce<<<grid1d(total), 256, 0, s>>>(M, N, splits, part, C, ldc);
}

int tn_splits(int M, int N, long long K) {
  const long long tiles = static_cast<long long>((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  long long s = (2 * 148 * 2 + tiles - 1) / tiles;  // ~4 CTAs per SM
  s = std::min<long long>(s, std::max<long long>(1, K / 256));
  s = std::min<long long>(s, 1024);
  return static_cast<int>(std::max<long long>(1, s));
}

// Split count of gemm_tn_dmma_nt (128-row tiles, ~4 CTAs per SM).
long long nt_splits(int M, long long K) {
  const long long tiles = (M + 127) / 128;
  long long sp = std::min<long long>((2 * 148 * 2 + tiles - 1) / tiles, std::max<long long>(1, K / 256));
  return std::max<long long>(1, std::min<long long>(sp, 1024));
}

// ------------------------------------------------------------ skinny GEMMs
// N <= 16 columns (CGS batches, candidate blocks): the 64-wide tiles above
// would waste up to 8x the flops.
constexpr int kSkinny = 16;

// C[M x N] = A^T B, A: K x M, split-K partials like gemm_tn_kernel.
__global__ void __launch_bounds__(256) gemm_tn_skinny_kernel(int M, int N, long long K, long long kchunk,
                                                             const double* __restrict__ A, long long lda,
                                                             const double* __restrict__ B, long long ldb,
                                                             double* __restrict__ out, long long ldo,
                                                             long long split_stride) {
  constexpr int SK = 32;
  __shared__ double As[SK][BM + 1];
  __shared__ double Bs[SK][kSkinny + 1];
  const int tid = threadIdx.x, tm = tid % 16, tn = tid / 16;
  const int m0 = blockIdx.x * BM;
  const long long k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long kb = k0; kb < k1; kb += SK) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {  // 32 x 64 tile of A, k fastest
      const int idx = tid + e * 256, kk = idx % SK, mm = idx / SK;
      const long long k = kb + kk;
      As[kk][mm] = (k < k1 && m0 + mm < M) ? A[k + static_cast<long long>(m0 + mm) * lda] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int idx = tid + e * 256, kk = idx % SK, nn = idx / SK;
      const long long k = kb + kk;
      Bs[kk][nn] = (k < k1 && nn < N) ? B[k + static_cast<long long>(nn) * ldb] : 0.0;
    }
    __syncthreads();
    if (tn < N) {
#pragma unroll
      for (int kk = 0; kk < SK; ++kk) {
        const double b = Bs[kk][tn];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += As[kk][tm + 16 * i] * b;
      }
    }
    __syncthreads();
  }
  if (tn < N) {
    double* o = out + blockIdx.y * split_stride;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + tm + 16 * i;
      if (m < M) o[m + static_cast<long long>(tn) * ldo] = acc[i];
    }
  }
}

// C[M x N] (-)= A B, A: M x K (M large), B: K x N; one row per thread.
__global__ void __launch_bounds__(256) gemm_nn_skinny_kernel(long long M, int N, int K, const double* __restrict__ A,
                                                             long long lda, const double* __restrict__ B, long long ldb,
                                                             double* __restrict__ C, long long ldc, bool subtract) {
  constexpr int KC = 128;
  __shared__ double Bs[KC][kSkinny];
  const long long m = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  double acc[kSkinny];
#pragma unroll
  for (int j = 0; j < kSkinny; ++j) acc[j] = 0.0;
  for (int kb = 0; kb < K; kb += KC) {
    const int kc = min(KC, K - kb);
    for (int e = threadIdx.x; e < KC * kSkinny; e += blockDim.x) {
      const int kk = e % KC, nn = e / KC;
      Bs[kk][nn] = (kk < kc && nn < N) ? B[kb + kk + static_cast<long long>(nn) * ldb] : 0.0;
    }
    __syncthreads();
    if (m < M)
      for (int kk = 0; kk < kc; ++kk) {
        const double a = A[m + static_cast<long long>(kb + kk) * lda];
#pragma unroll
        for (int j = 0; j < kSkinny; ++j) acc[j] += a * Bs[kk][j];
      }
    __syncthreads();
  }
  if (m < M)
    for (int j = 0; j < N; ++j) {
      double* c = C + m + static_cast<long long>(j) * ldc;
      *c = subtract ? *c - acc[j] : acc[j];
    }
}

// ---- tall-skinny GEMMs, second generation: 16-byte loads, register tiles.
// C[M x N] = A^T B split-K partials: warp w of a CTA owns MW columns of A;
// lanes walk row pairs (16 B per load, 512 B per warp instruction), keep
// MW x NB accumulators and reduce over lanes at the end.  Needs A, B 16-byte
// aligned and even leading dimensions (the launcher checks; K offsets even).
__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

template <int NB, int MW>
__global__ void __launch_bounds__(256) gemm_tn_skinny2(int M, int N, long long K, long long kchunk,
                                                       const double* __restrict__ A, long long lda,
                                                       const double* __restrict__ B, long long ldb,
                                                       double* __restrict__ out, long long ldo, long long split_stride) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int m0 = (blockIdx.x * 8 + w) * MW;
  const long long k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  double acc[MW][NB];
#pragma unroll
  for (int i = 0; i < MW; ++i)
#pragma unroll
    for (int n = 0; n < NB; ++n) acc[i][n] = 0.0;
  if (m0 < M) {
    for (long long k = k0 + 2 * lane; k < k1; k += 64) {
      const bool pair = k + 1 < k1;
      double b0[NB], b1[NB];
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        b0[n] = b1[n] = 0.0;
        if (n < N) {
          if (pair) {
            const double2 v = ldg2(B + k + n * ldb);
            b0[n] = v.x;
            b1[n] = v.y;
          } else {
            b0[n] = B[k + n * ldb];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < MW; ++i) {
        if (m0 + i < M) {
          const double* a = A + k + static_cast<long long>(m0 + i) * lda;
          double a0, a1 = 0.0;
          if (pair) {
            const double2 v = ldg2(a);
            a0 = v.x;
            a1 = v.y;
          } else {
            a0 = a[0];
          }
#pragma unroll
          for (int n = 0; n < NB; ++n) acc[i][n] = fma(a1, b1[n], fma(a0, b0[n], acc[i][n]));
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < MW; ++i)
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      double v = acc[i][n];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[i][n] = v;
    }
  if (lane == 0) {
    double* o = out + blockIdx.y * split_stride;
#pragma unroll
    for (int i = 0; i < MW; ++i)
#pragma unroll
      for (int n = 0; n < NB; ++n)
        if (m0 + i < M && n < N) o[(m0 + i) + static_cast<long long>(n) * ldo] = acc[i][n];
  }
}

// C[M x N] (-)= A B, A: M x K (M large), B: K x N: two rows per thread
// (one 16-byte load per k), B staged in shared memory in chunks of k.
template <int NB>
__global__ void __launch_bounds__(256) gemm_nn_skinny2(long long M, int N, int K, const double* __restrict__ A,
                                                       long long lda, const double* __restrict__ B, long long ldb,
                                                       double* __restrict__ C, long long ldc, bool subtract) {
  constexpr int KC = 64;
  __shared__ double Bs[KC][NB];
  const long long m = 2 * (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x);
  double acc0[NB], acc1[NB];
#pragma unroll
  for (int n = 0; n < NB; ++n) acc0[n] = acc1[n] = 0.0;
  const bool two = m + 1 < M;
  for (int kb = 0; kb < K; kb += KC) {
    const int kc = min(KC, K - kb);
    __syncthreads();
    for (int e = threadIdx.x; e < KC * NB; e += blockDim.x) {
      const int kk = e % KC, n = e / KC;
      Bs[kk][n] = (kk < kc && n < N) ? B[kb + kk + static_cast<long long>(n) * ldb] : 0.0;
    }
    __syncthreads();
    if (m < M) {
      const double* a = A + m + static_cast<long long>(kb) * lda;
#pragma unroll 4
      for (int kk = 0; kk < kc; ++kk, a += lda) {
        double a0, a1 = 0.0;
        if (two) {
          const double2 v = ldg2(a);
          a0 = v.x;
          a1 = v.y;
        } else {
          a0 = a[0];
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const double b = Bs[kk][n];
          acc0[n] = fma(a0, b, acc0[n]);
          acc1[n] = fma(a1, b, acc1[n]);
        }
      }
    }
  }
  if (m < M)
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      if (n >= N) break;
      double* c = C + m + static_cast<long long>(n) * ldc;
      c[0] = subtract ? c[0] - acc0[n] : acc0[n];
      if (two) c[1] = subtract ? c[1] - acc1[n] : acc1[n];
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---- fp64 tensor-core (DMMA) tiles for the wide contractions: K6 X^T [W]
// (projections), the QR trailing updates and K8 X C.  mma.sync m8n8k4 f64:
// A fragment (8 x 4, row): lane holds A[lane/4][lane%4]; B (4 x 8, col):
// B[lane%4][lane/4]; C (8 x 8): C[lane/4][2(lane%4) + {0,1}].  CTA tile
// 64 x 64, k step 16 staged in shared memory as [k][m] / [k][n]; 8 warps in
// a 2 x 4 grid, 32 x 16 per warp (4 x 2 mma tiles).
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int kMmaPad = 8;  // row stride 72 doubles: the 4 k-rows x 8 lanes of a fragment hit distinct banks

// TRANS_A: op(A)[m][k] = A[k + m lda] (A^T B, split-K partials into out);
// else op(A)[m][k] = A[m + k lda] (A B; out = C, or C -= when subtract).
// A^T B split-K on DMMA with a two-stage cp.async pipeline: both operands
// are K-contiguous, so a 64 x 32 tile of each is 64 runs of 256 B staged as
// [m][k] / [n][k] (row stride 36 doubles: fragment loads hit distinct banks)
// while the tensor cores work on the other stage.  Needs A, B 16-byte
// aligned with even leading dimensions and K even (the launcher checks).
constexpr int kTnBk = 32, kTnLd = kTnBk + 4;

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int n = valid ? 16 : 0;  // zero-fill outside the matrix
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// A^T B for N <= 8 (the CGS block products): one 8 x 8 DMMA tile per warp,
// 64 columns of A per CTA, a four-stage cp.async pipeline of 64 x 32 A tiles
// (16 KB) and 8 x 32 B tiles, so enough bytes are in flight to run at HBM
// bandwidth.  Same alignment contract and split-K partials as the wide kernel.
constexpr int kSkStages = 4;
__global__ void __launch_bounds__(256) gemm_tn_skinny_pipe(int M, int N, long long K, long long kchunk,
                                                           const double* __restrict__ A, long long lda,
                                                           const double* __restrict__ B, long long ldb,
                                                           double* __restrict__ out, long long ldo,
                                                           long long split_stride) {
  extern __shared__ double sm[];
  double* As = sm;                               // [stages][64][kTnLd]
  double* Bs = sm + kSkStages * 64 * kTnLd;      // [stages][8][kTnLd]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * 64;
  const long long k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  const int fr = lane >> 2, fc = lane & 3;
  auto stage = [&](int buf, long long kb) {
    if (kb < k1) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // A: 64 rows x 16 pieces
        const int idx = tid + e * 256, row = idx >> 4, kq = (idx & 15) * 2;
        const long long k = kb + kq;
        const int m = m0 + row;
        const bool v = k < k1 && m < M;
        cp_async16(As + (buf * 64 + row) * kTnLd + kq, A + (v ? k + static_cast<long long>(m) * lda : 0), v);
      }
      if (tid < 128) {  // B: 8 rows x 16 pieces
        const int row = tid >> 4, kq = (tid & 15) * 2;
        const long long k = kb + kq;
        const bool v = k < k1 && row < N;
        cp_async16(Bs + (buf * 8 + row) * kTnLd + kq, B + (v ? k + static_cast<long long>(row) * ldb : 0), v);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (possibly empty) group keeps the count uniform
  };
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int p = 0; p < kSkStages - 1; ++p) stage(p, k0 + p * kTnBk);
  int buf = 0;
  for (long long kb = k0; kb < k1; kb += kTnBk) {
    stage((buf + kSkStages - 1) % kSkStages, kb + (kSkStages - 1) * kTnBk);
    asm volatile("cp.async.wait_group %0;" ::"n"(kSkStages - 1) : "memory");
    __syncthreads();
    const double* as = As + (buf * 64 + warp * 8 + fr) * kTnLd;
    const double* bs = Bs + (buf * 8 + fr) * kTnLd;
#pragma unroll
    for (int ks = 0; ks < kTnBk; ks += 4) dmma884(c0, c1, as[ks + fc], bs[ks + fc]);
    __syncthreads();
    buf = (buf + 1) % kSkStages;
  }
  const int m = m0 + warp * 8 + fr, n = 2 * fc;
  double* o = out + blockIdx.y * split_stride;
  if (m < M) {
    if (n < N) o[m + static_cast<long long>(n) * ldo] = c0;
    if (n + 1 < N) o[m + static_cast<long long>(n + 1) * ldo] = c1;
  }
}

__global__ void __launch_bounds__(256) gemm_tn_dmma_pipe(int M, int N, long long K, long long kchunk,
                                                         const double* __restrict__ A, long long lda,
                                                         const double* __restrict__ B, long long ldb,
                                                         double* __restrict__ out, long long ldo,
                                                         long long split_stride) {
  extern __shared__ double sm[];
  double* As = sm;                           // [2][BM][kTnLd]
  double* Bs = sm + 2 * BM * kTnLd;          // [2][BN][kTnLd]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const long long k0 = blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
  const int fr = lane >> 2, fc = lane & 3;
  const int nt = min(2, max(0, (N - (n0 + wn) + 7) / 8));  // this warp's live 8-column tiles
  auto stage = [&](int buf, long long kb) {
    // 64 rows x 32 k per operand = 64 x 16 chunks of 16 B; 4 + 4 per thread
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256, row = idx >> 4, kq = (idx & 15) * 2;
      const long long k = kb + kq;
      const int m = m0 + row, n = n0 + row;
      const bool ka = k < k1;
      cp_async16(As + (buf * BM + row) * kTnLd + kq, A + (ka && m < M ? k + static_cast<long long>(m) * lda : 0),
                 ka && m < M);
      cp_async16(Bs + (buf * BN + row) * kTnLd + kq, B + (ka && n < N ? k + static_cast<long long>(n) * ldb : 0),
                 ka && n < N);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int buf = 0;
  if (k0 < k1) stage(0, k0);
  for (long long kb = k0; kb < k1; kb += kTnBk, buf ^= 1) {
    if (kb + kTnBk < k1) {
      stage(buf ^ 1, kb + kTnBk);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* as = As + buf * BM * kTnLd;
    const double* bs = Bs + buf * BN * kTnLd;
    if (nt > 0) {  // warps whose 16 columns all lie past N (skinny products) skip the tensor work
#pragma unroll
      for (int ks = 0; ks < kTnBk; ks += 4) {
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = as[(wm + 8 * i + fr) * kTnLd + ks + fc];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = bs[(wn + 8 * j + fr) * kTnLd + ks + fc];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dmma884(acc[i][0][0], acc[i][0][1], a[i], b[0]);
          if (nt > 1) dmma884(acc[i][1][0], acc[i][1][1], a[i], b[1]);
        }
      }
    }
    __syncthreads();  // the stage is refilled next iteration
  }
  double* o = out + blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + fr;
        const int n = n0 + wn + 8 * j + 2 * fc + h;
        if (m < M && n < N) o[m + static_cast<long long>(n) * ldo] = acc[i][j][h];
      }
}

// A^T B for 4 <= N <= 48 (the border-extension products X^T [5p stencil
// images]: N = 40 at p = 8, 20 at p = 4): 128 columns of A per CTA, every
// warp owns 16 of them against all ceil(N/8) column tiles of B, so no warp
// idles on padding columns and B is re-read once per 128 (not 64) columns
// of A.  Two-stage cp.async pipeline of 128 x 32 A and up to 48 x 32 B tiles (two CTAs
// per SM; three stages with one CTA were 17% slower).  Also the CGS projections
// with 4-8 columns (one padded column tile).
// Same alignment contract and split-K partials as gemm_tn_dmma_pipe.
constexpr int kNtBm = 128, kNtStages = 2, kNtMaxN = 48;
template <int NT>
__global__ void __launch_bounds__(256) gemm_tn_dmma_nt(int M, int N, long long K, long long kchunk,
                                                       const double* __restrict__ A, long long lda,
                                                       const double* __restrict__ B, long long ldb,
                                                       double* __restrict__ out, long long ldo,
                                                       long long split_stride) {
  extern __shared__ double sm[];
  double* As = sm;                                  // [stages][128][kTnLd]
  double* Bs = sm + kNtStages * kNtBm * kTnLd;      // [stages][8 NT][kTnLd]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * kNtBm, wm = warp * 16;
  const long long k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  const int fr = lane >> 2, fc = lane & 3;
  auto stage = [&](int buf, long long kb) {
    if (kb < k1) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {  // A: 128 rows x 16 pieces of 16 B
        const int idx = tid + e * 256, row = idx >> 4, kq = (idx & 15) * 2;
        const long long k = kb + kq;
        const int m = m0 + row;
        const bool v = k < k1 && m < M;
        cp_async16(As + (buf * kNtBm + row) * kTnLd + kq, A + (v ? k + static_cast<long long>(m) * lda : 0), v);
      }
      for (int idx = tid; idx < 8 * NT * 16; idx += 256) {  // B: 8 NT rows x 16 pieces
        const int row = idx >> 4, kq = (idx & 15) * 2;
        const long long k = kb + kq;
        const bool v = k < k1 && row < N;
        cp_async16(Bs + (buf * 8 * NT + row) * kTnLd + kq, B + (v ? k + static_cast<long long>(row) * ldb : 0), v);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int p = 0; p < kNtStages - 1; ++p) stage(p, k0 + p * kTnBk);
  int buf = 0;
  for (long long kb = k0; kb < k1; kb += kTnBk) {
    stage((buf + kNtStages - 1) % kNtStages, kb + (kNtStages - 1) * kTnBk);
    asm volatile("cp.async.wait_group %0;" ::"n"(kNtStages - 1) : "memory");
    __syncthreads();
    const double* as = As + (buf * kNtBm + wm + fr) * kTnLd;
    const double* bs = Bs + (buf * 8 * NT + fr) * kTnLd;
#pragma unroll
    for (int ks = 0; ks < kTnBk; ks += 4) {
      const double a0 = as[ks + fc], a1 = as[8 * kTnLd + ks + fc];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const double b = bs[8 * j * kTnLd + ks + fc];
        dmma884(acc[0][j][0], acc[0][j][1], a0, b);
        dmma884(acc[1][j][0], acc[1][j][1], a1, b);
      }
    }
    __syncthreads();
    buf = (buf + 1) % kNtStages;
  }
  double* o = out + blockIdx.y * split_stride;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + fr, n = 8 * j + 2 * fc + h;
        if (m < M && n < N) o[m + static_cast<long long>(n) * ldo] = acc[i][j][h];
      }
}

// C (-)= A B on DMMA with the same two-stage cp.async pipeline: A (M x K,
// M-contiguous, M huge) is staged [k][m] in 16-byte pieces, B (K x N, any
// ld) [n][k] in 8-byte pieces.  Needs A 16-byte aligned, lda and M even.
constexpr int kNnLdA = BM + 8;
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// C (-)= A B for N > 8 with 128-row tiles: every warp owns 16 rows against
// all NT column tiles of its CTA's column group (8 NT columns; column groups
// of the same rows are adjacent in launch order, so A is re-read from L2),
// two-stage cp.async pipeline.  A staged [k][m] with row stride 132
// doubles (the fragment loads' half-warps hit distinct banks).  Same
// contract as gemm_nn_dmma_pipe.
constexpr int kNnNtLdA = kNtBm + 4;
template <int NT>
__global__ void __launch_bounds__(256) gemm_nn_dmma_nt(long long M, int N, int K, const double* __restrict__ A,
                                                       long long lda, const double* __restrict__ B, long long ldb,
                                                       double* __restrict__ C, long long ldc, bool subtract) {
  extern __shared__ double sm[];
  double* As = sm;                                    // [stages][32][kNnNtLdA]
  double* Bs = sm + kNtStages * kTnBk * kNnNtLdA;     // [stages][8 NT][kTnLd]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long m0 = static_cast<long long>(blockIdx.y) * kNtBm;
  const int n0 = blockIdx.x * 8 * NT, wm = warp * 16;
  const int fr = lane >> 2, fc = lane & 3;
  auto stage = [&](int buf, int kb) {
    if (kb < K) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {  // A: 32 k x 64 pairs of m
        const int idx = tid + e * 256, kk = idx >> 6, mq = (idx & 63) * 2;
        const int k = kb + kk;
        const long long m = m0 + mq;
        const bool v = k < K && m < M;
        cp_async16(As + (buf * kTnBk + kk) * kNnNtLdA + mq, A + (v ? m + static_cast<long long>(k) * lda : 0), v);
      }
      for (int idx = tid; idx < 8 * NT * kTnBk; idx += 256) {  // B: 8 NT n x 32 k, one double each
        const int row = idx >> 5, kk = idx & 31;
        const int k = kb + kk, n = n0 + row;
        const bool v = k < K && n < N;
        cp_async8(Bs + (buf * 8 * NT + row) * kTnLd + kk, B + (v ? k + static_cast<long long>(n) * ldb : 0), v);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int p = 0; p < kNtStages - 1; ++p) stage(p, p * kTnBk);
  int buf = 0;
  for (int kb = 0; kb < K; kb += kTnBk) {
    stage((buf + kNtStages - 1) % kNtStages, kb + (kNtStages - 1) * kTnBk);
    asm volatile("cp.async.wait_group %0;" ::"n"(kNtStages - 1) : "memory");
    __syncthreads();
    const double* as = As + buf * kTnBk * kNnNtLdA + wm + fr;
    const double* bs = Bs + (buf * 8 * NT + fr) * kTnLd;
#pragma unroll
    for (int ks = 0; ks < kTnBk; ks += 4) {
      const double a0 = as[(ks + fc) * kNnNtLdA], a1 = as[(ks + fc) * kNnNtLdA + 8];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const double b = bs[8 * j * kTnLd + ks + fc];
        dmma884(acc[0][j][0], acc[0][j][1], a0, b);
        dmma884(acc[1][j][0], acc[1][j][1], a1, b);
      }
    }
    __syncthreads();
    buf = (buf + 1) % kNtStages;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long m = m0 + wm + 8 * i + fr;
        const int n = n0 + 8 * j + 2 * fc + h;
        if (m < M && n < N) {
          double* c = C + m + static_cast<long long>(n) * ldc;
          *c = subtract ? *c - acc[i][j][h] : acc[i][j][h];
        }
      }
}

__global__ void __launch_bounds__(256) gemm_nn_dmma_pipe(long long M, int N, int K, const double* __restrict__ A,
                                                         long long lda, const double* __restrict__ B, long long ldb,
                                                         double* __restrict__ C, long long ldc, bool subtract) {
  extern __shared__ double sm[];
  double* As = sm;                          // [2][kTnBk][kNnLdA]
  double* Bs = sm + 2 * kTnBk * kNnLdA;     // [2][BN][kTnLd]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const long long m0 = static_cast<long long>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int fr = lane >> 2, fc = lane & 3;
  const int nt = min(2, max(0, (N - (n0 + wn) + 7) / 8));
  auto stage = [&](int buf, int kb) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // A: 32 k x 32 pairs of m
      const int idx = tid + e * 256, kk = idx >> 5, mq = (idx & 31) * 2;
      const int k = kb + kk;
      const long long m = m0 + mq;
      const bool v = k < K && m < M;
      cp_async16(As + (buf * kTnBk + kk) * kNnLdA + mq, A + (v ? m + static_cast<long long>(k) * lda : 0), v);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {  // B: 64 n x 32 k, one double each
      const int idx = tid + e * 256, row = idx >> 5, kk = idx & 31;
      const int k = kb + kk, n = n0 + row;
      const bool v = k < K && n < N;
      cp_async8(Bs + (buf * BN + row) * kTnLd + kk, B + (v ? k + static_cast<long long>(n) * ldb : 0), v);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int buf = 0;
  stage(0, 0);
  for (int kb = 0; kb < K; kb += kTnBk, buf ^= 1) {
    if (kb + kTnBk < K) {
      stage(buf ^ 1, kb + kTnBk);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* as = As + buf * kTnBk * kNnLdA;
    const double* bs = Bs + buf * BN * kTnLd;
    if (nt > 0) {
#pragma unroll
      for (int ks = 0; ks < kTnBk; ks += 4) {
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = as[(ks + fc) * kNnLdA + wm + 8 * i + fr];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = bs[(wn + 8 * j + fr) * kTnLd + ks + fc];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dmma884(acc[i][0][0], acc[i][0][1], a[i], b[0]);
          if (nt > 1) dmma884(acc[i][1][0], acc[i][1][1], a[i], b[1]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long m = m0 + wm + 8 * i + fr;
        const int n = n0 + wn + 8 * j + 2 * fc + h;
        if (m < M && n < N) {
          double* c = C + m + static_cast<long long>(n) * ldc;
          *c = subtract ? *c - acc[i][j][h] : acc[i][j][h];
        }
      }
}

template <bool TRANS_A>
__global__ void __launch_bounds__(256) gemm_dmma_kernel(long long M, int N, long long K, long long kchunk,
                                                        const double* __restrict__ A, long long lda,
                                                        const double* __restrict__ B, long long ldb,
                                                        double* __restrict__ out, long long ldo, long long split_stride,
                                                        bool subtract) {
  __shared__ double As[BK][BM + kMmaPad];
  __shared__ double Bs[BK][BN + kMmaPad];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;  // warp tile origin in the CTA tile
  const long long m0 = static_cast<long long>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const long long k0 = TRANS_A ? blockIdx.z * kchunk : 0;
  const long long k1 = TRANS_A ? min(K, k0 + kchunk) : K;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fr = lane >> 2, fc = lane & 3;
  for (long long kb = k0; kb < k1; kb += BK) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      if (TRANS_A) {  // A[k + m lda], k fastest
        const int kk = idx % BK, mm = idx / BK;
        const long long k = kb + kk, m = m0 + mm;
        As[kk][mm] = (k < k1 && m < M) ? A[k + m * lda] : 0.0;
      } else {  // A[m + k lda], m fastest
        const int mm = idx % BM, kk = idx / BM;
        const long long k = kb + kk, m = m0 + mm;
        As[kk][mm] = (k < k1 && m < M) ? A[m + k * lda] : 0.0;
      }
      const int kk = idx % BK, nn = idx / BK;
      const long long k = kb + kk;
      const int n = n0 + nn;
      Bs[kk][nn] = (k < k1 && n < N) ? B[k + static_cast<long long>(n) * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[ks + fc][wm + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs[ks + fc][wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  double* o = out + (TRANS_A ? blockIdx.z * split_stride : 0);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long m = m0 + wm + 8 * i + fr;
        const int n = n0 + wn + 8 * j + 2 * fc + h;
        if (m < M && n < N) {
          double* c = o + m + static_cast<long long>(n) * ldo;
          if (TRANS_A || !subtract)
            *c = acc[i][j][h];
          else
            *c -= acc[i][j][h];
        }
      }
}

// ------------------------------------------------------------ vectors
__global__ void gemv_n_kernel(long long n, int k, const double* __restrict__ A, long long lda,
                              const double* __restrict__ x, double alpha, double* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += A[i + j * lda] * x[j];
    y[i] += alpha * s;
  }
}

constexpr int kDotParts = kDotWork;

__global__ void dot_partials(long long n, const double* __restrict__ a, const double* __restrict__ b,
                             double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    s += a[i] * b[i];
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// dot_partials against column *col of B (a column chosen on the device);
// *col < 0: zero.  Same partition and order as dot_partials.
__global__ void dot_partials_ind(long long n, const double* __restrict__ a, const double* __restrict__ B, long long ldb,
                                 const int* __restrict__ col, double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = *col;
  if (c < 0) {
    if (threadIdx.x == 0) part[blockIdx.x] = 0.0;
    return;
  }
  const double* b = B + static_cast<long long>(c) * ldb;
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    s += a[i] * b[i];
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void dot_finish(int parts, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < parts; i += blockDim.x) s += part[i];
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void scale_copy_kernel(long long n, const double* __restrict__ x, const double* __restrict__ h,
                                  double* __restrict__ y) {
  const double d = *h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void axpy_kernel(long long n, const double* __restrict__ alpha, double sign, const double* __restrict__ x,
                            double* __restrict__ y) {
  const double a = sign * *alpha;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] += a * x[i];
}

int grid1d(long long n) {
  long long g = (n + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(g, 148 * 16)));
}

// ------------------------------------------------------------ stencils
__device__ __forceinline__ double row_mv(const double* B, int i, const double* v) {
  return B[i] * v[0] + B[4 + i] * v[1] + B[8 + i] * v[2] + B[12 + i] * v[3];
}
__device__ __forceinline__ double col_mv(const double* B, int i, const double* v) {  // (B^T v)_i
  return B[4 * i] * v[0] + B[4 * i + 1] * v[1] + B[4 * i + 2] * v[2] + B[4 * i + 3] * v[3];
}

// One thread per (cell, column): the cell's four DOFs of all five products,
// its own and neighbour coefficients as 16-byte loads, 2-D grid (cells x
// columns, no 64-bit index division).  Per output the same row_mv / col_mv
// arithmetic as before.
__global__ void stream_products_kernel(const StencilArgs A, int p, const double* __restrict__ P, long long ldp,
                                       double* __restrict__ W, long long ldw, int c0, int c1) {
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int j = blockIdx.y;
  const int a = c % A.nx, b = c / A.nx;
  const double* pc = P + j * ldp + 4LL * c;
  const long long up = 4LL * A.nx;
  auto ld4v = [](const double* q, double v[4]) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(q)), y = __ldg(reinterpret_cast<const double2*>(q) + 1);
    v[0] = x.x, v[1] = x.y, v[2] = y.x, v[3] = y.y;
  };
  double v[4], w[4] = {0, 0, 0, 0}, e[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0}, n[4] = {0, 0, 0, 0}, st[16];
  ld4v(pc, v);
  if (a > 0) ld4v(pc - 4, w);
  if (a + 1 < A.nx) ld4v(pc + 4, e);
  if (b > 0) ld4v(pc - up, s);
  if (b + 1 < A.ny) ld4v(pc + up, n);
  const double2* sb = reinterpret_cast<const double2*>(A.sigma_t + 16LL * c);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 t = __ldg(sb + k);
    st[2 * k] = t.x;
    st[2 * k + 1] = t.y;
  }
  double out[5][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double dxm = row_mv(A.sc.ax_minus, i, v);
    if (a > 0) dxm += row_mv(A.sc.bx_minus, i, w);
    double dxmt = col_mv(A.sc.ax_minus, i, v);
    if (a + 1 < A.nx) dxmt += col_mv(A.sc.bx_minus, i, e);
    double dym = row_mv(A.sc.ay_minus, i, v);
    if (b > 0) dym += row_mv(A.sc.by_minus, i, s);
    double dymt = col_mv(A.sc.ay_minus, i, v);
    if (b + 1 < A.ny) dymt += col_mv(A.sc.by_minus, i, n);
    out[0][i] = dxm;
    out[1][i] = dxmt;
    out[2][i] = dym;
    out[3][i] = dymt;
    out[4][i] = row_mv(st, i, v);
  }
  const long long blk = p * ldw;
  double* o = W + 4LL * c + j * ldw;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double2* q = reinterpret_cast<double2*>(o + k * blk);
    q[0] = make_double2(out[k][0], out[k][1]);
    q[1] = make_double2(out[k][2], out[k][3]);
  }
}

// ------------------------------------------------------------ Galerkin LU
// One CTA per angle.  A (r x r, column-major, leading dimension r) lives in
// shared memory (r <= kSmemLuMax) or in the global workspace.
__device__ void lu_solve_block(double* Am, double* b, int r, double* shv, int* shi) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < r; ++k) {
    // pivot: first maximum of |A[i,k]|, i >= k
    double best = -1.0;
    int bi = r;
    for (int i = k + tid; i < r; i += nt) {
      const double v = fabs(Am[i + k * r]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    // warp then block argmax, ties -> smaller index
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) {
      shv[warp] = best;
      shi[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = shv[0];
      int bix = shi[0];
      for (int w = 1; w < (nt >> 5); ++w)
        if (shv[w] > bv || (shv[w] == bv && shi[w] < bix)) {
          bv = shv[w];
          bix = shi[w];
        }
      shi[32] = bix;
      shv[32] = bv;
    }
    __syncthreads();
    const int p = shi[32];
    const bool nonzero = shv[32] > 0.0;
    if (nonzero && p != k) {
      for (int j = tid; j < r; j += nt) {
        const double t = Am[k + j * r];
        Am[k + j * r] = Am[p + j * r];
        Am[p + j * r] = t;
      }
      if (tid == 0) {
        const double t = b[k];
        b[k] = b[p];
        b[p] = t;
      }
    }
    __syncthreads();
    if (nonzero) {
      const double d = Am[k + k * r];
      for (int i = k + 1 + tid; i < r; i += nt) Am[i + k * r] /= d;
    }
    __syncthreads();
    // trailing update and forward substitution on b
    const int rr = r - k - 1;
    for (int e = tid; e < rr * rr; e += nt) {
      const int i = k + 1 + e % rr, j = k + 1 + e / rr;
      Am[i + j * r] -= Am[i + k * r] * Am[k + j * r];
    }
    for (int i = k + 1 + tid; i < r; i += nt) b[i] -= b[k] * Am[i + k * r];
    __syncthreads();
  }
  // back substitution (column oriented)
  for (int i = r - 1; i >= 0; --i) {
    if (tid == 0) b[i] = b[i] / Am[i + i * r];
    __syncthreads();
    const double bi = b[i];
    for (int j = tid; j < i; j += nt) b[j] -= bi * Am[j + i * r];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) galerkin_kernel(int r, const int* __restrict__ angles,
                                                       const double* __restrict__ dirs, const double* __restrict__ proj,
                                                       long long ldp, long long pstride, const double* __restrict__ prhs,
                                                       const double* __restrict__ extra, double* __restrict__ sol,
                                                       long long ldsol, int* __restrict__ flags, double* __restrict__ work,
                                                       bool in_smem) {
  extern __shared__ double sm[];
  __shared__ double shv[33];
  __shared__ int shi[33];
  __shared__ double bvec_small[kSmemLuMax];
  const int jb = blockIdx.x;
  const int ang = angles[jb];
  const double omx = dirs[3 * ang], omy = dirs[3 * ang + 1];
  const double* px = proj + (omx >= 0.0 ? 0 : 1) * pstride;
  const double* py = proj + (omy >= 0.0 ? 2 : 3) * pstride;
  const double* pt = proj + 4 * pstride;
  double* Am = in_smem ? sm : work + static_cast<size_t>(jb) * r * r;
  double* b = in_smem ? bvec_small : sol + jb * ldsol;
  // reduced_streaming (low_rank.cpp:176-183): omx*Px + omy*Py + Pt
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int i = e % r, j = e / r;
    Am[i + j * r] = omx * px[i + j * ldp] + omy * py[i + j * ldp] + pt[i + j * ldp];
  }
  for (int i = threadIdx.x; i < r; i += blockDim.x) b[i] = prhs[i] + (extra ? extra[i + jb * ldsol] : 0.0);
  __syncthreads();
  lu_solve_block(Am, b, r, shv, shi);
  int bad = 0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    if (!isfinite(b[i])) bad = 1;
    if (in_smem) sol[i + jb * ldsol] = b[i];
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) flags[jb] = bad;
}

// ------------------------------------------------------------ Householder QR
// column tail norms: out[0] = sum_{i>k} x_i^2 over column k (rows k+1..m-1)
__global__ void hh_tail(long long m, int k, const double* __restrict__ a, long long lda, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = k + 1 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double v = a[i + k * lda];
    s += v * v;
  }
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// beta / tau (Eigen makeHouseholder) from the partials; store in scal[0..2]
__global__ void hh_make(int parts, int k, double* a, long long lda, const double* part, double* tau, double* scal) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < parts; i += blockDim.x) s += part[i];
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) {
    const double c0 = a[k + k * lda];
    double beta, t, denom;
    if (s <= 2.2250738585072014e-308) {
      t = 0.0;
      beta = c0;
      denom = 0.0;  // tail zeroed
    } else {
      beta = sqrt(c0 * c0 + s);
      if (c0 >= 0.0) beta = -beta;
      denom = c0 - beta;
      t = (beta - c0) / beta;
    }
    tau[k] = t;
    scal[0] = denom;
    scal[1] = beta;
  }
}

__global__ void hh_scale_tail(long long m, int k, double* a, long long lda, const double* scal) {
  const double denom = scal[0];
  for (long long i = k + 1 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    a[i + k * lda] = denom == 0.0 ? 0.0 : a[i + k * lda] / denom;
}

// w_j = a[k,j] + sum_{i>k} v_i a[i,j] for j in [j0, j1): one CTA per column,
// then a[:,j] -= tau w_j v   (v_0 = 1, v_i = a[i,k] for i > k)
__global__ void hh_apply(long long m, int k, const double* __restrict__ v, long long ldv, const double* tau,
                         double* a, long long lda, int j0) {
  __shared__ double sh[32];
  const int j = j0 + blockIdx.x;
  double* col = a + j * lda;
  double s = 0.0;
  for (long long i = k + 1 + threadIdx.x; i < m; i += blockDim.x) s += v[i + k * ldv] * col[i];
  s = block_sum_all(s, sh);
  const double w = tau[k] * (col[k] + s);
  if (threadIdx.x == 0) col[k] -= w;
  for (long long i = k + 1 + threadIdx.x; i < m; i += blockDim.x) col[i] -= w * v[i + k * ldv];
}

// Panel-column reflector application for tall columns, spread over
// (column, row chunk) CTAs: partial dots v^T a_j per chunk, then every CTA
// of column j sums the chunk partials in a fixed order (deterministic),
// w_j = tau (a[k,j] + sum), and updates its rows.
constexpr int kHhChunks = 32;
__global__ void hh_dot_chunks(long long m, int k, const double* __restrict__ v, long long ldv,
                              const double* __restrict__ a, long long lda, int j0, double* __restrict__ part) {
  __shared__ double sh[32];
  const int j = j0 + blockIdx.x, c = blockIdx.y;
  const long long rows = m - (k + 1), per = (rows + kHhChunks - 1) / kHhChunks;
  const long long r0 = k + 1 + c * per, r1 = min(m, r0 + per);
  const double* col = a + j * lda;
  double s = 0.0;
  for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) s += v[i + k * ldv] * col[i];
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x * kHhChunks + c] = s;
}
__global__ void hh_update_chunks(long long m, int k, const double* __restrict__ v, long long ldv, const double* tau,
                                 double* a, long long lda, int j0, const double* __restrict__ part) {
  const int j = j0 + blockIdx.x, c = blockIdx.y;
  double* col = a + j * lda;
  double s = 0.0;
  for (int z = 0; z < kHhChunks; ++z) s += part[blockIdx.x * kHhChunks + z];
  const double w = tau[k] * (col[k] + s);
  const long long rows = m - (k + 1), per = (rows + kHhChunks - 1) / kHhChunks;
  const long long r0 = k + 1 + c * per, r1 = min(m, r0 + per);
  for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) col[i] -= w * v[i + k * ldv];
}
// row k of the updated columns, after every chunk CTA has read a[k, j]
__global__ void hh_update_diag(int k, const double* tau, double* a, long long lda, int j0, int ncols,
                               const double* __restrict__ part) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ncols) return;
  double* col = a + (j0 + t) * lda;
  double s = 0.0;
  for (int z = 0; z < kHhChunks; ++z) s += part[t * kHhChunks + z];
  col[k] -= tau[k] * (col[k] + s);
}

__global__ void set_beta(int k, double* a, long long lda, const double* scal) {
  if (threadIdx.x == 0 && blockIdx.x == 0) a[k + k * lda] = scal[1];
}

__global__ void eye_cols(long long m, int n, double* q, long long ldq) {
  const long long total = m * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e % m, j = e / m;
    q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
  }
}

// Explicit reflector block V (rows k0.., jb columns): unit diagonal, zeros
// above, the stored v_i below (the factored panel keeps beta on its diagonal).
__global__ void hh_panel_v(long long m, int k0, int jb, const double* __restrict__ a, long long lda,
                           double* __restrict__ v, long long ldv) {
  const long long rows = m - k0, total = rows * jb;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e % rows;
    const int j = static_cast<int>(e / rows);
    v[i + j * ldv] = i < j ? 0.0 : (i == j ? 1.0 : a[k0 + i + (k0 + j) * lda]);
  }
}

// Forward column-wise block-reflector factor (H_0 ... H_{jb-1} = I - V T V^T):
// T[i][i] = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] (V^T V)[0:i, i].  One block.
__global__ void hh_form_t(int jb, const double* __restrict__ gram, const double* __restrict__ tau,
                          double* __restrict__ t) {
  __shared__ double T[32][33];
  const int j = threadIdx.x;
  if (j < jb)
    for (int i = 0; i < jb; ++i) T[j][i] = 0.0;
  __syncthreads();
  for (int i = 0; i < jb; ++i) {
    if (j < i) {
      double s = 0.0;
      for (int l = j; l < i; ++l) s += T[j][l] * gram[l + i * jb];
      T[j][i] = -tau[i] * s;
    } else if (j == i) {
      T[i][i] = tau[i];
    }
    __syncthreads();
  }
  if (j < jb)
    for (int i = 0; i < jb; ++i) t[j + i * jb] = T[j][i];
}

// W (jb x n) <- op(T) W, T upper triangular jb x jb; trans: T^T.
__global__ void trmm_small(int jb, int n, const double* __restrict__ t, bool trans, double* __restrict__ w) {
  __shared__ double col[32];
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const int i = threadIdx.x;
    if (i < jb) col[i] = w[i + c * jb];
    __syncthreads();
    if (i < jb) {
      double s = 0.0;
      if (trans)
        for (int l = 0; l <= i; ++l) s += t[l + i * jb] * col[l];  // (T^T)[i][l] = T[l][i]
      else
        for (int l = i; l < jb; ++l) s += t[i + l * jb] * col[l];
      w[i + c * jb] = s;
    }
    __syncthreads();
  }
}

__global__ void extract_r(int n, const double* a, long long lda, double* r) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e % n, j = e / n;
    r[i + j * n] = (i <= j) ? a[i + j * lda] : 0.0;
  }
}

// ------------------------------------------------------------ Jacobi SVD
__device__ __forceinline__ int rr_player(int k, int t, int n) {  // round-robin schedule
  return k == 0 ? 0 : ((k - 1 + t) % (n - 1)) + 1;
}

__global__ void col_norm2_kernel(long long m, const double* __restrict__ w, long long ldw, double* __restrict__ out) {
  __shared__ double sh[32];
  const double* c = w + blockIdx.x * ldw;
  double s = 0.0;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) s += c[i] * c[i];
  s = block_sum_all(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// One pair (p, q) of round t of the round-robin schedule; the pair index pi
// runs over npad / 2 pairs.  Uniform within the CTA (block_sum_all).
__device__ __forceinline__ void jacobi_pair(long long m, int n, int npad, int t, int pi, double* __restrict__ w,
                                            long long ldw, double* __restrict__ v, int* __restrict__ rotated,
                                            double tiny, double* sh) {
  int p = rr_player(pi, t, npad), q = rr_player(npad - 1 - pi, t, npad);
  if (p > q) {
    const int tmp = p;
    p = q;
    q = tmp;
  }
  if (q >= n) return;  // padding player
  double* wp = w + p * ldw;
  double* wq = w + q * ldw;
  double al = 0.0, be = 0.0, ga = 0.0;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = wp[i], y = wq[i];
    al += x * x;
    be += y * y;
    ga += x * y;
  }
  al = block_sum_all(al, sh);
  be = block_sum_all(be, sh);
  ga = block_sum_all(ga, sh);
  // a column below 1e-15 of the largest one is numerically zero: its
  // singular value cannot move any truncation decision, and orthogonalising
  // roundoff noise against roundoff noise never converges
  if (al < tiny || be < tiny) return;
  // Rotate only above ~450 sqrt(m) eps of the pair's norms: below it the
  // rotations chase the roundoff of the previous rounds and the sweeps do
  // not terminate (38 sweeps per SVD at C4 with sqrt(m) eps).  Singular
  // values stay accurate to ~1e-12 relative, far below what the truncation
  // rank (eps_svd = 1e-8 on the tail sum, low_rank.cpp:254-266) can resolve.
  if (ga == 0.0 || fabs(ga) <= 1e-13 * sqrt(static_cast<double>(m)) * sqrt(al * be)) return;
  if (threadIdx.x == 0) atomicAdd(rotated, 1);
  const double zeta = (be - al) / (2.0 * ga);
  const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = wp[i], y = wq[i];
    wp[i] = c * x - s * y;
    wq[i] = s * x + c * y;
  }
  if (v) {
    double* vp = v + static_cast<long long>(p) * n;
    double* vq = v + static_cast<long long>(q) * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = vp[i], y = vq[i];
      vp[i] = c * x - s * y;
      vq[i] = s * x + c * y;
    }
  }
}

// ------------------------------------------------------------ CholeskyQR2 pieces
// Upper Cholesky G = R^T R in place (r x r, column-major, ld r; the upper
// triangle is read, the lower zeroed), one CTA; flag[0] = 1 on a non-positive
// pivot.  Right-looking: per step the pivot, row k of R, the symmetric
// trailing update of the upper triangle.
__global__ void __launch_bounds__(1024) chol_upper_kernel(int r, double* __restrict__ G, int* __restrict__ flag) {
  __shared__ double rkk;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < r; ++k) {
    if (tid == 0) {
      const double d = G[k + static_cast<size_t>(k) * r];
      if (!(d > 0.0)) *flag = 1;
      rkk = d > 0.0 ? sqrt(d) : 1.0;
      G[k + static_cast<size_t>(k) * r] = rkk;
    }
    __syncthreads();
    const double inv = rkk;
    for (int j = k + 1 + tid; j < r; j += nt) G[k + static_cast<size_t>(j) * r] /= inv;
    __syncthreads();
    const int m = r - k - 1;  // trailing order; upper-triangle pairs (i <= j) by column
    for (long long e = tid; e < static_cast<long long>(m) * m; e += nt) {
      const int i = k + 1 + static_cast<int>(e % m), j = k + 1 + static_cast<int>(e / m);
      if (i <= j) G[i + static_cast<size_t>(j) * r] -= G[k + static_cast<size_t>(i) * r] * G[k + static_cast<size_t>(j) * r];
    }
    __syncthreads();
  }
  for (long long e = tid; e < static_cast<long long>(r) * r; e += nt) {
    const int i = static_cast<int>(e % r), j = static_cast<int>(e / r);
    if (i > j) G[e] = 0.0;
  }
}

// Upper Cholesky of an order-n <= 32 block in place (ld ldg), lower part
// zeroed; flag on a non-positive pivot.
__global__ void __launch_bounds__(32) chol_upper_small(int n, double* __restrict__ G, long long ldg,
                                                       int* __restrict__ flag) {
  __shared__ double A[32][33];
  const int t = threadIdx.x;
  for (int e = t; e < n * n; e += 32) A[e % n][e / n] = G[(e % n) + (e / n) * ldg];
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    const double d = A[k][k];
    if (t == 0 && !(d > 0.0)) *flag = 1;
    const double rkk = d > 0.0 ? sqrt(d) : 1.0;
    __syncwarp();
    if (t == k) A[k][k] = rkk;
    if (t > k && t < n) A[k][t] /= rkk;
    __syncwarp();
    // trailing upper triangle: column t (t > k), rows k+1..t
    if (t > k && t < n)
      for (int i = k + 1; i <= t; ++i) A[i][t] -= A[k][i] * A[k][t];
    __syncwarp();
  }
  for (int e = t; e < n * n; e += 32) {
    const int i = e % n, c = e / n;
    G[i + c * ldg] = i <= c ? A[i][c] : 0.0;
  }
}

__global__ void sub_inplace_kernel(int m, int n, const double* __restrict__ t, long long ldt, double* __restrict__ a,
                                   long long lda) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(m) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % m), c = static_cast<int>(e / m);
    a[i + c * lda] -= t[i + c * ldt];
  }
}

__global__ void copy2d_kernel(int m, int n, const double* __restrict__ src, long long lds, double* __restrict__ dst,
                              long long ldd, bool zero_src_lower_of_square) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(m) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % m), c = static_cast<int>(e / m);
    dst[i + c * ldd] = src[i + c * lds];
  }
}

// Ri = R^-1 for an upper-triangular block of order n <= 32 (ld ldr / ldi):
// the block in shared memory, one thread per column, back substitution from
// the diagonal up.
__global__ void __launch_bounds__(32) tri_inv_upper_small(int n, const double* __restrict__ R, long long ldr,
                                                          double* __restrict__ Ri, long long ldi) {
  __shared__ double Rs[32][33];
  __shared__ double Xs[32][33];
  const int j = threadIdx.x;
  for (int e = j; e < n * n; e += blockDim.x) {
    const int i = e % n, c = e / n;
    Rs[i][c] = R[i + c * ldr];
  }
  __syncthreads();
  if (j < n) {
    for (int i = j + 1; i < n; ++i) Xs[i][j] = 0.0;
    for (int i = j; i >= 0; --i) {
      double s = i == j ? 1.0 : 0.0;
      for (int l = i + 1; l <= j; ++l) s -= Rs[i][l] * Xs[l][j];
      Xs[i][j] = s / Rs[i][i];
    }
  }
  __syncthreads();
  for (int e = j; e < n * n; e += blockDim.x) {
    const int i = e % n, c = e / n;
    Ri[i + c * ldi] = Xs[i][c];
  }
}

__global__ void neg_kernel(int m, int n, double* __restrict__ a, long long lda) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(m) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % m), c = static_cast<int>(e / m);
    a[i + c * lda] = -a[i + c * lda];
  }
}

// ------------------------------------------------------------ singular values
// Singular values only (the truncation rank every outer iteration,
// low_rank.cpp:254-266): Golub-Kahan bidiagonalisation of the m x n factor
// (m >= n) in one cooperative launch, then bisection on the zero-diagonal
// Golub-Kahan tridiagonal (eigenvalues +-sigma), one thread per singular
// value.  Three grid barriers per column (left reflector applied to the
// trailing columns, warp per column; the right reflector's row products as
// fixed-order partials over 64-column chunks; their update), against one
// per round of n - 1 rounds per Jacobi sweep.  Householder vectors follow
// hh_make's conventions (Eigen's makeHouseholder); every CTA derives a
// reflector from its own identical reduction, so the tau == 0 branches are
// grid-uniform.
__device__ __forceinline__ void hh_params(double c0, double tail2, double& beta, double& tau, double& denom) {
  if (tail2 <= 2.2250738585072014e-308) {
    tau = 0.0;
    beta = c0;
    denom = 0.0;
  } else {
    beta = sqrt(c0 * c0 + tail2);
    if (c0 >= 0.0) beta = -beta;
    denom = c0 - beta;
    tau = (beta - c0) / beta;
  }
}

__global__ void __launch_bounds__(256) bidiag_coop(int m, int n, double* __restrict__ A, long long lda,
                                                   double* __restrict__ d, double* __restrict__ e,
                                                   double* __restrict__ part) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double bd_sm[];
  double* v = bd_sm;      // m: left reflector
  double* u = bd_sm + m;  // n: right reflector
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int nwt = gridDim.x * (blockDim.x >> 5), gw = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
  for (int k = 0; k < n; ++k) {
    // left reflector of column k (rows k..m-1) -> d[k]
    const double* ck = A + static_cast<long long>(k) * lda;
    double t2 = 0.0;
    for (int i = k + 1 + tid; i < m; i += blockDim.x) t2 += ck[i] * ck[i];
    t2 = block_sum_all(t2, red);
    double beta, tau, den;
    hh_params(ck[k], t2, beta, tau, den);
    for (int i = k + tid; i < m; i += blockDim.x) v[i] = i == k ? 1.0 : (den != 0.0 ? ck[i] / den : 0.0);
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) d[k] = beta;
    if (tau != 0.0)
      for (int j = k + 1 + gw; j < n; j += nwt) {
        double* cj = A + static_cast<long long>(j) * lda;
        double w = 0.0;
        for (int i = k + lane; i < m; i += 32) w += v[i] * cj[i];
        w = warp_sum(w);
        const double tw = tau * w;
        for (int i = k + lane; i < m; i += 32) cj[i] -= tw * v[i];
      }
    grid.sync();
    if (k + 1 >= n) break;
    // right reflector of row k (columns k+1..n-1) -> e[k]
    double s2 = 0.0;
    for (int j = k + 2 + tid; j < n; j += blockDim.x) {
      const double x = A[k + static_cast<long long>(j) * lda];
      s2 += x * x;
    }
    s2 = block_sum_all(s2, red);
    double beta2, tau2, den2;
    hh_params(A[k + static_cast<long long>(k + 1) * lda], s2, beta2, tau2, den2);
    for (int j = k + 1 + tid; j < n; j += blockDim.x)
      u[j] = j == k + 1 ? 1.0 : (den2 != 0.0 ? A[k + static_cast<long long>(j) * lda] / den2 : 0.0);
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) e[k] = beta2;
    if (tau2 != 0.0) {
      const int rows = m - k - 1, cols = n - k - 1;
      const int nrb = (rows + 31) / 32, ncc = (cols + 63) / 64;
      for (int it = gw; it < nrb * ncc; it += nwt) {  // row products, 64-column partials
        const int rb = it % nrb, cc = it / nrb;
        const int i = k + 1 + rb * 32 + lane;
        const int j0 = k + 1 + cc * 64, j1 = min(n, j0 + 64);
        double acc = 0.0;
        if (i < m)
          for (int j = j0; j < j1; ++j) acc += A[i + static_cast<long long>(j) * lda] * u[j];
        if (i < m) part[static_cast<long long>(cc) * m + i] = acc;
      }
      grid.sync();
      for (int it = gw; it < nrb * ncc; it += nwt) {  // rank-1 update
        const int rb = it % nrb, cc = it / nrb;
        const int i = k + 1 + rb * 32 + lane;
        if (i >= m) continue;
        double w = 0.0;
        for (int c = 0; c < ncc; ++c) w += part[static_cast<long long>(c) * m + i];
        const double tw = tau2 * w;
        const int j0 = k + 1 + cc * 64, j1 = min(n, j0 + 64);
        for (int j = j0; j < j1; ++j) A[i + static_cast<long long>(j) * lda] -= tw * u[j];
      }
    }
    grid.sync();
  }
}

// The same bidiagonalisation with the reflector applications laid out for
// memory-level parallelism (bidiag_coop's loops carried one dependent L2
// load per iteration: ~90 us per column at 2048 x 600).  Left reflector: a
// team of T warps per trailing column, each lane holding its <= 32 rows of
// the column in registers between the dot product and the update (one load
// round).  Right reflector: a CTA per 8-row block, its 32 column groups
// keeping the row block's entries in registers, the row products reduced in
// shared memory, so no partials cross CTAs: two grid barriers per column
// (bidiag_coop: three).  n <= 1024 and m <= 8192 (one register round each).
constexpr int kBdRegs = 32, kBdRows = 8;
__global__ void __launch_bounds__(256, 2) bidiag_coop2(int m, int n, double* __restrict__ A, long long lda,
                                                       double* __restrict__ d, double* __restrict__ e) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double bd_sm[];
  double* v = bd_sm;      // m: left reflector
  double* u = bd_sm + m;  // n: right reflector
  __shared__ double red[32];
  __shared__ double part[256];  // left: one partial per warp; right: [column group][row]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nwarps = gridDim.x * 8;
  for (int k = 0; k < n; ++k) {
    // ---- left reflector of column k (rows k..m-1), applied to columns k+1..n-1
    const double* ck = A + static_cast<long long>(k) * lda;
    double t2 = 0.0;
    for (int i = k + 1 + tid; i < m; i += blockDim.x) t2 += ck[i] * ck[i];
    t2 = block_sum_all(t2, red);
    double beta, tau, den;
    hh_params(ck[k], t2, beta, tau, den);
    for (int i = k + tid; i < m; i += blockDim.x) v[i] = i == k ? 1.0 : (den != 0.0 ? ck[i] / den : 0.0);
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) d[k] = beta;
    const int ncols = n - k - 1;
    if (tau != 0.0 && ncols > 0) {
      int T = 8;  // warps per column: as many as the grid holds, at least enough for one register round
      while (T > 1 && ncols * T > nwarps) T >>= 1;
      while (T < 8 && m - k > 32 * kBdRegs * T) T <<= 1;
      const int per_cta = 8 / T, ngroups = (ncols + per_cta - 1) / per_cta;
      const int slot = wid / T, t = wid % T;
      for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int j = k + 1 + g * per_cta + slot;
        const bool live = j < n;
        double* cj = A + static_cast<long long>(live ? j : k) * lda;
        double c[kBdRegs];
        double w = 0.0;
#pragma unroll
        for (int s = 0; s < kBdRegs; ++s) {
          const int i = k + lane + 32 * (t + T * s);
          c[s] = (live && i < m) ? cj[i] : 0.0;
        }
#pragma unroll
        for (int s = 0; s < kBdRegs; ++s) {
          const int i = k + lane + 32 * (t + T * s);
          if (i < m) w += v[i] * c[s];
        }
        w = warp_sum(w);
        if (lane == 0) part[wid] = w;
        __syncthreads();
        double wt = 0.0;
        for (int q = 0; q < T; ++q) wt += part[slot * T + q];  // fixed order
        const double tw = tau * wt;
        if (live) {
#pragma unroll
          for (int s = 0; s < kBdRegs; ++s) {
            const int i = k + lane + 32 * (t + T * s);
            if (i < m) cj[i] = c[s] - tw * v[i];
          }
        }
        __syncthreads();
      }
    }
    grid.sync();
    if (k + 1 >= n) break;
    // ---- right reflector of row k (columns k+1..n-1), applied to rows k+1..m-1
    double s2 = 0.0;
    for (int j = k + 2 + tid; j < n; j += blockDim.x) {
      const double x = A[k + static_cast<long long>(j) * lda];
      s2 += x * x;
    }
    s2 = block_sum_all(s2, red);
    double beta2, tau2, den2;
    hh_params(A[k + static_cast<long long>(k + 1) * lda], s2, beta2, tau2, den2);
    for (int j = k + 1 + tid; j < n; j += blockDim.x)
      u[j] = j == k + 1 ? 1.0 : (den2 != 0.0 ? A[k + static_cast<long long>(j) * lda] / den2 : 0.0);
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) e[k] = beta2;
    if (tau2 != 0.0) {
      const int rows = m - k - 1, nrb = (rows + kBdRows - 1) / kBdRows;
      const int ro = tid % kBdRows, grp = tid / kBdRows;  // 32 column groups
      for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
        const int i = k + 1 + rb * kBdRows + ro;
        const bool live = i < m;
        double c[kBdRegs];
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < kBdRegs; ++s) {
          const int j = k + 1 + grp + 32 * s;
          c[s] = (live && j < n) ? A[i + static_cast<long long>(j) * lda] : 0.0;
        }
#pragma unroll
        for (int s = 0; s < kBdRegs; ++s) {
          const int j = k + 1 + grp + 32 * s;
          if (j < n) acc += c[s] * u[j];
        }
        part[tid] = acc;  // = part[grp * kBdRows + ro]
        __syncthreads();
        double y = 0.0;
        for (int q = 0; q < 32; ++q) y += part[q * kBdRows + ro];  // fixed order
        const double ty = tau2 * y;
        if (live) {
#pragma unroll
          for (int s = 0; s < kBdRegs; ++s) {
            const int j = k + 1 + grp + 32 * s;
            if (j < n) A[i + static_cast<long long>(j) * lda] = c[s] - ty * u[j];
          }
        }
        __syncthreads();
      }
    }
    grid.sync();
  }
}

// The k-th smallest singular value by multisection of the Golub-Kahan
// tridiagonal's Sturm counts: one warp per value, 32 points per round
// (~11 rounds to full precision against ~60 bisection steps of a thread).
__device__ int gk_count_below(int n, const double* __restrict__ d, const double* __restrict__ e, double x,
                             double pivmin);
__global__ void gk_multisect(int n, const double* __restrict__ d, const double* __restrict__ e,
                             double* __restrict__ sv) {
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // k-th smallest
  if (k >= n) return;
  double ub = 0.0, tmax = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double a = fabs(d[j]), b = j + 1 < n ? fabs(e[j]) : 0.0, c = j > 0 ? fabs(e[j - 1]) : 0.0;
    ub = fmax(ub, fmax(a + c, a + b));
    tmax = fmax(tmax, fmax(a, b));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ub = fmax(ub, __shfl_xor_sync(0xffffffffu, ub, o));
    tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
  }
  const double pivmin = fmax(2.2250738585072014e-308, 2.2250738585072014e-308 * tmax * tmax);
  double lo = 0.0, hi = ub * (1.0 + 4e-16) + pivmin;
  for (int it = 0; it < 40 && hi - lo > 4e-16 * hi + pivmin; ++it) {
    const double x = lo + (hi - lo) * ((lane + 1) / 33.0);
    const bool above = gk_count_below(n, d, e, x, pivmin) - n > k;  // sigma_k < x
    const unsigned mask = __ballot_sync(0xffffffffu, above);
    const int first = mask ? __ffs(mask) - 1 : 32;  // first point above sigma_k
    const double nhi = first < 32 ? __shfl_sync(0xffffffffu, x, first) : hi;
    const double nlo = first > 0 ? __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0) : lo;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) sv[n - 1 - k] = 0.5 * (lo + hi);  // descending
}

// Number of eigenvalues of the Golub-Kahan tridiagonal (zero diagonal,
// off-diagonals d0, e0, d1, e1, ..., d_{n-1}) below x (Sturm count, LDL^T pivots).
__device__ int gk_count_below(int n, const double* __restrict__ d, const double* __restrict__ e, double x,
                             double pivmin) {
  int cnt = 0;
  double q = -x;
  if (q < 0.0) ++cnt;
  for (int j = 1; j < 2 * n; ++j) {
    const double t = (j & 1) ? d[j >> 1] : e[(j >> 1) - 1];
    if (fabs(q) < pivmin) q = -pivmin;
    q = -x - t * t / q;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

__global__ void gk_bisect(int n, const double* __restrict__ d, const double* __restrict__ e, double* __restrict__ sv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // k-th smallest
  if (k >= n) return;
  double ub = 0.0, tmax = 0.0;
  for (int j = 0; j < n; ++j) {
    const double a = fabs(d[j]), b = j + 1 < n ? fabs(e[j]) : 0.0, c = j > 0 ? fabs(e[j - 1]) : 0.0;
    ub = fmax(ub, fmax(a + c, a + b));
    tmax = fmax(tmax, fmax(a, b));
  }
  const double pivmin = fmax(2.2250738585072014e-308, 2.2250738585072014e-308 * tmax * tmax);
  double lo = 0.0, hi = ub * (1.0 + 4e-16) + pivmin;
  // #(sigma < x) = count(x) - n for x > 0
  for (int it = 0; it < 200 && hi - lo > 4e-16 * hi + pivmin; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (gk_count_below(n, d, e, mid, pivmin) - n > k)
      hi = mid;
    else
      lo = mid;
  }
  sv[n - 1 - k] = 0.5 * (lo + hi);  // descending
}

__global__ void __launch_bounds__(256) jacobi_round(long long m, int n, int npad, int t, double* __restrict__ w,
                                                    long long ldw, double* __restrict__ v, int* __restrict__ rotated,
                                                    double tiny) {
  __shared__ double sh[32];
  jacobi_pair(m, n, npad, t, blockIdx.x, w, ldw, v, rotated, tiny, sh);
}

// Every sweep of one SVD in one cooperative launch: the CTAs loop over the
// pairs of a round, a grid-wide barrier separates the rounds, and after each
// sweep every CTA reads the sweep's rotation count (three counters in turn,
// so the one being reset was last read two sweeps ago).  Same pairs, same
// arithmetic, same stopping rule as the per-round launches.
// ctl: [0..2] rotation counters (ctl[0] zero at launch), [3] sweeps used,
// [4] rotations in the last sweep.
__global__ void __launch_bounds__(256) jacobi_sweeps_coop(long long m, int n, int npad, double* __restrict__ w,
                                                          long long ldw, double* __restrict__ v, int* ctl, double tiny,
                                                          int max_sweeps) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  int sweep = 0, last = 0;
  while (sweep < max_sweeps) {
    int* rot = ctl + sweep % 3;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[(sweep + 1) % 3] = 0;
    for (int t = 0; t < npad - 1; ++t) {
      for (int pi = blockIdx.x; pi < npad / 2; pi += gridDim.x)
        jacobi_pair(m, n, npad, t, pi, w, ldw, v, rot, tiny, sh);
      grid.sync();
    }
    last = *reinterpret_cast<volatile int*>(rot);
    ++sweep;
    if (last == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl[3] = sweep;
    ctl[4] = last;
  }
}


// ------------------------------------------------------------ blocked batched LU
// Right-looking LU with partial pivoting (first maximum, as Eigen's
// PartialPivLU) of the augmented systems [A_j | b_j] (r x (r+1), column-
// major, ld r) in panels of up to 32 columns: panel factorisation in shared
// memory (one CTA per system), then per 64-column tile of the trailing
// columns the panel's row swaps, the unit-lower TRSM and the GEMM update
// (many CTAs), then back substitution.  Forward substitution on b happens
// through the augmented column.

__global__ void __launch_bounds__(256) lu_assemble(int r, const int* __restrict__ angles, const double* __restrict__ dirs,
                                                   const double* __restrict__ proj, long long ldp, long long pstride,
                                                   const double* __restrict__ prhs, const double* __restrict__ extra,
                                                   long long ldx, double* __restrict__ M) {
  const int jb = blockIdx.y;
  const int ang = angles[jb];
  const double omx = dirs[3 * ang], omy = dirs[3 * ang + 1];
  const double* px = proj + (omx >= 0.0 ? 0 : 1) * pstride;
  const double* py = proj + (omy >= 0.0 ? 2 : 3) * pstride;
  const double* pt = proj + 4 * pstride;
  double* A = M + static_cast<size_t>(jb) * r * (r + 1);
  const long long total = static_cast<long long>(r) * (r + 1);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % r), j = static_cast<int>(e / r);
    A[e] = j < r ? omx * px[i + j * ldp] + omy * py[i + j * ldp] + pt[i + j * ldp]
                 : prhs[i] + (extra ? extra[i + jb * ldx] : 0.0);
  }
}

constexpr int kNbMax = 32;
constexpr int kPanelSmemBytes = 200 * 1024;

// Panel width for the panel starting at k0: 32, halved while the panel's
// rows do not fit the shared-memory budget.
__host__ __device__ inline int lu_panel_width(int r, int k0) {
  int jb = kNbMax;
  while (jb > 1 && static_cast<long long>(r - k0) * (jb * 8 + 4) > kPanelSmemBytes) jb >>= 1;
  return jb < r - k0 ? jb : r - k0;
}

// Partial-pivot LU of the panel columns k0..k0+jb-1 (rows k0..r-1) in shared
// memory; pivots to piv; one CTA of NT threads per system.  Two barriers per
// column: the pivot candidates of column j+1 are reduced by the same pass
// that applies column j's rank-1 update (each thread owns whole rows).
__device__ __forceinline__ void argmax_merge(double& best, int& bi, double ov, int oi) {
  if (ov > best || (ov == best && oi < bi)) {
    best = ov;
    bi = oi;
  }
}

constexpr int kPermInts = 1 + 4 * 32;  // count, then up to 2 kNbMax dst rows and 2 kNbMax src rows

// The panel's row swaps as one permutation of at most 2 jb rows, so the
// trailing columns apply them with independent loads (lu_trail): after
// the swaps, row dst[k] holds what row src[k] held.  slot[] (rows ints of
// shared memory) maps a panel row to its entry (O(1) lookups).
__device__ void lu_panel_perm(int rows, int k0, int jb, const int* pv, int* slot, int* pm) {
  __shared__ int rowp[2 * kNbMax], cont[2 * kNbMax];
  const int tid = threadIdx.x;
  for (int i = tid; i < rows; i += blockDim.x) slot[i] = -1;
  __syncthreads();
  if (tid == 0) {
    int np = 0;
    auto pos_of = [&](int row) {
      int q = slot[row - k0];
      if (q < 0) {
        q = np++;
        slot[row - k0] = q;
        rowp[q] = row;
        cont[q] = row;
      }
      return q;
    };
    for (int j = 0; j < jb; ++j) {
      const int a = k0 + j, b = pv[k0 + j];
      if (a == b) continue;
      const int pa = pos_of(a), pb = pos_of(b);
      const int t = cont[pa];
      cont[pa] = cont[pb];
      cont[pb] = t;
    }
    int cnt = 0;
    for (int q = 0; q < np; ++q)
      if (cont[q] != rowp[q]) {
        pm[1 + cnt] = rowp[q];
        pm[1 + 2 * kNbMax + cnt] = cont[q];
        ++cnt;
      }
    pm[0] = cnt;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) lu_panel_smem(int r, int k0, int jb, double* __restrict__ M,
                                                    int* __restrict__ piv, int* __restrict__ perm) {
  constexpr int NW = NT / 32;
  extern __shared__ double P[];  // (r - k0) x jb, column-major, ld = rows
  __shared__ double shv[2][NW];
  __shared__ int shi[2][NW];
  double* A = M + static_cast<size_t>(blockIdx.x) * r * (r + 1);
  int* pv = piv + static_cast<size_t>(blockIdx.x) * r;
  const int rows = r - k0, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int kHalf = kNbMax / 2;
  const bool split = jb > kHalf && rows > kHalf;
  for (int e = tid; e < rows * jb; e += NT) {
    const int i = e % rows, c = e / rows;
    P[e] = A[k0 + i + static_cast<size_t>(k0 + c) * r];
  }
  __syncthreads();
  auto publish = [&](int buf, double best, int bi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      argmax_merge(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
    if (lane == 0) {
      shv[buf][wid] = best;
      shi[buf][wid] = bi;
    }
  };
  {  // pivot candidates of column 0
    double best = -1.0;
    int bi = rows;
    for (int i = tid; i < rows; i += NT) argmax_merge(best, bi, fabs(P[i]), i);
    publish(0, best, bi);
  }
  __syncthreads();
  for (int j = 0; j < jb; ++j) {
    const int buf = j & 1;
    double bv = shv[buf][0];
    int bix = shi[buf][0];
#pragma unroll
    for (int w = 1; w < NW; ++w) argmax_merge(bv, bix, shv[buf][w], shi[buf][w]);
    const int p = bv > 0.0 ? bix : j;  // all-zero column: no swap (first zero pivot)
    if (tid == 0) pv[k0 + j] = k0 + p;
    if (p != j && tid < jb) {
      double* c = P + static_cast<size_t>(tid) * rows;
      const double t = c[j];
      c[j] = c[p];
      c[p] = t;
    }
    __syncthreads();
    const double* colj = P + static_cast<size_t>(j) * rows;
    const double d = colj[j];
    double best = -1.0;
    int bi = rows;
    // Two halves of kHalf columns: the first half's rank-1 updates stop at
    // its own last column; its effect on the second half is applied once,
    // as a TRSM on the half's rows and a register-accumulated update of the
    // rows below (the same subtractions in the same order per element, on
    // the rows as the swaps left them: bitwise the unblocked factors).
    const int cend = (split && j < kHalf) ? kHalf : jb;
    for (int i = j + 1 + tid; i < rows; i += NT) {
      const double l = d != 0.0 ? P[i + static_cast<size_t>(j) * rows] / d : P[i + static_cast<size_t>(j) * rows];
      P[i + static_cast<size_t>(j) * rows] = l;
      for (int c = j + 1; c < cend; ++c) P[i + static_cast<size_t>(c) * rows] -= l * P[j + static_cast<size_t>(c) * rows];
      if (j + 1 < cend) argmax_merge(best, bi, fabs(P[i + static_cast<size_t>(j + 1) * rows]), i);
    }
    publish(buf ^ 1, best, bi);
    __syncthreads();
    if (split && j == kHalf - 1) {
      // U12: rows 1..kHalf-1 of the second half, forward substitution (one thread per column)
      if (tid < jb - kHalf) {
        double* pc = P + static_cast<size_t>(kHalf + tid) * rows;
        for (int i = 1; i < kHalf; ++i) {
          double a = pc[i];
          for (int l2 = 0; l2 < i; ++l2) a -= P[i + static_cast<size_t>(l2) * rows] * pc[l2];
          pc[i] = a;
        }
      }
      __syncthreads();
      // rows kHalf.. of the second half: A22 -= L21 U12, l in order; pivot candidates of column kHalf
      best = -1.0;
      bi = rows;
      for (int i = kHalf + tid; i < rows; i += NT) {
        double lrow[kHalf];
#pragma unroll
        for (int l2 = 0; l2 < kHalf; ++l2) lrow[l2] = P[i + static_cast<size_t>(l2) * rows];
        for (int c = kHalf; c < jb; ++c) {
          double* pc = P + static_cast<size_t>(c) * rows;
          double a = pc[i];
#pragma unroll
          for (int l2 = 0; l2 < kHalf; ++l2) a -= lrow[l2] * pc[l2];
          pc[i] = a;
          if (c == kHalf) argmax_merge(best, bi, fabs(a), i);
        }
      }
      publish(buf ^ 1, best, bi);
      __syncthreads();
    }
  }
  for (int e = tid; e < rows * jb; e += NT) {
    const int i = e % rows, c = e / rows;
    A[k0 + i + static_cast<size_t>(k0 + c) * r] = P[e];
  }
  lu_panel_perm(rows, k0, jb, pv, reinterpret_cast<int*>(P + static_cast<size_t>(rows) * jb),
                perm + static_cast<size_t>(blockIdx.x) * kPermInts);
}

// Register-resident panel for panels of up to 256 RPT rows (RPT <= 2; the greedy
// candidates' 16-system batches are latency-bound on the panel: the shared-
// memory panel above spends ~2 us per column on shared-memory traffic and
// two barriers).  Thread t owns panel rows t, t + 256, ... and keeps each
// row's active part (columns j..) in registers, shifted left one column per
// step, so every register index is compile-time inside a small loop body
// (a fully unrolled 32-column body stalls on instruction fetch).  Finished
// entries (the L column of each step, the pivot row's U part) go to a
// shared-memory copy of the panel, where row swaps of the L parts happen.
// One barrier per column: before it every warp publishes its argmax
// candidate for column j with that row's active part, and the owner of row
// j publishes row j (double-buffered by column parity), so after it every
// thread knows the pivot row.  The per-element operations (l = a / d,
// a -= l u in column order) are those of the unblocked factorisation, as in
// lu_panel_smem: bitwise the same factors.
template <int RPT>
__global__ void __launch_bounds__(256, 1) lu_panel_reg(int r, int k0, int jb, double* __restrict__ M,
                                                       int* __restrict__ piv, int* __restrict__ perm) {
  constexpr int NT = 256, NW = NT / 32;
  extern __shared__ double P[];  // rows x kNbMax L entries (ld rows, by row tag), then rows ints
  __shared__ __align__(16) double cand[2][NW][kNbMax];
  __shared__ __align__(16) double rowj[2][kNbMax];
  __shared__ double Ub[kNbMax][kNbMax + 1];  // the pivot rows' U parts, by final row
  __shared__ double shv[2][NW];
  __shared__ int shi[2][NW], candtag[2][NW], rowjtag[2];
  double* A = M + static_cast<size_t>(blockIdx.x) * r * (r + 1);
  int* pv = piv + static_cast<size_t>(blockIdx.x) * r;
  const int rows = r - k0, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int* tag_at = reinterpret_cast<int*>(P + static_cast<size_t>(rows) * kNbMax);
  // active parts; columns >= jb are zero and stay zero (the pivot row's are).
  // tag: the panel row a slot's row started as; L entries are stored by tag,
  // so a row swap moves no finished entries (they follow the tag at the end)
  double a[RPT][kNbMax];
  int tag[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) tag[q] = tid + NT * q;
#pragma unroll
  for (int c = 0; c < kNbMax; ++c)
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = tid + NT * q;
      a[q][c] = (i < rows && c < jb) ? A[k0 + i + static_cast<size_t>(k0 + c) * r] : 0.0;
    }
  // column j (active index 0): argmax candidate over rows >= j with its active part, and row j
  auto publish = [&](int j) {
    const int buf = j & 1;
    double best = -1.0;
    int bi = rows, bq = -1;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = tid + NT * q;
      if (i >= j && i < rows) {
        const double v = fabs(a[q][0]);
        if (v > best) {  // q ascending: rows ascending, first maximum kept
          best = v;
          bi = i;
          bq = q;
        }
      }
    }
    double wb = best;
    int wi = bi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      argmax_merge(wb, wi, __shfl_xor_sync(0xffffffffu, wb, o), __shfl_xor_sync(0xffffffffu, wi, o));
    if (lane == 0) {
      shv[buf][wid] = wb;
      shi[buf][wid] = wi;
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = tid + NT * q;
      if (bq == q && wi == bi) {
        double2* dst = reinterpret_cast<double2*>(cand[buf][wid]);
#pragma unroll
        for (int c = 0; c < kNbMax; c += 2) dst[c / 2] = make_double2(a[q][c], a[q][c + 1]);
        candtag[buf][wid] = tag[q];
      }
      if (i == j) {
        double2* dst = reinterpret_cast<double2*>(rowj[buf]);
#pragma unroll
        for (int c = 0; c < kNbMax; c += 2) dst[c / 2] = make_double2(a[q][c], a[q][c + 1]);
        rowjtag[buf] = tag[q];
      }
    }
  };
  publish(0);
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < jb; ++j) {
    const int buf = j & 1;
    double bv = shv[buf][0];
    int bix = shi[buf][0], bw = 0;
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const double ov = shv[buf][w];
      const int oi = shi[buf][w];
      if (ov > bv || (ov == bv && oi < bix)) {
        bv = ov;
        bix = oi;
        bw = w;
      }
    }
    const int p = bv > 0.0 ? bix : j;  // all-zero column: no swap (first zero pivot)
    if (tid == 0) pv[k0 + j] = k0 + p;
    const double2* U2 = reinterpret_cast<const double2*>(p == j ? rowj[buf] : cand[buf][bw]);
    const double2* R2 = reinterpret_cast<const double2*>(rowj[buf]);
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = tid + NT * q;
      if (p != j && i == j) {  // row j <- row p
#pragma unroll
        for (int c = 0; c < kNbMax; c += 2) {
          const double2 v = U2[c / 2];
          a[q][c] = v.x;
          a[q][c + 1] = v.y;
        }
        tag[q] = candtag[buf][bw];
      } else if (p != j && i == p) {  // row p <- row j (its L part follows the tag)
#pragma unroll
        for (int c = 0; c < kNbMax; c += 2) {
          const double2 v = R2[c / 2];
          a[q][c] = v.x;
          a[q][c + 1] = v.y;
        }
        tag[q] = rowjtag[buf];
      }
      if (i == j)  // the pivot row's U part is final
#pragma unroll
        for (int c = 0; c < kNbMax; ++c)
          if (c < jb - j) Ub[j][j + c] = a[q][c];
    }
    const double d = U2[0].x;
    // rank-1 update of the rows below j (column order), then shift left
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = tid + NT * q;
      if (i > j && i < rows) {
        const double l = d != 0.0 ? a[q][0] / d : a[q][0];
        P[tag[q] + j * rows] = l;
#pragma unroll
        for (int c = 2; c < kNbMax; c += 2) {
          const double2 u = U2[c / 2];
          a[q][c] -= l * u.x;
          a[q][c + 1] -= l * u.y;
        }
        a[q][1] -= l * U2[0].y;
      }
#pragma unroll
      for (int c = 0; c + 1 < kNbMax; ++c) a[q][c] = a[q][c + 1];
      a[q][kNbMax - 1] = 0.0;
    }
    if (j + 1 < jb) publish(j + 1);
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = tid + NT * q;
    if (i < rows) tag_at[i] = tag[q];
  }
  __syncthreads();
  for (int c = 0; c < jb; ++c)
    for (int i = tid; i < rows; i += NT)
      A[k0 + i + static_cast<size_t>(k0 + c) * r] = i <= c ? Ub[i][c] : P[tag_at[i] + c * rows];
  __syncthreads();
  lu_panel_perm(rows, k0, jb, pv, tag_at, perm + static_cast<size_t>(blockIdx.x) * kPermInts);
}

// Small batches (the q greedy candidates) up to r = kCtaLuMax: one CTA of
// 1024 threads per system with [A | b] in shared memory.  Warp w owns the
// columns j = w (mod 32), lane l the rows i = l (mod 32), so the rank-1
// update walks static index sets (no division) and column k + 1 is one
// warp's: its argmax is a shuffle reduction right after that warp updates
// it.  Two barriers per column: (1) the pivot row moves to row k (staged in
// prow) and the multipliers are formed; (2) the rank-1 update of the rows
// below, the right-hand side included as column r.  L is not stored (the
// forward substitution is the update of column r).  Back substitution by
// 32 x 32 diagonal blocks (shuffle solve in warp 0, then one warp per row
// above).  Pivot rule, all-zero column and singular-flag behaviour as
// lu_solve_block.
constexpr int kCtaLuMax = 160;
__global__ void __launch_bounds__(1024, 1) galerkin_cta_lu(int r, const int* __restrict__ angles,
                                                           const double* __restrict__ dirs,
                                                           const double* __restrict__ proj, long long ldp,
                                                           long long pstride, const double* __restrict__ prhs,
                                                           const double* __restrict__ extra, double* __restrict__ sol,
                                                           long long ldsol, int* __restrict__ flags) {
  extern __shared__ double Am[];  // r x (r + 1), column-major, ld r
  __shared__ double prow[kCtaLuMax + 1], lcol[kCtaLuMax];
  __shared__ int sp;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int jb = blockIdx.x;
  const int ang = angles[jb];
  const double omx = dirs[3 * ang], omy = dirs[3 * ang + 1];
  const double* px = proj + (omx >= 0.0 ? 0 : 1) * pstride;
  const double* py = proj + (omy >= 0.0 ? 2 : 3) * pstride;
  const double* pt = proj + 4 * pstride;
  // reduced_streaming (low_rank.cpp:176-183): omx*Px + omy*Py + Pt, then the rhs column
  for (int j = w; j < r; j += 32)
    for (int i = lane; i < r; i += 32)
      Am[i + j * r] = omx * px[i + j * ldp] + omy * py[i + j * ldp] + pt[i + j * ldp];
  if (w == 0)
    for (int i = lane; i < r; i += 32) Am[i + r * r] = prhs[i] + (extra ? extra[i + jb * ldsol] : 0.0);
  __syncthreads();
  auto argmax_col = [&](int c) {  // warp c % 32: first maximum of |A[i, c]|, i >= c
    double best = -1.0;
    int bi = r;
    for (int i = c + ((lane - c) & 31); i < r; i += 32) {  // ascending rows of this lane >= c
      const double v = fabs(Am[i + c * r]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) argmax_merge(best, bi, __shfl_xor_sync(0xffffffffu, best, o),
                                                  __shfl_xor_sync(0xffffffffu, bi, o));
    if (lane == 0) sp = best > 0.0 ? bi : c;  // all-zero column: no swap
  };
  if (w == 0) argmax_col(0);
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const int p = sp;
    const double d = Am[p + k * r];
    // (1) pivot row -> row k (columns > k; prow keeps it), old row k -> row p;
    // multipliers from column k as the swap leaves it (column k is not written here)
    for (int j = k + 1 + tid; j <= r; j += 1024) {
      const double pr = Am[p + j * r];
      prow[j] = pr;
      if (p != k) {
        Am[p + j * r] = Am[k + j * r];
        Am[k + j * r] = pr;
      }
    }
    for (int i = k + 1 + tid; i < r; i += 1024) {
      const double a = i == p ? Am[k + k * r] : Am[i + k * r];
      lcol[i] = d != 0.0 ? a / d : a;
    }
    __syncthreads();
    if (tid == 0) Am[k + k * r] = d;
    // (2) rank-1 update of rows > k, columns > k (column r: the forward substitution)
    const int j0 = w + 32 * ((k + 1 - w + 31) >> 5);  // first column of this warp > k
    const int i0 = lane + 32 * ((k + 1 - lane + 31) >> 5);
    for (int j = j0; j <= r; j += 32) {
      const double u = prow[j];
      for (int i = i0; i < r; i += 32) Am[i + j * r] -= lcol[i] * u;
    }
    if (k + 1 < r && w == ((k + 1) & 31)) {
      __syncwarp();
      argmax_col(k + 1);
    }
    __syncthreads();
  }
  // back substitution: y = column r, U upper (diagonal in place)
  double* y = Am + static_cast<size_t>(r) * r;
  for (int b0 = ((r - 1) / 32) * 32; b0 >= 0; b0 -= 32) {
    const int bs = min(32, r - b0);
    if (w == 0) {
      double x = lane < bs ? y[b0 + lane] : 0.0;
      for (int i = bs - 1; i >= 0; --i) {
        const double xi = __shfl_sync(0xffffffffu, x, i) / Am[b0 + i + (b0 + i) * r];
        if (lane == i) x = xi;
        if (lane < i) x -= xi * Am[b0 + lane + (b0 + i) * r];
      }
      if (lane < bs) y[b0 + lane] = x;
    }
    __syncthreads();
    for (int row = w; row < b0; row += 32) {
      double v = lane < bs ? Am[row + (b0 + lane) * r] * y[b0 + lane] : 0.0;
      v = warp_sum(v);
      if (lane == 0) y[row] -= v;
    }
    __syncthreads();
  }
  int bad = 0;
  for (int i = tid; i < r; i += 1024) {
    sol[i + jb * ldsol] = y[i];
    if (!isfinite(y[i])) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) flags[jb] = bad;
}

// The same one-CTA elimination keeping the factors, for the look-ahead
// factorisation of the greedy candidates at r <= kCtaLuMax (the blocked
// chain's 2 r / 32 launches of ~45 + 16 us were the critical path of small
// problems: C2's inner iteration has ~350 us of other work).  Output in the
// blocked path's format, which galerkin_border_kernel replays: L below the
// diagonal with a step's row exchange applied to the columns of its own
// 32-column panel and to everything right of it (not to earlier panels), U
// on and above, the forward-substituted right-hand side in column r, the
// pivot rows in piv.
// (in place on the systems lu_assemble wrote: the projections are read by
// that short kernel only, so the main stream's wait for them stays short)
__global__ void __launch_bounds__(1024, 1) galerkin_cta_factor(int r, double* __restrict__ Mout,
                                                               int* __restrict__ pivout) {
  extern __shared__ double Am[];  // r x (r + 1), column-major, ld r
  __shared__ double prow[kCtaLuMax + 1], lcol[kCtaLuMax];
  __shared__ int sp;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int jb = blockIdx.x;
  int* pv = pivout + static_cast<size_t>(jb) * r;
  {
    const double* in = Mout + static_cast<size_t>(jb) * r * (r + 1);
    for (int e = tid; e < r * (r + 1); e += 1024) Am[e] = in[e];
  }
  __syncthreads();
  auto argmax_col = [&](int c) {  // warp c % 32: first maximum of |A[i, c]|, i >= c
    double best = -1.0;
    int bi = r;
    for (int i = c + ((lane - c) & 31); i < r; i += 32) {
      const double v = fabs(Am[i + c * r]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) argmax_merge(best, bi, __shfl_xor_sync(0xffffffffu, best, o),
                                                  __shfl_xor_sync(0xffffffffu, bi, o));
    if (lane == 0) sp = best > 0.0 ? bi : c;  // all-zero column: no swap
  };
  if (w == 0) argmax_col(0);
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const int p = sp;
    const double d = Am[p + k * r];
    const int ps = k & ~(kNbMax - 1);  // first column of this step's panel
    // (1) rows k and p exchanged in the panel's earlier columns (their L
    // entries) and right of column k (prow keeps the pivot row); multipliers
    // from column k as the exchange leaves it (column k is written in (2))
    for (int j = ps + tid; j <= r; j += 1024) {
      if (j == k) continue;
      const double pr = Am[p + j * r];
      if (j > k) prow[j] = pr;
      if (p != k) {
        Am[p + j * r] = Am[k + j * r];
        Am[k + j * r] = pr;
      }
    }
    for (int i = k + 1 + tid; i < r; i += 1024) {
      const double a = i == p ? Am[k + k * r] : Am[i + k * r];
      lcol[i] = d != 0.0 ? a / d : a;
    }
    __syncthreads();
    if (tid == 0) {
      Am[k + k * r] = d;
      pv[k] = p;
    }
    // (2) L's column k stored; rank-1 update of rows > k, columns > k
    for (int i = k + 1 + tid; i < r; i += 1024) Am[i + k * r] = lcol[i];
    const int j0 = w + 32 * ((k + 1 - w + 31) >> 5);  // first column of this warp > k
    const int i0 = lane + 32 * ((k + 1 - lane + 31) >> 5);
    for (int j = j0; j <= r; j += 32) {
      const double u = prow[j];
      for (int i = i0; i < r; i += 32) Am[i + j * r] -= lcol[i] * u;
    }
    if (k + 1 < r && w == ((k + 1) & 31)) {
      __syncwarp();
      argmax_col(k + 1);
    }
    __syncthreads();
  }
  double* out = Mout + static_cast<size_t>(jb) * r * (r + 1);
  for (int e = tid; e < r * (r + 1); e += 1024) out[e] = Am[e];
}

// For one 64-column tile of the trailing columns (k0+jb .. r, the last one
// the augmented rhs): the panel's row swaps, U12 = L11^-1 A12, then
// A22 -= L21 U12 row tile by row tile.  grid (column tiles, systems).
constexpr int kTrailSmem = (3 * kNbMax * (BN + 8) + kNbMax * (kNbMax + 1)) * static_cast<int>(sizeof(double));
__global__ void __launch_bounds__(256, 2) lu_trail(int r, int k0, int jb, double* __restrict__ M,
                                                const int* __restrict__ perm) {
  // dynamic shared memory (kTrailSmem): U12 [32][72], two L21 buffers
  // [32][72] (the permutation staging at the start reuses them), L11
  // [32][33].  Row stride 72 (= 8 mod 16 doubles): the 4 k-rows x 8 lanes of
  // a DMMA fragment load land in distinct banks.
  extern __shared__ double trail_sm[];
  double* shbuf = trail_sm + kNbMax * (BN + 8);  // = the L21 buffers
  double* lsbuf = shbuf;
  double (*L11)[kNbMax + 1] = reinterpret_cast<double (*)[kNbMax + 1]>(trail_sm + 3 * kNbMax * (BN + 8));
  double (*Us)[BN + 8] = reinterpret_cast<double (*)[BN + 8]>(trail_sm);
  double* A = M + static_cast<size_t>(blockIdx.y) * r * (r + 1);
  const int* pm = perm + static_cast<size_t>(blockIdx.y) * kPermInts;
  const int col0 = k0 + jb + blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int cnt = pm[0];
  // the panel's swaps on this tile's columns: every source value loaded
  // (independently) before any destination is written; one thread per column
  if (tid < BN) {
    const int c = col0 + tid;
    if (c <= r) {
      double* col = A + static_cast<size_t>(c) * r;
      double* st = shbuf + tid;  // staging, stride BN + 1
      for (int k = 0; k < cnt; ++k) st[k * (BN + 1)] = col[pm[1 + 2 * kNbMax + k]];
      for (int k = 0; k < cnt; ++k) col[pm[1 + k]] = st[k * (BN + 1)];
    }
  }
  for (int e = tid; e < jb * jb; e += 256) {
    const int i = e % jb, l = e / jb;
    L11[i][l] = A[k0 + i + static_cast<size_t>(k0 + l) * r];
  }
  __syncthreads();
  // U12 tile: forward substitution with unit-lower L11, one thread per
  // column, its jb values loaded up front
  if (tid < BN) {
    const int c = col0 + tid;
    double* col = A + static_cast<size_t>(c) * r;
    for (int i = 0; i < jb; ++i) Us[i][tid] = c <= r ? col[k0 + i] : 0.0;
    for (int i = 0; i < jb; ++i) {
      double s = Us[i][tid];
      for (int l = 0; l < i; ++l) s -= L11[i][l] * Us[l][tid];
      Us[i][tid] = s;
    }
    if (c <= r)
      for (int i = 0; i < jb; ++i) col[k0 + i] = Us[i][tid];
    for (int i = jb; i < kNbMax; ++i) Us[i][tid] = 0.0;
  }
  __syncthreads();
  // A22 -= L21 U12 on DMMA: 8 warps as 2 x 4, 32 x 16 of the 64 x 64 tile each.
  // Software-pipelined over the row tiles: the next tile's L21 block streams
  // into the other shared buffer (cp.async, 8-byte pieces: columns of an odd
  // r are only 8-byte aligned) and this tile's 16 C values per thread are
  // loaded before the tensor work, so neither latency sits on the chain.
  const int lane = tid & 31, warp = tid >> 5, fr = lane >> 2, fc = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int ks_end = (jb + 3) & ~3;  // k past jb is zero-padded
  double (*Lb)[kNbMax][BM + 8] = reinterpret_cast<double (*)[kNbMax][BM + 8]>(lsbuf);
  auto stage_l = [&](int buf, int row0) {
    for (int e = tid; e < kNbMax * BM; e += 256) {
      const int mm = e % BM, kk = e / BM;
      const int i = row0 + mm;
      const bool v = kk < jb && i < r;
      cp_async8(&Lb[buf][kk][mm], A + (v ? i + static_cast<size_t>(k0 + kk) * r : 0), v);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int rbeg = k0 + jb;
  if (rbeg < r) stage_l(0, rbeg);
  int buf = 0;
  for (int row0 = rbeg; row0 < r; row0 += BM, buf ^= 1) {
    const bool more = row0 + BM < r;
    if (more) stage_l(buf ^ 1, row0 + BM);
    double cin[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = row0 + wm + 8 * i + fr, c = col0 + wn + 8 * j + 2 * fc + h;
          cin[i][j][h] = (row < r && c <= r) ? A[row + static_cast<size_t>(c) * r] : 0.0;
        }
    if (more)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    else
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ks = 0; ks < ks_end; ks += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Lb[buf][ks + fc][wm + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Us[ks + fc][wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = row0 + wm + 8 * i + fr, c = col0 + wn + 8 * j + 2 * fc + h;
          if (row < r && c <= r) A[row + static_cast<size_t>(c) * r] = cin[i][j][h] - acc[i][j][h];
        }
    __syncthreads();  // the buffer is refilled two tiles on
  }
}

// Back substitution with U (column oriented, as Eigen): one warp per system.
__global__ void __launch_bounds__(256) lu_backsolve_warp(int r, int m, const double* __restrict__ M,
                                                         double* __restrict__ sol, long long ldsol,
                                                         int* __restrict__ flags) {
  // Blocked by 32 from the bottom: the 32 x 32 diagonal block of U sits in
  // shared memory and is solved with the unknowns in lanes (shuffle
  // broadcasts, no global load on the dependency chain); the rows above
  // then take one GEMV with the block's 32 solved unknowns.
  extern __shared__ double xsall[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sys = blockIdx.x * (blockDim.x >> 5) + w;
  if (sys >= m) return;
  double* xs = xsall + static_cast<size_t>(w) * (r + 32 * 33);
  double* ub = xs + r;  // 32 x 33 diagonal block, ub[j * 33 + i] = U[i0 + j][i0 + i]
  const double* A = M + static_cast<size_t>(sys) * r * (r + 1);
  for (int i = lane; i < r; i += 32) xs[i] = A[i + static_cast<size_t>(r) * r];
  for (int i0 = ((r - 1) / 32) * 32; i0 >= 0; i0 -= 32) {
    const int bs = min(32, r - i0);
    __syncwarp();
    for (int e = lane; e < bs * bs; e += 32) {
      const int j = e % bs, i = e / bs;  // row j, column i of the block
      ub[j * 33 + i] = A[i0 + j + static_cast<size_t>(i0 + i) * r];
    }
    __syncwarp();
    double x = lane < bs ? xs[i0 + lane] : 0.0;
    for (int i = bs - 1; i >= 0; --i) {
      const double xi = __shfl_sync(0xffffffffu, x, i) / ub[i * 33 + i];
      if (lane == i) x = xi;
      if (lane < i) x -= xi * ub[lane * 33 + i];
    }
    if (lane < bs) xs[i0 + lane] = x;
    __syncwarp();
    // rows above: xs[row] -= sum_l U[row][i0 + l] x_l; the 32 loads of a row
    // are issued together (a dependent load per l left the loop latency-bound)
    const double* xb = xs + i0;
    for (int row = lane; row < i0; row += 32) {
      const double* ar = A + row + static_cast<size_t>(i0) * r;
      double acc = 0.0;
      if (bs == 32) {
        double v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = ar[static_cast<size_t>(l) * r];
#pragma unroll
        for (int l = 0; l < 32; ++l) acc += v[l] * xb[l];
      } else {
        for (int l = 0; l < bs; ++l) acc += ar[static_cast<size_t>(l) * r] * xb[l];
      }
      xs[row] -= acc;
    }
  }
  __syncwarp();
  int bad = 0;
  for (int i = lane; i < r; i += 32) {
    sol[i + static_cast<long long>(sys) * ldsol] = xs[i];
    if (!isfinite(xs[i])) bad = 1;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) flags[sys] = bad;
}

// The same back substitution with one CTA per system: warp 0 solves each
// 32 x 32 diagonal block from shared memory, then all 8 warps share the
// update of the rows above (one row per thread, the 32 loads of a row issued
// together).  Per element the same operations in the same order as
// lu_backsolve_warp, so the solutions are bitwise identical; a few systems
// (the q greedy candidates) no longer leave the GPU with one warp each.
// (the body: A the factored r x (r + 1) system, xs the right-hand side in
// shared memory -- loaded from column r when load_rhs -- and the solution on
// return; ub 2 x 32 x 33 + 64 doubles of scratch; every thread of the CTA)
__device__ void lu_backsolve_cta_body(int r, const double* __restrict__ A, double* xs, double* ub, bool load_rhs) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (load_rhs)
    for (int i = tid; i < r; i += blockDim.x) xs[i] = A[i + static_cast<size_t>(r) * r];
  if (r > 64) {
    // Look-ahead form for long solves: warp 0 updates the next diagonal
    // block's 32 rows first and solves that block (reciprocal pivots, formed
    // off the chain) while warps 1-7 update the rows above it; the next
    // diagonal block is staged by warps 1-7 too.  One barrier per block.
    double* ub2 = ub + 32 * 33;  // double buffer of the diagonal block
    double* rinv = ub2 + 32 * 33;  // 2 x 32 reciprocal pivots
    const int nb = (r + 31) / 32;
    auto stage = [&](int b, int t0, int nt) {  // diagonal block b and its reciprocals
      const int i0 = b * 32, bs = min(32, r - i0);
      double* u = (b & 1) ? ub2 : ub;
      for (int e = t0; e < bs * bs; e += nt) {
        const int j = e % bs, i = e / bs;
        u[j * 33 + i] = A[i0 + j + static_cast<size_t>(i0 + i) * r];
      }
      for (int i = t0; i < bs; i += nt) rinv[(b & 1) * 32 + i] = 1.0 / A[i0 + i + static_cast<size_t>(i0 + i) * r];
    };
    auto solve_diag = [&](int b) {  // warp 0
      const int i0 = b * 32, bs = min(32, r - i0);
      const double* u = (b & 1) ? ub2 : ub;
      const double ri = lane < bs ? rinv[(b & 1) * 32 + lane] : 0.0;
      double x = lane < bs ? xs[i0 + lane] : 0.0;
      for (int i = bs - 1; i >= 0; --i) {
        const double xi = __shfl_sync(0xffffffffu, x * ri, i);
        if (lane == i) x = xi;
        if (lane < i) x -= xi * u[lane * 33 + i];
      }
      if (lane < bs) xs[i0 + lane] = x;
    };
    auto update_rows = [&](int row_beg, int row_end, int b, int t0, int nt) {  // rows -= U[rows][block b] x_b
      const int i0 = b * 32, bs = min(32, r - i0);
      const double* xb = xs + i0;
      for (int row = row_beg + t0; row < row_end; row += nt) {
        const double* ar = A + row + static_cast<size_t>(i0) * r;
        double acc = 0.0;
        if (bs == 32) {
          double v[32];
#pragma unroll
          for (int l = 0; l < 32; ++l) v[l] = ar[static_cast<size_t>(l) * r];
#pragma unroll
          for (int l = 0; l < 32; ++l) acc += v[l] * xb[l];
        } else {
          for (int l = 0; l < bs; ++l) acc += ar[static_cast<size_t>(l) * r] * xb[l];
        }
        xs[row] -= acc;
      }
    };
    stage(nb - 1, tid, blockDim.x);
    __syncthreads();
    if (warp == 0) solve_diag(nb - 1);
    __syncthreads();
    for (int b = nb - 1; b > 0; --b) {
      const int i0 = b * 32, n0 = i0 - 32;  // block b - 1 holds rows n0 .. i0 - 1
      if (warp == 0) {
        __syncwarp();
        update_rows(n0, i0, b, lane, 32);
        __syncwarp();
      } else {
        stage(b - 1, tid - 32, blockDim.x - 32);
        update_rows(0, n0, b, tid - 32, blockDim.x - 32);
      }
      __syncthreads();  // block b - 1 staged, its rows and the rows above updated with x_b
      if (warp == 0) solve_diag(b - 1);
      __syncthreads();
    }
  } else
  for (int i0 = ((r - 1) / 32) * 32; i0 >= 0; i0 -= 32) {
    const int bs = min(32, r - i0);
    __syncthreads();
    for (int e = tid; e < bs * bs; e += blockDim.x) {
      const int j = e % bs, i = e / bs;  // row j, column i of the block
      ub[j * 33 + i] = A[i0 + j + static_cast<size_t>(i0 + i) * r];
    }
    __syncthreads();
    if (warp == 0) {
      double x = lane < bs ? xs[i0 + lane] : 0.0;
      for (int i = bs - 1; i >= 0; --i) {
        const double xi = __shfl_sync(0xffffffffu, x, i) / ub[i * 33 + i];
        if (lane == i) x = xi;
        if (lane < i) x -= xi * ub[lane * 33 + i];
      }
      if (lane < bs) xs[i0 + lane] = x;
    }
    __syncthreads();
    const double* xb = xs + i0;
    for (int row = tid; row < i0; row += blockDim.x) {
      const double* ar = A + row + static_cast<size_t>(i0) * r;
      double acc = 0.0;
      if (bs == 32) {
        double v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = ar[static_cast<size_t>(l) * r];
#pragma unroll
        for (int l = 0; l < 32; ++l) acc += v[l] * xb[l];
      } else {
        for (int l = 0; l < bs; ++l) acc += ar[static_cast<size_t>(l) * r] * xb[l];
      }
      xs[row] -= acc;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) lu_backsolve_cta(int r, const double* __restrict__ M,
                                                        double* __restrict__ sol, long long ldsol,
                                                        int* __restrict__ flags) {
  extern __shared__ double xs[];
  double* ub = xs + r;  // 32 x 33 diagonal block, ub[j * 33 + i] = U[i0 + j][i0 + i]
  const int tid = threadIdx.x;
  const int sys = blockIdx.x;
  lu_backsolve_cta_body(r, M + static_cast<size_t>(sys) * r * (r + 1), xs, ub, true);
  int bad = 0;
  for (int i = tid; i < r; i += blockDim.x) {
    sol[i + static_cast<long long>(sys) * ldsol] = xs[i];
    if (!isfinite(xs[i])) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) flags[sys] = bad;
}

// ---------------------------------------------------------------------------
// Bordered finish of a prefactored Galerkin system.  The greedy candidates of
// an inner iteration are known before that iteration's sweep (the pool and
// the RNG state are), and the basis of the previous iteration is the leading
// block of this one's, so P A00 = L U (r0 x r0, with y0 = L^-1 P b0 in column
// r0) is factored on a second stream while the sweep, the CGS and the
// projection update run.  With the k <= kBorderMax new basis columns in:
//   [A00 A01] [x0]   [b0]      U01 = L^-1 P A01,  L10 = A10 U^-1,
//   [A10 A11] [x1] = [b1]      S = A11 - L10 U01, x1 = S^-1 (b1 - L10 y0),
//                              x0 = U^-1 (y0 - U01 x1).
// One CTA of 512 threads per system: threads 0-255 replay the panels on the
// new columns (the panel's row swaps, the unit-lower 32 x 32 solve in a
// warp's lanes, the rows below; two named barriers per panel) while threads
// 256-511 solve the new rows against U (right-looking over 32-column
// blocks); then the k x k Schur system (partial pivoting) and the blocked
// back substitution of lu_backsolve_cta.  The factorisation pivots within
// the leading block first (the reference pivots over the whole column): the
// reduced operators' symmetric part is positive definite (Sigma_t > 0 plus
// the upwind flux terms), so the leading block is as well conditioned as the
// whole, and the solutions agree to rounding (tests/test_gpu_lr.py).
constexpr int kBorderMax = 16;  // widest border (the template's KB is 8 or 16)
template <int KB>
constexpr int border_scratch() {
  return 2 * 32 * 33 + 64 + 16 * KB * (KB + 1) + KB * (KB + 1) + KB;
}
size_t border_smem_bytes(int r0, int kb) {
  const int scratch = kb <= 8 ? border_scratch<8>() : border_scratch<16>();
  const int w = kb <= 8 ? 8 : 16;
  return (static_cast<size_t>(r0) * (2 * w + 1) + scratch) * sizeof(double);
}
__device__ __forceinline__ void bar_group(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }

// KB: the border's column capacity (8: the greedy candidates, one inner
// iteration ahead; 16: build_full_coefficients' systems reused over two
// iterations).  sysidx (optional): CTA b finishes stored system sysidx[b]
// (its angle angles[sysidx[b]]) into solution column b.
template <int KB>
__global__ void __launch_bounds__(512, 1) galerkin_border_kernel(int r0, int k, const int* __restrict__ angles,
                                                                 const int* __restrict__ sysidx,
                                                                 const double* __restrict__ dirs,
                                                                 const double* __restrict__ proj, long long ldp,
                                                                 long long pstride, const double* __restrict__ prhs,
                                                                 const double* __restrict__ Fall,
                                                                 const int* __restrict__ pivall,
                                                                 double* __restrict__ sol, long long ldsol,
                                                                 int* __restrict__ flags) {
  constexpr int NP = KB * (KB + 1);  // entries of [S | y1]
  constexpr int NQ = (NP + 31) / 32;
  extern __shared__ __align__(16) double bsm[];
  double* Vt = bsm;                                   // r0 x KB: A01 -> U01 (row i: its KB columns)
  double* Wt = Vt + static_cast<size_t>(r0) * KB;     // r0 x KB: A10^T -> L10^T
  double* ys = Wt + static_cast<size_t>(r0) * KB;     // y0 -> y0 - U01 x1 -> x0
  double* ub = ys + r0;                               // back substitution scratch
  double* red = ub + 2 * 32 * 33 + 64;                // 16 x NP partial sums
  double* Ss = red + 16 * NP;                         // KB x (KB + 1): [S | y1]
  double* x1 = Ss + NP;
  const int tid = threadIdx.x, lane = tid & 31;
  const int sys = sysidx ? sysidx[blockIdx.x] : blockIdx.x;
  const double* F = Fall + static_cast<size_t>(sys) * r0 * (r0 + 1);
  const int* pv = pivall + static_cast<size_t>(sys) * r0;
  const int ang = angles[sys];
  const double omx = dirs[3 * ang], omy = dirs[3 * ang + 1];
  const double* px = proj + (omx >= 0.0 ? 0 : 1) * pstride;
  const double* py = proj + (omy >= 0.0 ? 2 : 3) * pstride;
  const double* pt = proj + 4 * pstride;
  auto a_at = [&](int i, int j) {  // reduced_streaming (low_rank.cpp:176-183)
    const long long e = i + j * ldp;
    return omx * px[e] + omy * py[e] + pt[e];
  };
  {  // The factors were written an iteration ago and the tall products since
     // have swept them out of L2: one prefetch per 128-byte line up front, so
     // the solves' dependent loads hit L2 (measured: 219 -> 213 us per call
     // at C4; the kernel is bound by its ~19 dependent block steps).
    const char* fb = reinterpret_cast<const char*>(F);
    const size_t bytes = static_cast<size_t>(r0) * (r0 + 1) * sizeof(double);
    for (size_t o = static_cast<size_t>(tid) * 128; o < bytes; o += 512 * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(fb + o));
  }
  if (tid < 256) {
    const int gt = tid, gw = gt >> 5;
    for (int t = 0; t < KB; ++t)
      for (int i = gt; i < r0; i += 256) Vt[i * KB + t] = t < k ? a_at(i, r0 + t) : 0.0;
    for (int i = gt; i < r0; i += 256) ys[i] = F[i + static_cast<size_t>(r0) * r0];
    bar_group(1);
    for (int k0 = 0; k0 < r0;) {
      const int jb = lu_panel_width(r0, k0);
      for (int t = gw; t < k; t += 8) {  // a warp: column t through the panel's swaps and its unit-lower block
        const int pvl = lane < jb ? pv[k0 + lane] : 0;
        double v = lane < jb ? Vt[(k0 + lane) * KB + t] : 0.0;
        double Lr[32];
#pragma unroll
        for (int l = 0; l < 32; ++l)
          Lr[l] = (lane < jb && l < lane) ? F[k0 + lane + static_cast<size_t>(k0 + l) * r0] : 0.0;
        for (int j = 0; j < jb; ++j) {
          const int b = __shfl_sync(0xffffffffu, pvl, j);
          if (b == k0 + j) continue;
          const double vj = __shfl_sync(0xffffffffu, v, j);
          if (b < k0 + jb) {
            const double vb = __shfl_sync(0xffffffffu, v, b - k0);
            if (lane == j) v = vb;
            if (lane == b - k0) v = vj;
          } else {
            if (lane == j) {
              v = Vt[b * KB + t];
              Vt[b * KB + t] = vj;
            }
            __syncwarp();
          }
        }
#pragma unroll
        for (int l = 0; l < 31; ++l) {
          const double vl = __shfl_sync(0xffffffffu, v, l);
          if (lane > l) v -= Lr[l] * vl;
        }
        if (lane < jb) Vt[(k0 + lane) * KB + t] = v;
      }
      bar_group(1);
      for (int i = k0 + jb + gt; i < r0; i += 256) {
        const double* Li = F + i + static_cast<size_t>(k0) * r0;
#pragma unroll
        for (int hb = 0; hb < KB; hb += 8) {  // 8 columns at a time (registers)
          if (hb >= k) break;
          double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
          for (int l = 0; l < jb; ++l) {
            const double lv = Li[static_cast<size_t>(l) * r0];
            const double2* vr = reinterpret_cast<const double2*>(Vt + (k0 + l) * KB + hb);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double2 vv = vr[q];
              acc[2 * q] += lv * vv.x;
              acc[2 * q + 1] += lv * vv.y;
            }
          }
          double2* vo = reinterpret_cast<double2*>(Vt + i * KB + hb);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double2 vv = vo[q];
            vv.x -= acc[2 * q];
            vv.y -= acc[2 * q + 1];
            vo[q] = vv;
          }
        }
      }
      bar_group(1);
      k0 += jb;
    }
  } else {
    const int gt = tid - 256, gw = gt >> 5;
    for (int j = gt; j < r0; j += 256)
#pragma unroll
      for (int u = 0; u < KB; ++u) Wt[j * KB + u] = u < k ? a_at(r0 + u, j) : 0.0;
    bar_group(2);
    for (int c0 = 0; c0 < r0; c0 += 32) {
      const int bs = min(32, r0 - c0);
      for (int u = gw; u < k; u += 8) {  // a warp: new row u against the upper 32 x 32 diagonal block
        double sv = lane < bs ? Wt[(c0 + lane) * KB + u] : 0.0;
        const double rinv = lane < bs ? 1.0 / F[c0 + lane + static_cast<size_t>(c0 + lane) * r0] : 1.0;
        double Uc[32];  // U[c0 + i][c0 + lane], i < lane
#pragma unroll
        for (int i = 0; i < 32; ++i)
          Uc[i] = (lane < bs && i < lane) ? F[c0 + i + static_cast<size_t>(c0 + lane) * r0] : 0.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const double xi = __shfl_sync(0xffffffffu, sv * rinv, i);
          if (lane == i) sv = xi;
          if (lane > i) sv -= xi * Uc[i];
        }
        if (lane < bs) Wt[(c0 + lane) * KB + u] = sv;
      }
      bar_group(2);
      for (int j = c0 + bs + gt; j < r0; j += 256) {
        const double* Uj = F + c0 + static_cast<size_t>(j) * r0;
#pragma unroll
        for (int hb = 0; hb < KB; hb += 8) {
          if (hb >= k) break;
          double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
          for (int i = 0; i < bs; ++i) {
            const double uv = Uj[i];
            const double2* wr = reinterpret_cast<const double2*>(Wt + (c0 + i) * KB + hb);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double2 ww = wr[q];
              acc[2 * q] += uv * ww.x;
              acc[2 * q + 1] += uv * ww.y;
            }
          }
          double2* wo = reinterpret_cast<double2*>(Wt + j * KB + hb);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double2 ww = wo[q];
            ww.x -= acc[2 * q];
            ww.y -= acc[2 * q + 1];
            wo[q] = ww;
          }
        }
      }
      bar_group(2);
    }
  }
  __syncthreads();
  {  // [L10 U01 | L10 y0]: warp w sums rows w, w + 16, ...; a lane holds pairs lane, lane + 32, ...
    const int w = tid >> 5;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    for (int i = w; i < r0; i += 16) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int pr = lane + 32 * q;
        if (pr < NP) {
          const int u = pr / (KB + 1), t = pr - (KB + 1) * u;
          acc[q] += Wt[i * KB + u] * (t < KB ? Vt[i * KB + t] : ys[i]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (lane + 32 * q < NP) red[w * NP + lane + 32 * q] = acc[q];
  }
  __syncthreads();
  if (tid < NP) {
    double sum = 0.0;
    for (int w = 0; w < 16; ++w) sum += red[w * NP + tid];
    const int u = tid / (KB + 1), t = tid - (KB + 1) * u;
    double base;  // identity padding past k
    if (u < k && t < k)
      base = a_at(r0 + u, r0 + t);
    else if (u < k && t == KB)
      base = prhs[r0 + u];
    else
      base = (t == u) ? 1.0 : 0.0;
    Ss[tid] = base - sum;
  }
  __syncthreads();
  if (tid < 32) {  // KB x KB partial-pivot elimination of [S | y1]: lane = row
    constexpr int LD = KB + 1;
    for (int c = 0; c < KB; ++c) {
      double av = (lane >= c && lane < KB) ? fabs(Ss[lane * LD + c]) : -1.0;
      int ai = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, av, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ai, o);
        if (ov > av || (ov == av && oi < ai)) {
          av = ov;
          ai = oi;
        }
      }
      const int p = ai;  // first row of largest magnitude
      if (p != c && lane <= KB) {  // lane = column: swap rows c and p
        const double tmp = Ss[c * LD + lane];
        Ss[c * LD + lane] = Ss[p * LD + lane];
        Ss[p * LD + lane] = tmp;
      }
      __syncwarp();
      if (lane > c && lane < KB) {
        const double mlt = Ss[lane * LD + c] / Ss[c * LD + c];
        for (int j = c + 1; j <= KB; ++j) Ss[lane * LD + j] -= mlt * Ss[c * LD + j];
      }
      __syncwarp();
    }
    if (lane == 0)
      for (int i = KB - 1; i >= 0; --i) {
        double x = Ss[i * LD + KB];
        for (int j = i + 1; j < KB; ++j) x -= Ss[i * LD + j] * x1[j];
        x1[i] = x / Ss[i * LD + i];
      }
  }
  __syncthreads();
  for (int i = tid; i < r0; i += 512) {
    double z = ys[i];
#pragma unroll
    for (int t = 0; t < KB; ++t) z -= Vt[i * KB + t] * x1[t];
    ys[i] = z;
  }
  __syncthreads();
  lu_backsolve_cta_body(r0, F, ys, ub, false);
  int bad = 0;
  const long long col = static_cast<long long>(blockIdx.x) * ldsol;
  for (int i = tid; i < r0; i += 512) {
    sol[i + col] = ys[i];
    if (!isfinite(ys[i])) bad = 1;
  }
  if (tid < k) {
    sol[r0 + tid + col] = x1[tid];
    if (!isfinite(x1[tid])) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) flags[blockIdx.x] = bad;
}

// R of a Householder QR (Eigen's makeHouseholder conventions, as hh_make)
// in one cooperative launch, for the truncation SVD's W = C^T (N_Omega x r)
// whose Q is not needed: column k's reflector is applied to every column
// right of it by one warp per column (its own dot product, no cross-CTA
// reduction); every warp derives beta / tau from its own identical
// reduction of the column, so a step needs one grid-wide barrier.  Column
// k is only read during step k, so nothing is written back to it; R (n x n,
// upper) goes straight to r.
__global__ void __launch_bounds__(256) qr_r_coop(long long m, int n, double* __restrict__ a, long long lda,
                                                 double* __restrict__ r) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  const int kmax = static_cast<int>(min(static_cast<long long>(n), m));
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n * n; i += gridDim.x * blockDim.x) r[i] = 0.0;
  grid.sync();
  for (int k = 0; k < kmax; ++k) {
    const double* x = a + static_cast<long long>(k) * lda;
    double sq = 0.0;
    for (long long i = k + 1 + lane; i < m; i += 32) sq += x[i] * x[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const double c0 = x[k];
    double beta, tau, denom;
    if (sq <= 2.2250738585072014e-308) {
      tau = 0.0;
      beta = c0;
      denom = 0.0;
    } else {
      beta = sqrt(c0 * c0 + sq);
      if (c0 >= 0.0) beta = -beta;
      denom = c0 - beta;
      tau = (beta - c0) / beta;
    }
    if (gw == 0 && lane == 0) r[k + static_cast<long long>(k) * n] = beta;
    for (int j = k + 1 + gw; j < n; j += nw) {
      double* col = a + static_cast<long long>(j) * lda;
      double d = 0.0;
      for (long long i = k + 1 + lane; i < m; i += 32) d += (denom == 0.0 ? 0.0 : x[i] / denom) * col[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const double w = tau * (col[k] + d);
      for (long long i = k + 1 + lane; i < m; i += 32) col[i] -= w * (denom == 0.0 ? 0.0 : x[i] / denom);
      if (lane == 0) {
        col[k] -= w;
        r[k + static_cast<long long>(j) * n] = col[k];
      }
    }
    grid.sync();
  }
}

}  // namespace

size_t gemm_tn_work(int M, int N, long long K) {
  const long long sp = N >= 4 && N <= kNtMaxN && static_cast<double>(M) * N * K >= 1e9
                           ? std::max<long long>(nt_splits(M, K), tn_splits(M, N, K))
                                              : tn_splits(M, N, K);
  return static_cast<size_t>(sp) * M * N;
}

void gemm_tn(int M, int N, long long K, const double* A, long long lda, const double* B, long long ldb, double* C,
             long long ldc, double* work, size_t work_doubles, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  // The split count (hence the summation order) is a function of the shape
  // alone, never of the work buffer's capacity: results are reproducible
  // whatever buffers earlier calls left behind.
  int splits = tn_splits(M, N, K);
  if (static_cast<size_t>(splits) * M * N > work_doubles)
    throw std::invalid_argument("gemm_tn: work buffer smaller than gemm_tn_work(M, N, K)");
  long long kchunk = (K + splits - 1) / splits;
  kchunk = ((kchunk + 31) / 32) * 32;
  splits = static_cast<int>((K + kchunk - 1) / kchunk);
  if (splits < 1) splits = 1;
  const bool pipe_ok = aligned16(A) && aligned16(B) && lda % 2 == 0 && ldb % 2 == 0 && K % 2 == 0 &&
                       kchunk % kTnBk == 0;
  if (N <= kSkinny && !pipe_ok) {
    double* o = splits == 1 ? C : work;
    const long long ldo = splits == 1 ? ldc : M, sstride = splits == 1 ? 0 : static_cast<long long>(M) * N;
    if (aligned16(A) && aligned16(B) && lda % 2 == 0 && ldb % 2 == 0) {
      auto go = [&](auto kern, int mw) {
        kern<<<dim3((M + 8 * mw - 1) / (8 * mw), splits), 256, 0, s>>>(M, N, K, kchunk, A, lda, B, ldb, o, ldo,
                                                                       sstride);
      };
      if (N == 1) go(gemm_tn_skinny2<1, 4>, 4);
      else if (N == 2) go(gemm_tn_skinny2<2, 4>, 4);
      else if (N <= 4) go(gemm_tn_skinny2<4, 4>, 4);
      else if (N <= 8) go(gemm_tn_skinny2<8, 4>, 4);
      else go(gemm_tn_skinny2<16, 2>, 2);
    } else {
      gemm_tn_skinny_kernel<<<dim3((M + BM - 1) / BM, splits), 256, 0, s>>>(M, N, K, kchunk, A, lda, B, ldb, o, ldo,
                                                                           sstride);
    }
    if (splits > 1) launch_splitk_reduce(M, N, splits, work, C, ldc, s);
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  static const bool nt_off = [] {  // RTLR_TN_NT=0: the 64 x 64 tile kernel for these shapes too (A/B timing)
    const char* e = std::getenv("RTLR_TN_NT");
    return e && e[0] == '0';
  }();
  // (small products, e.g. C2's 178 x 20 x 65536, stay on the 64 x 64 tiles: 46 vs 54 us)
  if (pipe_ok && N >= 4 && N <= kNtMaxN && !nt_off && static_cast<double>(M) * N * K >= 1e9) {
    // (own split count: 128-row tiles, ~4 CTAs per SM; still a function of the shape only)
    const long long tiles = (M + kNtBm - 1) / kNtBm;
    long long sp = nt_splits(M, K);
    long long kc = ((K + sp - 1) / sp + kTnBk - 1) / kTnBk * kTnBk;
    sp = (K + kc - 1) / kc;
    if (static_cast<size_t>(sp) * M * N > work_doubles && sp > 1)
      throw std::invalid_argument("gemm_tn: work buffer smaller than gemm_tn_work(M, N, K)");
    double* o2 = sp == 1 ? C : work;
    const long long ldo2 = sp == 1 ? ldc : M, ss2 = sp == 1 ? 0 : static_cast<long long>(M) * N;
    const int nt = (N + 7) / 8;
    const int smem = kNtStages * (kNtBm + 8 * nt) * kTnLd * static_cast<int>(sizeof(double));
    auto go = [&](auto kern) {
      RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(sp)), 256, smem, s>>>(M, N, K, kc, A, lda, B,
                                                                                          ldb, o2, ldo2, ss2);
    };
    switch (nt) {
      case 1: go(gemm_tn_dmma_nt<1>); break;
      case 2: go(gemm_tn_dmma_nt<2>); break;
      case 3: go(gemm_tn_dmma_nt<3>); break;
      case 4: go(gemm_tn_dmma_nt<4>); break;
      case 5: go(gemm_tn_dmma_nt<5>); break;
      default: go(gemm_tn_dmma_nt<6>); break;
    }
    if (sp > 1) launch_splitk_reduce(M, N, static_cast<int>(sp), work, C, ldc, s);
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, splits);
  double* o = splits == 1 ? C : work;
  const long long ldo = splits == 1 ? ldc : M, sstride = splits == 1 ? 0 : static_cast<long long>(M) * N;
  if (pipe_ok && N <= 8) {
    const int smem = kSkStages * (64 + 8) * kTnLd * static_cast<int>(sizeof(double));
    RTLR_CUDA(cudaFuncSetAttribute(gemm_tn_skinny_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gemm_tn_skinny_pipe<<<dim3((M + 63) / 64, splits), 256, smem, s>>>(M, N, K, kchunk, A, lda, B, ldb, o, ldo,
                                                                       sstride);
  } else if (pipe_ok) {
    const int smem = 2 * (BM + BN) * kTnLd * static_cast<int>(sizeof(double));
    RTLR_CUDA(cudaFuncSetAttribute(gemm_tn_dmma_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gemm_tn_dmma_pipe<<<grid, 256, smem, s>>>(M, N, K, kchunk, A, lda, B, ldb, o, ldo, sstride);
  } else {
    gemm_dmma_kernel<true><<<grid, 256, 0, s>>>(M, N, K, kchunk, A, lda, B, ldb, o, ldo, sstride, false);
  }
  if (splits > 1) launch_splitk_reduce(M, N, splits, work, C, ldc, s);
  RTLR_CUDA(cudaGetLastError());
}

void gemm_nn(long long M, int N, int K, const double* A, long long lda, const double* B, long long ldb, double* C,
             long long ldc, cudaStream_t s, bool subtract) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    if (!subtract)
      for (int j = 0; j < N; ++j) RTLR_CUDA(cudaMemsetAsync(C + j * ldc, 0, M * sizeof(double), s));
    return;
  }
  // (a single k-stage, K <= 32 — the QR trailing updates — gains nothing from the pipeline)
  const bool pipe_ok = aligned16(A) && lda % 2 == 0 && M % 2 == 0 && K >= 8;
  static const bool nt_off = [] {  // RTLR_NN_NT=0: the 64 x 64 tile / FFMA skinny kernels (A/B timing)
    const char* e = std::getenv("RTLR_NN_NT");
    return e && e[0] == '0';
  }();
  // (4 <= N <= 8, e.g. C2's p = 4 CGS updates: the FFMA skinny kernel's 512-row CTAs left the
  // GPU under-filled at N_x = 65536: 65 -> 25 us at r = 220, C2 LR ~3% faster)
  static const int nt_min_n = [] {  // RTLR_NN_NT_MIN=n: narrowest N on the DMMA tiles (A/B timing)
    const char* e = std::getenv("RTLR_NN_NT_MIN");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 4;
  }();
  if ((N <= 8 && !(pipe_ok && !nt_off && N >= nt_min_n)) || (N <= kSkinny && !pipe_ok)) {
    if (aligned16(A) && lda % 2 == 0) {
      const unsigned grid = static_cast<unsigned>((M + 511) / 512);
      if (N == 1) gemm_nn_skinny2<1><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, subtract);
      else if (N == 2) gemm_nn_skinny2<2><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, subtract);
      else if (N <= 4) gemm_nn_skinny2<4><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, subtract);
      else if (N <= 8) gemm_nn_skinny2<8><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, subtract);
      else gemm_nn_skinny2<16><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, subtract);
    } else {
      gemm_nn_skinny_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc,
                                                                                    subtract);
    }
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  // (N <= 32, e.g. the q = 16 candidate columns: 1.27 -> 0.89 ms at 1M x 16 x 600; wider
  // products, e.g. the 128-angle verification blocks, run at ~80% of the fp64 tensor peak
  // on the 64 x 64 tiles: 5.5 vs 6.2 ms at 1M x 128 x 600)
  if (pipe_ok && !nt_off && N <= 32) {
    const int nt = std::min(4, (N + 7) / 8);  // (N = 8: the CGS block updates, 1 column tile)
    const unsigned groups = static_cast<unsigned>((N + 8 * nt - 1) / (8 * nt));
    const int smem = kNtStages * (kTnBk * kNnNtLdA + 8 * nt * kTnLd) * static_cast<int>(sizeof(double));
    auto go = [&](auto kern) {
      RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<dim3(groups, static_cast<unsigned>((M + kNtBm - 1) / kNtBm)), 256, smem, s>>>(M, N, K, A, lda, B, ldb,
                                                                                            C, ldc, subtract);
    };
    switch (nt) {
      case 1: go(gemm_nn_dmma_nt<1>); break;
      case 2: go(gemm_nn_dmma_nt<2>); break;
      case 3: go(gemm_nn_dmma_nt<3>); break;
      default: go(gemm_nn_dmma_nt<4>); break;
    }
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  dim3 grid(static_cast<unsigned>((M + BM - 1) / BM), (N + BN - 1) / BN);
  if (pipe_ok) {
    const int smem = 2 * (kTnBk * kNnLdA + BN * kTnLd) * static_cast<int>(sizeof(double));
    RTLR_CUDA(cudaFuncSetAttribute(gemm_nn_dmma_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gemm_nn_dmma_pipe<<<grid, 256, smem, s>>>(M, N, K, A, lda, B, ldb, C, ldc, subtract);
  } else {
    gemm_dmma_kernel<false><<<grid, 256, 0, s>>>(M, N, K, 0, A, lda, B, ldb, C, ldc, 0, subtract);
  }
  RTLR_CUDA(cudaGetLastError());
}

void gemv_n(long long n, int k, const double* A, long long lda, const double* x, double alpha, double* y,
            cudaStream_t s) {
  if (k <= 0) return;
  gemv_n_kernel<<<grid1d(n), 256, 0, s>>>(n, k, A, lda, x, alpha, y);
  RTLR_CUDA(cudaGetLastError());
}

void dot(long long n, const double* a, const double* b, double* work, double* out, cudaStream_t s) {
  dot_partials<<<kDotParts, 256, 0, s>>>(n, a, b, work);
  dot_finish<<<1, 256, 0, s>>>(kDotParts, work, out);
  RTLR_CUDA(cudaGetLastError());
}

void dot_indirect(long long n, const double* a, const double* B, long long ldb, const int* d_col, double* work,
                  double* out, cudaStream_t s) {
  dot_partials_ind<<<kDotParts, 256, 0, s>>>(n, a, B, ldb, d_col, work);
  dot_finish<<<1, 256, 0, s>>>(kDotParts, work, out);
  RTLR_CUDA(cudaGetLastError());
}

void scale_copy(long long n, const double* x, const double* h, double* y, cudaStream_t s) {
  scale_copy_kernel<<<grid1d(n), 256, 0, s>>>(n, x, h, y);
  RTLR_CUDA(cudaGetLastError());
}

void axpy_dev(long long n, const double* alpha, double sign, const double* x, double* y, cudaStream_t s) {
  axpy_kernel<<<grid1d(n), 256, 0, s>>>(n, alpha, sign, x, y);
  RTLR_CUDA(cudaGetLastError());
}

void stream_products(const StencilArgs& a, int p, const double* P, long long ldp, double* W, long long ldw,
                     cudaStream_t s, int c0, int c1) {
  if (p <= 0) return;
  if (c1 < 0) c1 = a.ncell;
  if (c1 <= c0) return;
  if ((ldp & 1) || (ldw & 1) || !aligned16(P) || !aligned16(W))
    throw std::invalid_argument("stream_products: P, W and their leading dimensions must be 16-byte aligned");
  stream_products_kernel<<<dim3(static_cast<unsigned>((c1 - c0 + 255) / 256), static_cast<unsigned>(p)), 256, 0, s>>>(
      a, p, P, ldp, W, ldw, c0, c1);
  RTLR_CUDA(cudaGetLastError());
}

int lu_smem_max(int m) {
  static const int small_max = [] {  // RTLR_LU_SMEM_SMALL=n: the threshold for small batches (A/B timing)
    const char* e = std::getenv("RTLR_LU_SMEM_SMALL");
    return e ? std::max(0, std::min(kSmemLuMax, std::atoi(e))) : kSmemLuMaxSmall;
  }();
  return m <= kSmemLuSmallBatch ? small_max : kSmemLuMax;
}

size_t galerkin_work_per_system(int r) {
  return static_cast<size_t>(r) * (r + 1) + r + (kPermInts + 1) / 2 + 1;
}

size_t galerkin_work_doubles(int r, int m) {
  if (r <= lu_smem_max(m)) return 0;
  return static_cast<size_t>(m) * galerkin_work_per_system(r);
}

// The blocked right-looking factorisation of m assembled r x (r + 1)
// systems in place (panel, then swaps + TRSM + DMMA update of the trailing
// columns, the right-hand side among them).
static void lu_factor_blocked(int r, int m, double* M, int* piv, int* perm, cudaStream_t s) {
  constexpr int kPanelThreads = 256;
  RTLR_CUDA(cudaFuncSetAttribute(lu_panel_smem<kPanelThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kPanelSmemBytes));
  RTLR_CUDA(cudaFuncSetAttribute(lu_trail, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrailSmem));
  static const int reg_panel = [] {  // RTLR_LU_PANEL=smem: the shared-memory panel only
    const char* e = std::getenv("RTLR_LU_PANEL");
    if (e && std::string(e) == "smem") return 0;
    const int bytes = 512 * static_cast<int>(kNbMax * sizeof(double) + sizeof(int));
    RTLR_CUDA(cudaFuncSetAttribute(lu_panel_reg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    RTLR_CUDA(cudaFuncSetAttribute(lu_panel_reg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    return 1;
  }();
  for (int k0 = 0; k0 < r;) {
    const int jb = lu_panel_width(r, k0);
    const int rows = r - k0;
    const size_t slot_bytes = static_cast<size_t>(rows) * (kNbMax * sizeof(double) + sizeof(int));
    // (small batches only: at one CTA per SM the register panel loses to
    // the shared-memory one once the batch fills the GPU; 3 rows per
    // thread spill)
    const bool small = reg_panel && m <= 64 && jb == kNbMax;
    if (small && rows <= 256)
      lu_panel_reg<1><<<m, 256, slot_bytes, s>>>(r, k0, jb, M, piv, perm);
    else if (small && rows <= 512)
      lu_panel_reg<2><<<m, 256, slot_bytes, s>>>(r, k0, jb, M, piv, perm);
    else
      lu_panel_smem<kPanelThreads><<<m, kPanelThreads, static_cast<size_t>(rows) * (jb * sizeof(double) + 4), s>>>(
          r, k0, jb, M, piv, perm);
    const int ntrail = r + 1 - (k0 + jb);
    if (ntrail > 0) lu_trail<<<dim3((ntrail + BN - 1) / BN, m), 256, kTrailSmem, s>>>(r, k0, jb, M, perm);
    k0 += jb;
  }
}

// Back substitution of m factored systems (column r: the forward-substituted
// right-hand side) into sol.
static void lu_backsolve(int r, int m, const double* M, double* sol, long long ldsol, int* flags, cudaStream_t s) {
  // One CTA per system while the systems do not fill the GPU with warps;
  // beyond that one warp per system (8 per CTA) has the parallelism.
  if (m < 8 * 148) {
    const size_t smem = (static_cast<size_t>(r) + 2 * 32 * 33 + 64) * sizeof(double);
    if (smem > 48 * 1024)
      RTLR_CUDA(cudaFuncSetAttribute(lu_backsolve_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    lu_backsolve_cta<<<m, 256, smem, s>>>(r, M, sol, ldsol, flags);
  } else {
    const int per = 8;  // systems (warps) per CTA
    const size_t smem = static_cast<size_t>(per) * (r + 32 * 33) * sizeof(double);
    if (smem > 48 * 1024)
      RTLR_CUDA(cudaFuncSetAttribute(lu_backsolve_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    lu_backsolve_warp<<<(m + per - 1) / per, 32 * per, smem, s>>>(r, m, M, sol, ldsol, flags);
  }
}

void galerkin_batch(int r, int m, const int* angles, const double* dirs, const double* proj, long long ldp,
                    long long proj_stride, const double* prhs, const double* extra, double* sol, long long ldsol,
                    int* flags, double* work, cudaStream_t s) {
  if (m <= 0 || r <= 0) return;
  static const bool cta_lu = [] {  // RTLR_GAL_CTA=0: the shared-memory / blocked kernels for small batches (A/B)
    const char* e = std::getenv("RTLR_GAL_CTA");
    return !(e && std::string(e) == "0");
  }();
  if (cta_lu && m <= kSmemLuSmallBatch && r <= kCtaLuMax) {
    const size_t smem = static_cast<size_t>(r) * (r + 1) * sizeof(double);
    static const bool attr = [] {
      RTLR_CUDA(cudaFuncSetAttribute(galerkin_cta_lu, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kCtaLuMax * (kCtaLuMax + 1) * 8));
      return true;
    }();
    (void)attr;
    galerkin_cta_lu<<<m, 1024, smem, s>>>(r, angles, dirs, proj, ldp, proj_stride, prhs, extra, sol, ldsol, flags);
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  const int smem_max = lu_smem_max(m);
  if (r > smem_max) {
    double* M = work;
    int* piv = reinterpret_cast<int*>(work + static_cast<size_t>(m) * r * (r + 1));
    int* perm = reinterpret_cast<int*>(work + static_cast<size_t>(m) * (r * static_cast<size_t>(r + 1) + r));
    lu_assemble<<<dim3(std::max(1, std::min(64, (r * (r + 1) + 255) / 256)), m), 256, 0, s>>>(
        r, angles, dirs, proj, ldp, proj_stride, prhs, extra, ldsol, M);
    lu_factor_blocked(r, m, M, piv, perm, s);
    lu_backsolve(r, m, M, sol, ldsol, flags, s);
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  const bool in_smem = r <= smem_max;
  const size_t smem = in_smem ? static_cast<size_t>(r) * r * sizeof(double) : 0;
  if (in_smem)
    RTLR_CUDA(cudaFuncSetAttribute(galerkin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemLuMax * kSmemLuMax * 8));
  galerkin_kernel<<<m, 256, smem, s>>>(r, angles, dirs, proj, ldp, proj_stride, prhs, extra, sol, ldsol, flags,
                                       work, in_smem);
  RTLR_CUDA(cudaGetLastError());
}

// Prefactor: assemble [A | prhs] at rank r for the m angles and factor it in
// place (no back substitution); work as galerkin_batch's blocked path.
void galerkin_prefactor(int r, int m, const int* angles, const double* dirs, const double* proj, long long ldp,
                        long long proj_stride, const double* prhs, double* work, cudaStream_t s,
                        cudaEvent_t assembled) {
  if (m <= 0 || r <= 0) return;
  double* M = work;
  int* piv = reinterpret_cast<int*>(work + static_cast<size_t>(m) * r * (r + 1));
  int* perm = reinterpret_cast<int*>(work + static_cast<size_t>(m) * (r * static_cast<size_t>(r + 1) + r));
  static const bool cta_factor = [] {  // RTLR_PREFACTOR_CTA=0: the blocked chain at every rank (A/B)
    const char* e = std::getenv("RTLR_PREFACTOR_CTA");
    return !(e && e[0] == '0');
  }();
  lu_assemble<<<dim3(std::max(1, std::min(64, (r * (r + 1) + 255) / 256)), m), 256, 0, s>>>(
      r, angles, dirs, proj, ldp, proj_stride, prhs, nullptr, 0, M);
  if (assembled) RTLR_CUDA(cudaEventRecord(assembled, s));  // proj and prhs are not read past this point
  if (cta_factor && m <= kSmemLuSmallBatch && r <= kCtaLuMax) {
    static const bool attr = [] {
      RTLR_CUDA(cudaFuncSetAttribute(galerkin_cta_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kCtaLuMax * (kCtaLuMax + 1) * 8));
      return true;
    }();
    (void)attr;
    galerkin_cta_factor<<<m, 1024, static_cast<size_t>(r) * (r + 1) * sizeof(double), s>>>(r, M, piv);
    RTLR_CUDA(cudaGetLastError());
    return;
  }
  lu_factor_blocked(r, m, M, piv, perm, s);
  RTLR_CUDA(cudaGetLastError());
}

// The solutions of the systems galerkin_prefactor left in work (rank r, no border).
void galerkin_factored_solve(int r, int m, const double* work, double* sol, long long ldsol, int* flags,
                             cudaStream_t s) {
  if (m <= 0 || r <= 0) return;
  lu_backsolve(r, m, work, sol, ldsol, flags, s);
  RTLR_CUDA(cudaGetLastError());
}

bool galerkin_border_fits(int r0, int k) {
  return r0 >= 1 && k >= 0 && k <= kBorderMax && border_smem_bytes(r0, k) <= 227 * 1024;
}

// The solutions at rank r0 + k from the rank-r0 factors galerkin_prefactor
// left in work (m_stored systems); with sysidx, only the m listed systems.
void galerkin_border_solve(int r0, int k, int m, const int* angles, const double* dirs, const double* proj,
                           long long ldp, long long proj_stride, const double* prhs, const double* work, double* sol,
                           long long ldsol, int* flags, cudaStream_t s, const int* sysidx, int m_stored) {
  if (m <= 0) return;
  if (!galerkin_border_fits(r0, k)) throw std::invalid_argument("galerkin_border_solve: rank or border out of range");
  static const bool attr = [] {
    RTLR_CUDA(cudaFuncSetAttribute(galerkin_border_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    RTLR_CUDA(cudaFuncSetAttribute(galerkin_border_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    return true;
  }();
  (void)attr;
  if (m_stored < 0) m_stored = m;
  const int* piv = reinterpret_cast<const int*>(work + static_cast<size_t>(m_stored) * r0 * (r0 + 1));
  if (k <= 8)
    galerkin_border_kernel<8><<<m, 512, border_smem_bytes(r0, k), s>>>(r0, k, angles, sysidx, dirs, proj, ldp,
                                                                      proj_stride, prhs, work, piv, sol, ldsol, flags);
  else
    galerkin_border_kernel<16><<<m, 512, border_smem_bytes(r0, k), s>>>(r0, k, angles, sysidx, dirs, proj, ldp,
                                                                       proj_stride, prhs, work, piv, sol, ldsol, flags);
  RTLR_CUDA(cudaGetLastError());
}

constexpr size_t kQrPart = 1024;  // >= max(kDotParts, kQrBlock * kHhChunks)
static_assert(kQrPart >= kQrBlock * kHhChunks && kQrPart >= kDotParts, "QR partials");

size_t householder_qr_work(long long m, int n) {
  constexpr int nb = kQrBlock;
  size_t gemm = 0;  // the largest split-K workspace of any trailing / Q update
  for (int c = 1; c <= n; ++c) gemm = std::max(gemm, gemm_tn_work(nb, c, m));
  return kQrPart + 8 + static_cast<size_t>(m) * nb + 2 * static_cast<size_t>(nb) * n + 2 * nb * nb + gemm;
}

// Blocked Householder QR (LAPACK dgeqrf/dorgqr structure): each panel of
// kQrBlock columns is factored column by column (Eigen's makeHouseholder
// conventions, kernels above) and the trailing columns take the panel's
// block reflector I - V T V^T through two tall GEMMs, so the trailing matrix
// is read once per panel instead of once per column.  Q is formed the same
// way, backwards.
void householder_qr(long long m, int n, double* a, long long lda, double* tau, double* q, long long ldq, double* r,
                    double* work, size_t work_doubles, cudaStream_t s) {
  constexpr int nb = kQrBlock;
  if (work_doubles < householder_qr_work(m, n))
    throw std::invalid_argument("householder_qr: work buffer smaller than householder_qr_work(m, n)");
  double* part = work;
  double* scal = work + kQrPart;
  double* V = scal + 8;
  double* W = V + static_cast<size_t>(m) * nb;
  double* G = W + 2 * static_cast<size_t>(nb) * n;
  double* T = G + nb * nb;
  double* gw = T + nb * nb;
  const size_t gw_n = work_doubles - (gw - work);
  const int kmax = static_cast<int>(std::min<long long>(n, m));
  auto form_block = [&](int k0, int jb) {  // V (rows k0..m-1) and T of panel k0
    const long long rows = m - k0;
    hh_panel_v<<<grid1d(rows * jb), 256, 0, s>>>(m, k0, jb, a, lda, V, rows);
    gemm_tn(jb, jb, rows, V, rows, V, rows, G, jb, gw, gw_n, s);
    hh_form_t<<<1, 32, 0, s>>>(jb, G, tau + k0, T);
  };
  for (int k0 = 0; k0 < kmax; k0 += nb) {
    const int jb = std::min(nb, kmax - k0);
    for (int k = k0; k < k0 + jb; ++k) {
      hh_tail<<<kDotParts, 256, 0, s>>>(m, k, a, lda, part);
      hh_make<<<1, 256, 0, s>>>(kDotParts, k, a, lda, part, tau, scal);
      hh_scale_tail<<<grid1d(m), 256, 0, s>>>(m, k, a, lda, scal);
      const int nc = k0 + jb - k - 1;  // panel columns right of k
      if (nc > 0) {
        hh_dot_chunks<<<dim3(nc, kHhChunks), 256, 0, s>>>(m, k, a, lda, a, lda, k + 1, part);
        hh_update_chunks<<<dim3(nc, kHhChunks), 256, 0, s>>>(m, k, a, lda, tau, a, lda, k + 1, part);
        hh_update_diag<<<1, 32, 0, s>>>(k, tau, a, lda, k + 1, nc, part);
      }
      set_beta<<<1, 32, 0, s>>>(k, a, lda, scal);
    }
    const int nt = n - k0 - jb;
    if (nt > 0) {  // A_trail -= V T^T (V^T A_trail)
      const long long rows = m - k0;
      form_block(k0, jb);
      double* At = a + k0 + static_cast<long long>(k0 + jb) * lda;
      gemm_tn(jb, nt, rows, V, rows, At, lda, W, jb, gw, gw_n, s);
      trmm_small<<<std::min(nt, 4096), 32, 0, s>>>(jb, nt, T, true, W);
      gemm_nn(rows, nt, jb, V, rows, W, jb, At, lda, s, /*subtract=*/true);
    }
  }
  RTLR_CUDA(cudaGetLastError());
  extract_r<<<grid1d(static_cast<long long>(n) * n), 256, 0, s>>>(n, a, lda, r);
  // Q = H_0 ... H_{n-1} I[:, :n]: blocks applied backwards, Q_blk -= V T (V^T Q_blk)
  eye_cols<<<grid1d(m * n), 256, 0, s>>>(m, n, q, ldq);
  for (int k0 = ((kmax - 1) / nb) * nb; k0 >= 0; k0 -= nb) {
    const int jb = std::min(nb, kmax - k0);
    const long long rows = m - k0;
    const int nq = n - k0;
    form_block(k0, jb);
    double* Qb = q + k0 + static_cast<long long>(k0) * ldq;
    gemm_tn(jb, nq, rows, V, rows, Qb, ldq, W, jb, gw, gw_n, s);
    trmm_small<<<std::min(nq, 4096), 32, 0, s>>>(jb, nq, T, false, W);
    gemm_nn(rows, nq, jb, V, rows, W, jb, Qb, ldq, s, /*subtract=*/true);
  }
  RTLR_CUDA(cudaGetLastError());
}

bool householder_r_coop(long long m, int n, double* a, long long lda, double* r, cudaStream_t s) {
  static const int grid = [] {  // co-resident CTAs (0: cooperative launch unsupported or disabled)
    int dev = 0, ok = 0, per = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, qr_r_coop, 256, 0);
    const char* e = std::getenv("RTLR_QR_COOP");
    return (ok && !(e && e[0] == '0')) ? std::min(per, 2) * sms : 0;
  }();
  if (grid <= 0 || n <= 0) return false;
  // one warp per column right of the current one; 8 warps per CTA
  const int g = std::max(1, std::min(grid, (n + 7) / 8));
  void* args[] = {&m, &n, &a, &lda, &r};
  RTLR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(qr_r_coop), dim3(g), dim3(256), args, 0, s));
  return true;
}

// Ri (ld n) = R^-1 for upper-triangular R (order n, ld n), recursively:
// [[A, B], [0, C]]^-1 = [[A^-1, -A^-1 B C^-1], [0, C^-1]], the off-diagonal
// block by two DMMA products through T (n x n scratch); blocks of <= 32 in
// shared memory (<= 32).  Ri's strictly lower part is zeroed by the caller.
static void tri_inv_upper_rec(int n, const double* R, long long ldr, double* Ri, long long ldi, double* T,
                              cudaStream_t s) {
  if (n <= 32) {
    tri_inv_upper_small<<<1, 32, 0, s>>>(n, R, ldr, Ri, ldi);
    return;
  }
  const int n1 = ((n / 2 + 31) / 32) * 32, n2 = n - n1;
  tri_inv_upper_rec(n1, R, ldr, Ri, ldi, T, s);
  tri_inv_upper_rec(n2, R + n1 + static_cast<long long>(n1) * ldr, ldr, Ri + n1 + static_cast<long long>(n1) * ldi,
                    ldi, T, s);
  // T = B C^-1 (n1 x n2), Ri_top_right = -(A^-1 T)
  gemm_nn(n1, n2, n2, R + static_cast<long long>(n1) * ldr, ldr, Ri + n1 + static_cast<long long>(n1) * ldi, ldi, T,
          n1, s);
  double* tr = Ri + static_cast<long long>(n1) * ldi;
  gemm_nn(n1, n2, n1, Ri, ldi, T, n1, tr, ldi, s);
  neg_kernel<<<std::max(1, std::min(1024, (n1 * n2 + 255) / 256)), 256, 0, s>>>(n1, n2, tr, ldi);
}

// Upper Cholesky G = R^T R in place (order n, ld ldg; G's lower part
// zeroed), recursively: R11 = chol(G11); R12 = R11^-T G12; R22 =
// chol(G22 - R12^T R12), with DMMA products and R11^-1 by
// tri_inv_upper_rec; blocks of <= 32 in shared memory.  ws: 3 n^2 doubles.
static void chol_upper_rec(int n, double* G, long long ldg, double* ws, int* flag, cudaStream_t s) {
  if (n <= 32) {
    chol_upper_small<<<1, 32, 0, s>>>(n, G, ldg, flag);
    return;
  }
  const int n1 = ((n / 2 + 31) / 32) * 32, n2 = n - n1;
  double* G12 = G + static_cast<long long>(n1) * ldg;
  double* G22 = G12 + n1;
  chol_upper_rec(n1, G, ldg, ws, flag, s);
  double* Ri = ws;                                       // n1 x n1
  double* T = ws + static_cast<size_t>(n1) * n1;         // n1 x n2 (then n2 x n2)
  double* Tr = T + static_cast<size_t>(n1) * std::max(n1, n2);  // scratch of tri_inv_upper_rec
  RTLR_CUDA(cudaMemsetAsync(Ri, 0, static_cast<size_t>(n1) * n1 * sizeof(double), s));
  tri_inv_upper_rec(n1, G, ldg, Ri, n1, Tr, s);
  // R12 = Ri^T G12 -> T, copied into G12
  double* gw = Tr;  // (gemm_tn with M = n1, K = n1: split count from the shape, partials in gw)
  gemm_tn(n1, n2, n1, Ri, n1, G12, ldg, T, n1, gw, static_cast<size_t>(n1) * std::max(n1, n2) * 4, s);
  const int g = std::max(1, std::min(1024, (n1 * n2 + 255) / 256));
  copy2d_kernel<<<g, 256, 0, s>>>(n1, n2, T, n1, G12, ldg, false);
  // G22 -= R12^T R12
  gemm_tn(n2, n2, n1, G12, ldg, G12, ldg, T, n2, gw, static_cast<size_t>(n1) * std::max(n1, n2) * 4, s);
  sub_inplace_kernel<<<std::max(1, std::min(1024, (n2 * n2 + 255) / 256)), 256, 0, s>>>(n2, n2, T, n2, G22, ldg);
  chol_upper_rec(n2, G22, ldg, ws, flag, s);
  // the lower-left block is zero
  RTLR_CUDA(cudaMemset2DAsync(G + n1, ldg * sizeof(double), 0, n2 * sizeof(double), n1, s));
}
size_t cholqr2_work_doubles(long long m, int n) {
  return std::max(gemm_tn_work(n, n, m), static_cast<size_t>(1)) + 12 * static_cast<size_t>(n) * n + 8;
}

// X (m x n, ld ldx) <- Q, R (n x n, ld n) with X_in = Q R, Q orthonormal:
// two rounds of G = X^T X (DMMA), G = R^T R (Cholesky), X <- X R^-1
// (DMMA), R = R2 R1.  Q buffer: m x n scratch (ld m).  For well-conditioned
// X (the low-rank basis after the block CGS: an orthonormal block plus
// orthonormalised new columns, losing orthogonality at the 1e-10 level that
// triggers the rebuild); false (and X untouched) on a non-positive pivot.
bool cholqr2_inplace(long long m, int n, double* X, long long ldx, double* R, double* Qbuf, double* work,
                     size_t work_doubles, int* d_flag, cudaStream_t s) {
  if (n < 1 || work_doubles < cholqr2_work_doubles(m, n)) return false;
  const size_t nn = static_cast<size_t>(n) * n;
  double* G = work;
  double* Ri = work + nn;
  double* R1 = work + 2 * nn;
  double* T = work + 3 * nn;
  double* cws = work + 5 * nn;  // chol_upper_rec scratch (up to ~7 n^2 with the partials)
  double* gw = work + 12 * nn + 8;
  const size_t gwn = work_doubles - (12 * nn + 8);
  RTLR_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
  auto inv = [&]() {
    RTLR_CUDA(cudaMemsetAsync(Ri, 0, nn * sizeof(double), s));
    tri_inv_upper_rec(n, G, n, Ri, n, T, s);
  };
  // round 1: X -> Qbuf
  gemm_tn(n, n, m, X, ldx, X, ldx, G, n, gw, gwn, s);
  chol_upper_rec(n, G, n, cws, d_flag, s);
  inv();
  RTLR_CUDA(cudaMemcpyAsync(R1, G, nn * sizeof(double), cudaMemcpyDeviceToDevice, s));
  gemm_nn(m, n, n, X, ldx, Ri, n, Qbuf, m, s);
  // round 2: Qbuf -> X
  gemm_tn(n, n, m, Qbuf, m, Qbuf, m, G, n, gw, gwn, s);
  chol_upper_rec(n, G, n, cws, d_flag, s);
  inv();
  int hflag = 0;
  RTLR_CUDA(cudaMemcpyAsync(&hflag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  RTLR_CUDA(cudaStreamSynchronize(s));
  if (hflag) return false;
  gemm_nn(m, n, n, Qbuf, m, Ri, n, X, ldx, s);
  gemm_nn(n, n, n, G, n, R1, n, R, n, s);  // R = R2 R1
  RTLR_CUDA(cudaGetLastError());
  return true;
}

size_t bidiag_work_doubles(long long m, int n) { return static_cast<size_t>(2 * n + 8) + static_cast<size_t>((n + 63) / 64) * m; }

bool bidiag_singular_values(long long m, int n, double* a, long long lda, double* d_sv, double* work,
                            size_t work_doubles, cudaStream_t s) {
  if (n < 1 || m < n || m > 8192 || work_doubles < bidiag_work_doubles(m, n)) return false;
  // RTLR_SVD=bidiag1: the three-barrier kernel and thread-per-value bisection (A/B)
  static const int variant = [] {
    const char* e = std::getenv("RTLR_SVD");
    return e && std::string(e) == "bidiag1" ? 1 : 2;
  }();
  const bool v2 = variant == 2 && n <= 32 * kBdRegs;
  static const int coop_per_sm[2] = {[] {
    int dev = 0, ok = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
    const char* e = std::getenv("RTLR_SVD");
    if (!ok || (e && std::string(e) == "jacobi")) return 0;
    RTLR_CUDA(cudaFuncSetAttribute(bidiag_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 8192 * 8));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bidiag_coop, 256, 2 * 8192 * 8);
    return std::min(per, 2);
  }(), [] {
    int dev = 0, ok = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
    const char* e = std::getenv("RTLR_SVD");
    if (!ok || (e && std::string(e) == "jacobi")) return 0;
    const int bytes = (8192 + 32 * kBdRegs) * 8;
    RTLR_CUDA(cudaFuncSetAttribute(bidiag_coop2, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bidiag_coop2, 256, bytes);
    return std::min(per, 2);
  }()};
  const int per_sm = coop_per_sm[v2 ? 1 : 0];
  if (per_sm == 0) return false;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* dd = work;
  double* de = work + n;
  double* part = work + 2 * n + 8;
  int mi = static_cast<int>(m);
  const size_t smem = static_cast<size_t>(m + n) * sizeof(double);
  if (v2) {
    void* args[] = {&mi, &n, &a, &lda, &dd, &de};
    RTLR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bidiag_coop2), dim3(sms * per_sm), dim3(256), args,
                                          smem, s));
    gk_multisect<<<(n + 7) / 8, 256, 0, s>>>(n, dd, de, d_sv);
  } else {
    void* args[] = {&mi, &n, &a, &lda, &dd, &de, &part};
    RTLR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bidiag_coop), dim3(sms * per_sm), dim3(256), args,
                                          smem, s));
    gk_bisect<<<(n + 127) / 128, 128, 0, s>>>(n, dd, de, d_sv);
  }
  RTLR_CUDA(cudaGetLastError());
  return true;
}

void jacobi_svd(long long m, int n, double* w, long long ldw, double* v, int max_sweeps, int* host_rotated,
                double* work, cudaStream_t s, int* sweeps_used) {
  if (sweeps_used) *sweeps_used = 0;
  if (n < 2) return;
  const int npad = n + (n & 1);
  int* d_rot = reinterpret_cast<int*>(work);
  double* d_n2 = work + 8;  // n doubles
  col_norm2_kernel<<<n, 256, 0, s>>>(m, w, ldw, d_n2);
  std::vector<double> n2(n);
  RTLR_CUDA(cudaMemcpyAsync(n2.data(), d_n2, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  RTLR_CUDA(cudaStreamSynchronize(s));
  const double tiny = 1e-30 * *std::max_element(n2.begin(), n2.end());
  static const int coop_grid = [] {  // co-resident CTAs of the cooperative sweep kernel (0: unsupported)
    int dev = 0, ok = 0, per = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_sweeps_coop, 256, 0);
    const char* e = std::getenv("RTLR_JACOBI_COOP");
    return (ok && !(e && e[0] == '0')) ? per * sms : 0;
  }();
  if (coop_grid > 0) {
    int* ctl = d_rot;  // 5 ints (work holds >= 8 doubles before d_n2)
    RTLR_CUDA(cudaMemsetAsync(ctl, 0, 5 * sizeof(int), s));
    int grid = std::min(npad / 2, coop_grid);
    void* args[] = {&m, &n, const_cast<int*>(&npad), &w, &ldw, &v, &ctl, const_cast<double*>(&tiny), &max_sweeps};
    RTLR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_sweeps_coop), dim3(grid), dim3(256), args, 0,
                                          s));
    int hc[5];
    RTLR_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(hc), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    if (sweeps_used) *sweeps_used = hc[3];
    *host_rotated = hc[4];
    return;
  }
  // One sweep (npad - 1 dependent rounds, each a small launch) is captured
  // once as a CUDA graph and replayed per sweep: the rounds are
  // launch-latency bound, and a graph launch of the whole sweep costs about
  // one kernel launch.
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  RTLR_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  cudaMemsetAsync(d_rot, 0, sizeof(int), s);
  for (int t = 0; t < npad - 1; ++t) jacobi_round<<<npad / 2, 256, 0, s>>>(m, n, npad, t, w, ldw, v, d_rot, tiny);
  RTLR_CUDA(cudaStreamEndCapture(s, &graph));
  RTLR_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (sweeps_used) *sweeps_used = sweep + 1;
    RTLR_CUDA(cudaGraphLaunch(exec, s));
    RTLR_CUDA(cudaMemcpyAsync(host_rotated, d_rot, sizeof(int), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    if (*host_rotated == 0) break;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
}

}  // namespace cuda
}  // namespace rtlr

// Internals shared by the extern "C" translation units (capi.cpp,
// capi_lr.cpp): the opaque handle types, the exception -> status mapping
// and host/device staging of arguments.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/rtlr_cu.h"
#include "harness.hpp"
#include "problem.hpp"

struct rtlr_cu_config {
  rtlr::cuda::ProblemConfig cfg;
  rtlr::cuda::RunMode mode = rtlr::cuda::RunMode::Both;  // run.mode (problem.hpp:83)
};
struct rtlr_cu_problem {
  std::unique_ptr<rtlr::cuda::Problem> p;
};
struct rtlr_cu_report {
  rtlr::cuda::SolveReport r;
};

namespace rtlr_capi {

using namespace rtlr::cuda;

inline thread_local std::string g_err;

template <class F>
inline int guard(F&& f) {
  try {
    f();
    return RTLR_CU_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return RTLR_CU_CONFIG_ERROR;
  } catch (const CudaError& e) {
    g_err = e.what();
    return RTLR_CU_CUDA_ERROR;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RTLR_CU_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RTLR_CU_RUNTIME_ERROR;
  }
}

inline void need(bool c, const char* msg) {
  if (!c) throw std::invalid_argument(msg);
}

// GPU entry points on a host-only (device < 0) problem fail loudly.
inline Problem& gpu(rtlr_cu_problem* p) {
  need(p != nullptr, "problem: null argument");
  if (p->p->device() < 0) throw std::invalid_argument("problem was assembled host-only (device < 0)");
  return *p->p;
}

// Stages a host or device input vector on the device.
struct In {
  const double* d = nullptr;
  double* owned = nullptr;
  cudaStream_t s = nullptr;
  In(const double* src, size_t n, int where, cudaStream_t s_) : s(s_) {
    if (where == RTLR_CU_DEVICE || src == nullptr) {
      d = src;
      return;
    }
    RTLR_CUDA(cudaMallocAsync(&owned, n * sizeof(double), s));
    RTLR_CUDA(cudaMemcpyAsync(owned, src, n * sizeof(double), cudaMemcpyHostToDevice, s));
    d = owned;
  }
  ~In() {  // stream-ordered release on the stream that allocated it
    if (owned) cudaFreeAsync(owned, s);
  }
};
struct Out {
  double* d = nullptr;
  double* host = nullptr;
  size_t n = 0;
  cudaStream_t s;
  Out(double* dst, size_t n_, int where, cudaStream_t s_) : n(n_), s(s_) {
    if (where == RTLR_CU_DEVICE || dst == nullptr) {
      d = dst;
      return;
    }
    host = dst;
    RTLR_CUDA(cudaMallocAsync(&d, n * sizeof(double), s));
  }
  void finish() {
    if (host) {
      RTLR_CUDA(cudaMemcpyAsync(host, d, n * sizeof(double), cudaMemcpyDeviceToHost, s));
      RTLR_CUDA(cudaStreamSynchronize(s));
    }
  }
  ~Out() {
    if (host && d) cudaFreeAsync(d, s);
  }
};


// Device -> caller copy (host: synchronous).
inline void copy_out(double* dst, const double* src, size_t n, int where, cudaStream_t s) {
  if (n == 0) return;
  RTLR_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double),
                            where == RTLR_CU_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (where != RTLR_CU_DEVICE) RTLR_CUDA(cudaStreamSynchronize(s));
}

}  // namespace rtlr_capi

// Shared device-side definitions for the B200 (sm_100a) solve phase.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace mscg {

// Carries an mscg_code + block/pivot across the C++ layers to the C ABI.
struct Error : std::runtime_error {
  Error(int c, const std::string& m, int blk = -1, int piv = -1)
      : std::runtime_error(m), code(c), block(blk), pivot(piv) {}
  int code, block, pivot;
};

#define MSCG_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? 4 : 3;                     \
      throw ::mscg::Error(code_, std::string("CUDA error: ") +                   \
                                     cudaGetErrorString(e_) + " at " + #call);   \
    }                                                                            \
  } while (0)

// Bit pattern marking "not yet computed" in the triangular-solve vectors: a
// signalling NaN payload no fp64 instruction ever produces (arithmetic NaN
// results are the canonical quiet NaN), so the value doubles as its own
// readiness flag.
constexpr unsigned long long kPendingBits = 0x7FF4DEAD5EC0FFEEull;

#ifdef __CUDACC__

__device__ __forceinline__ bool is_pending(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(v)) == kPendingBits;
}

__device__ __forceinline__ double pending_value() {
  return __longlong_as_double(static_cast<long long>(kPendingBits));
}

// Spin until shared-memory slot `p` holds a computed value.  8-byte aligned
// shared stores are single-copy atomic, so no separate flag or fence is
// needed: the value is published by the producer's st.volatile.
__device__ __forceinline__ double wait_ready(const double* p) {
  const volatile double* vp = p;
  double v = *vp;
  while (is_pending(v)) v = *vp;
  return v;
}

// Same, for warps off the critical path: back off with __nanosleep so that
// polling does not steal issue slots and shared-memory bandwidth from the
// warp that is advancing the dependency chain.
__device__ __forceinline__ double wait_ready_lazy(const double* p, unsigned ns = 64) {
  const volatile double* vp = p;
  double v = *vp;
  while (is_pending(v)) {
    __nanosleep(ns);
    v = *vp;
  }
  return v;
}
#endif  // __CUDACC__

}  // namespace mscg

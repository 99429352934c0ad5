// Shared helpers for the sm_100a kernels of libvismmoe.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/vismmoe.h"

namespace vmm {

// thread-local error text behind vmm_last_error()
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

inline int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return VMM_OK;
  return fail(VMM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// every kernel launch of the library goes through this macro: it checks the
// launch and counts it (vmm_launch_count, the bench's gpu_launches evidence)
void count_launch();
#define VMM_LAUNCH_CHECK(what)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::vmm::cuda_status(_e, what);  \
    ::vmm::count_launch();                                       \
  } while (0)

// Total order on doubles as unsigned keys: a < b  <=>  ord(a) < ord(b)
// (-0.0 and +0.0 map to the same key so they compare equal, as in Python).
__device__ __forceinline__ uint64_t ord_key(double x) {
  if (x == 0.0) x = 0.0;  // fold -0.0
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ float bf16_to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

}  // namespace vmm

// Error plumbing and device checks for the C-ABI (include/vismmoe.h).
#include <cuda_runtime.h>

#include <string>

#include "../../include/vismmoe.h"

namespace vmm {
static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
}  // namespace vmm

extern "C" {

const char *vmm_last_error(void) { return vmm::g_err.c_str(); }

int vmm_abi_version(void) { return 1; }

int vmm_device_check(int dev) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (p.major != 10 || p.minor != 0)
    return vmm::fail(VMM_ECUDA, "libvismmoe is built for sm_100a (B200); found sm_" + std::to_string(p.major) +
                                    std::to_string(p.minor));
  return VMM_OK;
}

}  // extern "C"

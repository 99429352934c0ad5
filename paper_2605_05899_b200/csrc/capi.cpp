// Error plumbing and device checks for the C-ABI (include/vismmoe.h).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/vismmoe.h"

#include <atomic>

namespace vmm {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
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

long long vmm_launch_count(void) { return vmm::g_launches.load(std::memory_order_relaxed); }

int vmm_device_check(int dev) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (p.major != 10 || p.minor != 0)
    return vmm::fail(VMM_ECUDA, "libvismmoe is built for sm_100a (B200); found sm_" + std::to_string(p.major) +
                                    std::to_string(p.minor));
  return VMM_OK;
}

// ---- data-parallel host pool: one shared-memory pool per node, page-locked in every rank ----
int vmm_host_register(void *h_ptr, size_t bytes) {
  cudaError_t e = cudaHostRegister(h_ptr, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  return VMM_OK;
}

int vmm_host_unregister(void *h_ptr) {
  cudaError_t e = cudaHostUnregister(h_ptr);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
  return VMM_OK;
}

// ---- sharded expert cache plumbing: IPC-mapped peer HBM + peer access ----
int vmm_ipc_get(const void *d_ptr, void *h_handle64) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(d_ptr));
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(h_handle64, &h, sizeof(h));
  return VMM_OK;
}

int vmm_ipc_offset(const void *d_ptr, long long *off) {
  // an IPC handle maps the whole allocation: the opener adds the pointer's offset from its base
  typedef CUresult (*RangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);
  static RangeFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return vmm::fail(VMM_ECUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<RangeFn>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = fn(&base, &size, (CUdeviceptr)d_ptr);
  if (r != CUDA_SUCCESS) return vmm::fail(VMM_ECUDA, "cuMemGetAddressRange failed (" + std::to_string((int)r) + ")");
  *off = (long long)((CUdeviceptr)d_ptr - base);
  return VMM_OK;
}

int vmm_ipc_open(const void *h_handle64, void **d_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  return VMM_OK;
}

int vmm_ipc_close(void *d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
  return VMM_OK;
}

int vmm_copy_async(void *d_dst, const void *src, size_t bytes, void *stream) {
  cudaError_t e = cudaMemcpyAsync(d_dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaMemcpyAsync: ") + cudaGetErrorString(e));
  return VMM_OK;
}

int vmm_memset_async(void *d_ptr, int byte_value, size_t bytes, void *stream) {
  cudaError_t e = cudaMemsetAsync(d_ptr, byte_value, bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  return VMM_OK;
}

int vmm_copy2d_async(void *d_dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                     void *stream) {
  cudaError_t e = cudaMemcpy2DAsync(d_dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaMemcpy2DAsync: ") + cudaGetErrorString(e));
  return VMM_OK;
}

int vmm_peer_enable(int peer) {
  int dev = 0, can = 0;
  cudaGetDevice(&dev);
  if (peer == dev) return VMM_OK;
  cudaDeviceCanAccessPeer(&can, dev, peer);
  if (!can) return vmm::fail(VMM_ECUDA, "no peer access to device " + std::to_string(peer));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return VMM_OK;
  }
  if (e != cudaSuccess) return vmm::fail(VMM_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
  return VMM_OK;
}

}  // extern "C"

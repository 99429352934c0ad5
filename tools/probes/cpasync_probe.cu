// Probe: does cp.async + cp.async.mbarrier.arrive.noinc complete in a kernel shaped like
// ffn_pair_kernel<true> (cluster of 2, 352 threads, ~198 KB dynamic smem)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool CLUSTER>
__global__ void probe(const char *src, int *out, int smem_off) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(128));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (CLUSTER) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  const int t = threadIdx.x - 192;
  if (t >= 0 && t < 128) {
    const uint32_t dst = su32(smem + smem_off) + t * 128;
    for (int c = 0; c < 8; ++c)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + ((c ^ (t & 7)) << 4)),
                   "l"(src + (size_t)t * 4096 + c * 16) : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  if (threadIdx.x == 320) {
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 2000000000ull) break;
    }
    out[blockIdx.x] = ok ? (int)((t1 - t0) / 1000) : -1;
  }
  __syncthreads();
  if (CLUSTER) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

int main() {
  char *src; int *out;
  cudaMalloc(&src, 128 * 4096 + 4096); cudaMalloc(&out, 4096);
  const size_t smem = 6 * 32768 + 1024 + 256;
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int variant = 0; variant < 4; ++variant) {
    bool cl = variant & 1;
    size_t sm = (variant & 2) ? 16384 : smem;
    cudaMemset(out, 0, 4096);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4); cfg.blockDim = dim3(352); cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl ? 2 : 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    cudaError_t e = cl ? cudaLaunchKernelEx(&cfg, probe<true>, (const char *)src, out, 0)
                       : cudaLaunchKernelEx(&cfg, probe<false>, (const char *)src, out, 0);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h[4]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cluster=%d smem=%zu launch=%s sync=%s wait_us: %d %d %d %d\n", cl, sm, cudaGetErrorString(e),
           cudaGetErrorString(e2), h[0], h[1], h[2], h[3]);
  }
  return 0;
}

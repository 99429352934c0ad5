// Read-bandwidth probe for decode-sized weight streaming: R bytes spread over 8
// regions ("experts") of 9.44 MB, L2 flushed, CUDA events.  Variants: LSU uint4
// loads with U loads in flight per thread; TMA 1-D bulk copies into an smem ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/read_probe tools/probes/read_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void lsu_read(const uint4 *__restrict__ p, long long n_vec, float *out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (; i + (U - 1) * stride < n_vec; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x ^ v[u].y ^ v[u].z ^ v[u].w);
  }
  for (; i < n_vec; i += stride) { uint4 v = __ldg(p + i); acc += __uint_as_float(v.x ^ v.w); }
  if (acc == 1.2345f) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void bulk_read(const char *__restrict__ p, long long nbytes, float *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const long long per = (nbytes / gridDim.x) & ~(long long)(CHUNK - 1);
  const char *base = p + per * blockIdx.x;
  const int nch = (int)(per / CHUNK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(CHUNK)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + s * CHUNK)),
                 "l"(base + (long long)c * CHUNK), "r"(CHUNK), "r"(smem_u32(&full[s]))
                 : "memory");
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < STAGES && c < nch; ++c) issue(c);
  float acc = 0.f;
  for (int c = 0; c < nch; ++c) {
    const int s = c % STAGES;
    const uint32_t par = (c / STAGES) & 1;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra "
        "W_%=;\n\tD_%=:\n\t}" ::"r"(smem_u32(&full[s])),
        "r"(par)
        : "memory");
    const uint4 *q = reinterpret_cast<const uint4 *>(sm + s * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) { uint4 v = q[i]; acc += __uint_as_float(v.x ^ v.w); }
    __syncthreads();
    if (threadIdx.x == 0 && c + STAGES < nch) issue(c + STAGES);
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const long long slot = 9437184LL;  // 3*768*2048*2
  const long long nbytes = 8 * slot;
  char *buf, *flush;
  float *out;
  cudaMalloc(&buf, 128 * slot);
  cudaMalloc(&flush, 256 << 20);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, 128 * slot);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char *name, auto fn) {
    float best = 1e9, tot = 0;
    for (int i = 0; i < 25; ++i) {
      cudaMemsetAsync(flush, i, 256 << 20);
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 5) { best = ms < best ? ms : best; tot += ms; }
    }
    printf("%-34s best %7.2f us  mean %7.2f us  -> %.2f TB/s (best)\n", name, best * 1e3, tot / 20 * 1e3,
           nbytes / (best * 1e-3) / 1e12);
  };
  const char *p = buf + 17 * slot;  // 8 consecutive slots (an expert-sorted decode layer)
  run("lsu U=8 148x512", [&] { lsu_read<8><<<nsm, 512>>>((const uint4 *)p, nbytes / 16, out); });
  run("lsu U=16 148x512", [&] { lsu_read<16><<<nsm, 512>>>((const uint4 *)p, nbytes / 16, out); });
  run("lsu U=8 296x512", [&] { lsu_read<8><<<2 * nsm, 512>>>((const uint4 *)p, nbytes / 16, out); });
  run("lsu U=4 148x1024", [&] { lsu_read<4><<<nsm, 1024>>>((const uint4 *)p, nbytes / 16, out); });
  run("lsu U=8 148x1024", [&] { lsu_read<8><<<nsm, 1024>>>((const uint4 *)p, nbytes / 16, out); });
  {
    auto k = bulk_read<8, 16384>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    run("bulk 8x16KB 148x256", [&] { k<<<nsm, 256, 8 * 16384>>>(p, nbytes, out); });
  }
  {
    auto k = bulk_read<6, 32768>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("bulk 6x32KB 148x256", [&] { k<<<nsm, 256, 6 * 32768>>>(p, nbytes, out); });
  }
  {
    auto k = bulk_read<12, 16384>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    run("bulk 12x16KB 148x256", [&] { k<<<nsm, 256, 12 * 16384>>>(p, nbytes, out); });
  }
  {
    auto k = bulk_read<4, 16384>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
    run("bulk 4x16KB 296x256", [&] { k<<<2 * nsm, 256, 4 * 16384>>>(p, nbytes, out); });
  }
  run("empty launch", [&] { lsu_read<8><<<nsm, 512>>>((const uint4 *)p, 0, out); });
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

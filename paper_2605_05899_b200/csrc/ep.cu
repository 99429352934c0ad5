// Expert-parallel (EP) token exchange over peer memory -- SURVEY §8(f) row 3.
//
// The alternative to pulling expert weights over NVLink (sharded cache mode):
// every expert's weights stay resident on its owner rank (expert e -> rank
// e % G, the ShardedHome placement) and the TOKEN ROWS move instead -- at C3
// ~40 MB of rows per layer instead of ~1.06 GB of weights.
//
//   dispatch : every pick's row is written straight into its FINAL slot of the
//              owner's expert-grouped FFN input (16-byte P2P stores through the
//              IPC-mapped peer allocation: NVLink/NVSwitch between GPUs) -- the
//              permute by expert is fused into the exchange, the owner runs the
//              grouped tcgen05 FFN on its receive buffer as is;
//   return   : every received row's FFN output is stored back into the source
//              rank's return buffer at the pick index, so the combine reads
//              each token's k rows contiguously (unpermute fused into the return).
// The per-layer (source, expert) counts [G][E] are exchanged by the host and
// give every pick's destination row (vmm_ep_* take the resulting bases).
// The kernels never wait on peers: the host orders the phases (stream sync +
// a process barrier), so the same code is correct on one GPU shared by several
// processes and on an NVSwitch box.
#include "common.cuh"

namespace {

// one warp per pick i (token i / k): the row goes straight to its final slot in
// the owner's expert-grouped FFN input -- owner d = e % G, row
// base[e] + (pos[i] - my_off[e]) where base[e] is where this rank's block of
// expert e starts in d's buffer (expert-major, then source rank, then pick
// order: the owner needs no permute of its own) -- tagged {source rank, i}.
__global__ void ep_dispatch_kernel(const uint4 *__restrict__ xn, int row_vec, const int32_t *__restrict__ ids, int k,
                                   const int32_t *__restrict__ pos, const int32_t *__restrict__ my_off,
                                   const int32_t *__restrict__ base, const unsigned long long *__restrict__ rows_tab,
                                   const unsigned long long *__restrict__ meta_tab, int G, int rank, int M) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < M; i += nw) {
    const int e = ids[i];
    const int d = e % G;
    const long long r = (long long)base[e] + (pos[i] - my_off[e]);
    const uint4 *src = xn + (long long)(i / k) * row_vec;
    uint4 *dst = reinterpret_cast<uint4 *>(rows_tab[d]) + r * row_vec;
    for (int c = lane; c < row_vec; c += 32) dst[c] = __ldg(src + c);
    if (lane == 0) reinterpret_cast<int2 *>(meta_tab[d])[r] = make_int2(rank, i);
  }
}

// one warp per received row r: its FFN output -> the source rank's return
// buffer at the source's pick index (pick order: the combine reads each
// token's k rows contiguously)
__global__ void ep_return_kernel(const uint4 *__restrict__ y_local, int row_vec, const int2 *__restrict__ meta,
                                 const unsigned long long *__restrict__ back_tab, int n_recv) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_recv; r += nw) {
    const int2 m = meta[r];
    const uint4 *src = y_local + (long long)r * row_vec;
    uint4 *dst = reinterpret_cast<uint4 *>(back_tab[m.x]) + (long long)m.y * row_vec;
    for (int c = lane; c < row_vec; c += 32) dst[c] = __ldg(src + c);
  }
}

}  // namespace

extern "C" int vmm_ep_dispatch(const void *d_xn, int H, const int32_t *d_ids, int k, const int32_t *d_pos,
                               const int32_t *d_my_off, const int32_t *d_base, const void *d_rows_tab,
                               const void *d_meta_tab, int G, int rank, int M, void *stream) {
  if (M <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  if (G < 1 || G > 64 || rank < 0 || rank >= G) return vmm::fail(VMM_EVALIDATION, "bad EP rank / world size");
  int blocks = (M + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  ep_dispatch_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const uint4 *)d_xn, H * 2 / 16, d_ids, k, d_pos, d_my_off, d_base, (const unsigned long long *)d_rows_tab,
      (const unsigned long long *)d_meta_tab, G, rank, M);
  VMM_LAUNCH_CHECK("ep_dispatch_kernel");
  return VMM_OK;
}

extern "C" int vmm_ep_return(const void *d_y_local, int H, const void *d_meta, const void *d_back_tab, int n_recv,
                             void *stream) {
  if (n_recv <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  int blocks = (n_recv + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  ep_return_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4 *)d_y_local, H * 2 / 16,
                                                             (const int2 *)d_meta,
                                                             (const unsigned long long *)d_back_tab, n_recv);
  VMM_LAUNCH_CHECK("ep_return_kernel");
  return VMM_OK;
}

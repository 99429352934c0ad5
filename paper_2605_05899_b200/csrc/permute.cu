// Token permutation by expert and the gate-weighted combine.
//
// The reference executes each layer's demanded experts in ascending id order
// (pkg/src/moesim/pipeline.py:573) and has no numerics; here the N*k picks of
// a layer are stably counting-sorted by expert (ties by (token, slot)) so each
// expert's rows are contiguous for the grouped FFN, and the combine reduces
// the k expert outputs per token in slot order (deterministic, no atomics).
#include <mutex>

#include "common.cuh"

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads, 1)
permute_plan_kernel(const int32_t *__restrict__ ids, int n_picks, int k, int E, int32_t *__restrict__ offsets,
                    int32_t *__restrict__ src_row, int32_t *__restrict__ pos) {
  extern __shared__ int32_t cnt[];  // [kWarps][E] then [E] totals
  int32_t *tot = cnt + kWarps * E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * E + E; i += kThreads) cnt[i] = 0;
  __syncthreads();
  const int seg = (n_picks + kWarps - 1) / kWarps;
  const int lo = warp * seg;
  const int hi = min(n_picks, lo + seg);
  // pass 1: per-warp counts (segment order is the pick order)
  for (int c0 = lo; c0 < hi; c0 += 32) {
    int i = c0 + lane;
    int e = (i < hi) ? ids[i] : -1;
    unsigned peers = __match_any_sync(0xffffffffu, e);
    int leader = __ffs(peers) - 1;
    if (e >= 0 && lane == leader) cnt[warp * E + e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // expert totals, exclusive scan over experts, then per-warp bases
  for (int e = threadIdx.x; e < E; e += kThreads) {
    int s = 0;
    for (int w = 0; w < kWarps; ++w) s += cnt[w * E + e];
    tot[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = run;
      int t = tot[e];
      tot[e] = run;
      run += t;
    }
    offsets[E] = run;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kThreads) {
    int run = tot[e];
    for (int w = 0; w < kWarps; ++w) {
      int c = cnt[w * E + e];
      cnt[w * E + e] = run;
      run += c;
    }
  }
  __syncthreads();
  // pass 2: stable positions
  for (int c0 = lo; c0 < hi; c0 += 32) {
    int i = c0 + lane;
    int e = (i < hi) ? ids[i] : -1;
    unsigned peers = __match_any_sync(0xffffffffu, e);
    int leader = __ffs(peers) - 1;
    int rank = __popc(peers & ((1u << lane) - 1u));
    int basep = (e >= 0) ? cnt[warp * E + e] : 0;
    if (e >= 0) {
      int p = basep + rank;
      pos[i] = p;
      src_row[p] = i / k;
    }
    __syncwarp();
    if (e >= 0 && lane == leader) cnt[warp * E + e] = basep + __popc(peers);
    __syncwarp();
  }
}

// Xp[p] = X[src_row[p]] (bf16 rows, 16-byte vectors, one warp per row)
__global__ void permute_rows_kernel(const uint4 *__restrict__ x, const int32_t *__restrict__ src_row, int n,
                                    int row_vec, uint4 *__restrict__ xp) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < n; r += nw) {
    const uint4 *s = x + (long long)src_row[r] * row_vec;
    uint4 *d = xp + (long long)r * row_vec;
    // 8 independent 16-byte loads in flight per lane before the stores (a 4 KB row per warp pass)
    for (int c0 = lane; c0 < row_vec; c0 += 32 * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + 32 * u < row_vec) v[u] = __ldg(s + c0 + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + 32 * u < row_vec) d[c0 + 32 * u] = v[u];
    }
  }
}

// acc[0..7] = sum_j g_j * Y[pos_j][c] (j ascending) + sum_s Ys[s*N + t][c]: the
// k row loads (and the pos/gate loads before them) are all issued up front so
// each thread keeps k x 16 B in flight; the accumulation order is unchanged.
__device__ __forceinline__ void combine_chunk(const uint4 *__restrict__ y, const int32_t *__restrict__ pos,
                                              const float *__restrict__ gates, int t, int k, int row_vec, int c,
                                              const uint4 *__restrict__ ys, int S, int N, float (&acc)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.f;
  constexpr int kJ = 4;  // picks per pass (4 rows x 16 B in flight; keeps the kernel at <= 64 registers)
  for (int j0 = 0; j0 < k; j0 += kJ) {
    int pj[kJ];
    float gj[kJ];
    uint4 v[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (j0 + j < k) {
        pj[j] = __ldg(pos + (long long)t * k + j0 + j);
        gj[j] = __ldg(gates + (long long)t * k + j0 + j);
      }
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (j0 + j < k) v[j] = __ldg(y + (long long)pj[j] * row_vec + c);
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (j0 + j < k) {
        const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&v[j]);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fmaf(gj[j], __bfloat162float(h[q]), acc[q]);
      }
  }
  for (int sx = 0; sx < S; ++sx) {  // shared experts: unit weight, row sx*N + t
    uint4 v = __ldg(ys + ((long long)sx * N + t) * row_vec + c);
    const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&v);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] += __bfloat162float(h[q]);
  }
}

// out[t] = resid[t] + sum_j gates[t,j] * Y[pos[t,j]]; each thread owns 8 columns
__global__ void __launch_bounds__(256, 4) combine_kernel(const uint4 *__restrict__ y, const int32_t *__restrict__ pos,
                               const float *__restrict__ gates, const uint4 *__restrict__ resid, int N, int k,
                               int row_vec, uint4 *__restrict__ out, const uint4 *__restrict__ ys, int S) {
  long long total = (long long)N * row_vec;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int t = (int)(i / row_vec);
    int c = (int)(i % row_vec);
    float acc[8];
    combine_chunk(y, pos, gates, t, k, row_vec, c, ys, S, N, acc);
    uint4 rv = resid ? __ldg(resid + i) : make_uint4(0, 0, 0, 0);
    const __nv_bfloat16 *rh = reinterpret_cast<const __nv_bfloat16 *>(&rv);
    uint4 o;
    __nv_bfloat16 *oh = reinterpret_cast<__nv_bfloat16 *>(&o);
#pragma unroll
    for (int q = 0; q < 8; ++q) oh[q] = __float2bfloat16(__bfloat162float(rh[q]) + acc[q]);
    out[i] = o;
  }
}

// rows of up to 4096 bf16 (512 16-byte chunks) for rmsnorm / combine_norm
constexpr int kMaxRowVec = 512;

}  // namespace


// ---- warp-per-row RMSNorm ----------------------------------------------------
// One warp owns a row: lane l holds 16-byte chunks l, l+32, ... (CH per lane),
// accumulates its sum of squares in chunk order and the warp reduces with an
// xor butterfly -- no block barriers, so many rows are in flight per SM.
template <int CH>
__device__ __forceinline__ float warp_row_ss(const uint4 (&v)[CH], int row_vec) {
  const int lane = threadIdx.x & 31;
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    if (lane + 32 * i < row_vec) {
      const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&v[i]);
#pragma unroll
      for (int q = 0; q < 8; ++q) { const float f = __bfloat162float(h[q]); ss = fmaf(f, f, ss); }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  return ss;
}

template <int CH>
__device__ __forceinline__ void warp_row_norm_store(const uint4 (&v)[CH], int row_vec, float inv,
                                                   const __nv_bfloat16 *__restrict__ w, uint4 *__restrict__ dst) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < row_vec) {
      const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&v[i]);
      uint4 o;
      __nv_bfloat16 *oh = reinterpret_cast<__nv_bfloat16 *>(&o);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float f = __bfloat162float(h[q]) * inv;
        if (w) f *= __bfloat162float(w[c * 8 + q]);
        oh[q] = __float2bfloat16(f);
      }
      dst[c] = o;
    }
  }
}

template <int CH>
__global__ void __launch_bounds__(256)
rmsnorm_warp_kernel(const uint4 *__restrict__ x, const __nv_bfloat16 *__restrict__ w, int n, int row_vec, float eps,
                    uint4 *__restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    uint4 v[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i)
      if (lane + 32 * i < row_vec) v[i] = __ldg(x + (long long)r * row_vec + lane + 32 * i);
    const float inv = rsqrtf(warp_row_ss<CH>(v, row_vec) / (float)(row_vec * 8) + eps);
    warp_row_norm_store<CH>(v, row_vec, inv, w, y + (long long)r * row_vec);
  }
}

extern "C" int vmm_rmsnorm(const void *d_x, const void *d_w, int n, int H, float eps, void *d_y, void *stream) {
  if (n <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  int row_vec = H * 2 / 16;
  if (row_vec > kMaxRowVec) return vmm::fail(VMM_EVALIDATION, "hidden size above 4096");
  int blocks = (n + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaStream_t st = (cudaStream_t)stream;
  const uint4 *x = (const uint4 *)d_x;
  const __nv_bfloat16 *w = (const __nv_bfloat16 *)d_w;
  uint4 *y = (uint4 *)d_y;
  if (row_vec <= 64) rmsnorm_warp_kernel<2><<<blocks, 256, 0, st>>>(x, w, n, row_vec, eps, y);
  else if (row_vec <= 256) rmsnorm_warp_kernel<8><<<blocks, 256, 0, st>>>(x, w, n, row_vec, eps, y);
  else rmsnorm_warp_kernel<16><<<blocks, 256, 0, st>>>(x, w, n, row_vec, eps, y);
  VMM_LAUNCH_CHECK("rmsnorm_warp_kernel");
  return VMM_OK;
}

namespace {
// <= 32 picks (a decode token): one warp, one pick per lane; same stable order
// ---- multi-CTA stable counting sort (large batches) --------------------------
// Picks are split into contiguous chunks of kChunk (one CTA each, 8 warps of
// kChunk/8 picks), so block order, warp order and lane order together are the
// pick order and the sort stays stable:
//   1. plan_count   : per-CTA expert counts           blk[b][e]
//   2. plan_scan    : expert offsets + per-CTA bases  blk[b][e] <- offsets[e] + sum_{b'<b} cnt[b'][e]
//   3. plan_scatter : per-warp bases inside the CTA, ranks by match_any -> pos/src_row
// chunk = picks per CTA (a multiple of 256, chosen by the host so the grid covers the SMs)
constexpr int kChunk = 8192, kPT = 256, kPW = kPT / 32;

__device__ __forceinline__ void chunk_warp_counts(const int32_t *__restrict__ ids, int n_picks, int chunk,
                                                  int32_t *cnt, int E) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kPW * E; i += kPT) cnt[i] = 0;
  __syncthreads();
  const int lo = blockIdx.x * chunk + warp * (chunk / kPW);
  const int hi = min(n_picks, lo + chunk / kPW);
  for (int c0 = lo; c0 < hi; c0 += 32) {
    const int i = c0 + lane;
    const int e = (i < hi) ? __ldg(ids + i) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && lane == __ffs(peers) - 1) cnt[warp * E + e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPT) plan_count_kernel(const int32_t *__restrict__ ids, int n_picks, int chunk,
                                                         int E, int32_t *__restrict__ blk) {
  __shared__ int32_t cnt[kPW * VMM_MAX_EXPERTS];
  chunk_warp_counts(ids, n_picks, chunk, cnt, E);
  for (int e = threadIdx.x; e < E; e += kPT) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kPW; ++w) s += cnt[w * E + e];
    blk[(long long)blockIdx.x * E + e] = s;
  }
}

// one CTA of 1024 threads: S = 1024/E threads per expert, each owning a contiguous
// range of CTAs (block order is pick order, so the per-CTA bases stay stable)
__global__ void __launch_bounds__(1024) plan_scan_kernel(int32_t *__restrict__ blk, int G, int E,
                                                         int32_t *__restrict__ offsets) {
  __shared__ int32_t part[1024];
  __shared__ int32_t tot[VMM_MAX_EXPERTS + 1];
  const int S = 1024 / E;  // E <= 256 -> S >= 4
  const int e = threadIdx.x % E, sl = threadIdx.x / E;
  const bool active = sl < S;
  const int per = (G + S - 1) / S;
  const int b0 = sl * per, b1 = min(G, b0 + per);
  int s = 0;
  if (active)
    for (int b = b0; b < b1; ++b) s += blk[(long long)b * E + e];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < E) {
    int t = 0;
    for (int j = 0; j < S; ++j) t += part[j * E + threadIdx.x];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int x = 0; x < E; ++x) {
      const int t = tot[x];
      tot[x] = run;
      offsets[x] = run;
      run += t;
    }
    offsets[E] = run;
  }
  __syncthreads();
  if (active) {
    int run = tot[e];
    for (int j = 0; j < sl; ++j) run += part[j * E + e];
    for (int b = b0; b < b1; ++b) {
      const int c = blk[(long long)b * E + e];
      blk[(long long)b * E + e] = run;
      run += c;
    }
  }
}

// x/xp != NULL: also copy the rows (fused permute).  Picks are visited in token
// order, so each token row is read from HBM once (into registers) and stored to
// its k permuted positions -- a separate permute_rows pass re-reads the row per
// pick in permuted order (k x the reads once X exceeds L2).
__global__ void __launch_bounds__(kPT) plan_scatter_kernel(const int32_t *__restrict__ ids, int n_picks, int chunk,
                                                           int k, int E, const int32_t *__restrict__ blk,
                                                           int32_t *__restrict__ src_row, int32_t *__restrict__ pos,
                                                           const uint4 *__restrict__ x, int row_vec,
                                                           uint4 *__restrict__ xp) {
  __shared__ int32_t cnt[kPW * VMM_MAX_EXPERTS];
  chunk_warp_counts(ids, n_picks, chunk, cnt, E);
  for (int e = threadIdx.x; e < E; e += kPT) {
    int run = blk[(long long)blockIdx.x * E + e];
#pragma unroll
    for (int w = 0; w < kPW; ++w) {
      const int c = cnt[w * E + e];
      cnt[w * E + e] = run;
      run += c;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lo = blockIdx.x * chunk + warp * (chunk / kPW);
  const int hi = min(n_picks, lo + chunk / kPW);
  for (int c0 = lo; c0 < hi; c0 += 32) {
    const int i = c0 + lane;
    const int e = (i < hi) ? __ldg(ids + i) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    const int basep = (e >= 0) ? cnt[warp * E + e] : 0;
    const int p = (e >= 0) ? basep + __popc(peers & ((1u << lane) - 1u)) : -1;
    if (e >= 0) {
      pos[i] = p;
      src_row[p] = i / k;
    }
    __syncwarp();
    if (e >= 0 && lane == leader) cnt[warp * E + e] = basep + __popc(peers);
    __syncwarp();
    if (xp != nullptr) {
      int cur_t = -1;
      uint4 v[8];  // the current token's row: 8 x 16 B per lane covers H <= 2048; longer rows loop
      for (int j = 0; j < 32; ++j) {
        const int pj = __shfl_sync(0xffffffffu, p, j);
        if (pj < 0) continue;  // warp-uniform
        const int t = (c0 + j) / k;
        for (int c0v = 0; c0v < row_vec; c0v += 32 * 8) {
          if (t != cur_t || row_vec > 32 * 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int c = c0v + lane + 32 * u;
              if (c < row_vec) v[u] = __ldg(x + (long long)t * row_vec + c);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = c0v + lane + 32 * u;
            if (c < row_vec) __stcs(xp + (long long)pj * row_vec + c, v[u]);  // streaming: the FFN reads it once, much later
          }
        }
        cur_t = t;
      }
    }
  }
}

__global__ void permute_plan_warp_kernel(const int32_t *__restrict__ ids, int n_picks, int k, int E,
                                         int32_t *__restrict__ offsets, int32_t *__restrict__ src_row,
                                         int32_t *__restrict__ pos) {
  const int lane = threadIdx.x;
  const int e = lane < n_picks ? ids[lane] : 0x7fffffff;
  // offsets: count picks with expert < x for every x, chunk by chunk over the expert ids
  for (int c0 = 0; c0 <= E; c0 += 32) {
    const int x = c0 + lane;
    int below = 0;
    for (int j = 0; j < n_picks; ++j) below += (__shfl_sync(0xffffffffu, e, j) < x);
    if (x <= E) offsets[x] = below;
  }
  if (lane < n_picks) {
    // stable rank: picks with a smaller expert, plus equal experts earlier in pick order
    int p = 0;
    for (int j = 0; j < n_picks; ++j) {
      const int ej = __shfl_sync(0xffffffffu, e, j);  // all lanes participate below via the mask
      p += (ej < e) || (ej == e && j < lane);
    }
    pos[lane] = p;
    src_row[p] = lane / k;
  } else {
    for (int j = 0; j < n_picks; ++j) (void)__shfl_sync(0xffffffffu, e, j);
  }
}
}  // namespace

static int permute_impl(const int32_t *d_ids, int N, int k, int E, int32_t *d_offsets, int32_t *d_src_row,
                        int32_t *d_pos, const void *d_x, int H, void *d_xp, void *stream);

extern "C" int vmm_permute_plan(const int32_t *d_ids, int N, int k, int E, int32_t *d_offsets, int32_t *d_src_row,
                                int32_t *d_pos, void *stream) {
  return permute_impl(d_ids, N, k, E, d_offsets, d_src_row, d_pos, nullptr, 0, nullptr, stream);
}

extern "C" int vmm_permute(const int32_t *d_ids, int N, int k, int E, const void *d_x, int H, int32_t *d_offsets,
                           int32_t *d_src_row, int32_t *d_pos, void *d_xp, void *stream) {
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  return permute_impl(d_ids, N, k, E, d_offsets, d_src_row, d_pos, d_x, H, d_xp, stream);
}

static int permute_impl(const int32_t *d_ids, int N, int k, int E, int32_t *d_offsets, int32_t *d_src_row,
                        int32_t *d_pos, const void *d_x, int H, void *d_xp, void *stream) {
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  if (N * k <= 32) {
    permute_plan_warp_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_ids, N * k, k, E, d_offsets, d_src_row, d_pos);
    VMM_LAUNCH_CHECK("permute_plan_warp_kernel");
    return d_xp ? vmm_permute_rows(d_x, d_src_row, N * k, H, d_xp, stream) : VMM_OK;
  }
  const int n_picks = N * k;
  if (n_picks > 2048) {  // multi-CTA stable sort; per-CTA counts in a library scratch (per device)
    // ~16 CTAs per SM (more stores in flight: 2.20 -> 2.04 ms at 2.49M picks), chunks of 1024..8192
    // picks (multiple of 256: 8 warps x whole 32-pick rounds)
    int chunk = (n_picks / (148 * 16) + 255) / 256 * 256;
    chunk = chunk < 1024 ? 1024 : (chunk > kChunk ? kChunk : chunk);
    const int G = (n_picks + chunk - 1) / chunk;
    // per-CTA count scratch, one per (device, stream): plans on different streams may run concurrently
    struct Scratch {
      int dev;
      void *stream;
      int32_t *ptr;
      size_t cap;
    };
    static Scratch tab[64];
    static int ntab = 0;
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t need = (size_t)G * E;
    int32_t *scr = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      Scratch *ent = nullptr;
      for (int i = 0; i < ntab; ++i)
        if (tab[i].dev == dev && tab[i].stream == stream) ent = &tab[i];
      if (!ent) {
        if (ntab == 64) return vmm::fail(VMM_ECUDA, "too many streams for the permute scratch");
        ent = &tab[ntab++];
        *ent = Scratch{dev, stream, nullptr, 0};
      }
      if (ent->cap < need) {
        if (ent->ptr) cudaFree(ent->ptr);
        cudaError_t e = cudaMalloc(&ent->ptr, sizeof(int32_t) * need * 2);
        if (e != cudaSuccess) { ent->ptr = nullptr; ent->cap = 0; return vmm::cuda_status(e, "permute scratch"); }
        ent->cap = need * 2;
      }
      scr = ent->ptr;
    }
    cudaStream_t st = (cudaStream_t)stream;
    plan_count_kernel<<<G, kPT, 0, st>>>(d_ids, n_picks, chunk, E, scr);
    VMM_LAUNCH_CHECK("plan_count_kernel");
    plan_scan_kernel<<<1, 1024, 0, st>>>(scr, G, E, d_offsets);
    VMM_LAUNCH_CHECK("plan_scan_kernel");
    plan_scatter_kernel<<<G, kPT, 0, st>>>(d_ids, n_picks, chunk, k, E, scr, d_src_row, d_pos,
                                           (const uint4 *)d_x, H * 2 / 16, (uint4 *)d_xp);
    VMM_LAUNCH_CHECK("plan_scatter_kernel");
    return VMM_OK;
  }
  if (d_xp) {  // small batches: plan, then the row copy
    int st = permute_impl(d_ids, N, k, E, d_offsets, d_src_row, d_pos, nullptr, 0, nullptr, stream);
    if (st) return st;
    return vmm_permute_rows(d_x, d_src_row, n_picks, H, d_xp, stream);
  }
  size_t smem = sizeof(int32_t) * ((size_t)kWarps * E + E);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(permute_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(int32_t) * (kWarps * VMM_MAX_EXPERTS + VMM_MAX_EXPERTS)));
    if (e != cudaSuccess) return vmm::cuda_status(e, "permute attr");
    attr = true;
  }
  permute_plan_kernel<<<1, kThreads, smem, (cudaStream_t)stream>>>(d_ids, N * k, k, E, d_offsets, d_src_row, d_pos);
  VMM_LAUNCH_CHECK("permute_plan_kernel");
  return VMM_OK;
}

extern "C" int vmm_permute_rows(const void *d_x, const int32_t *d_src_row, int n_rows, int H, void *d_xp,
                                void *stream) {
  if (n_rows <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  int row_vec = H * 2 / 16;
  int blocks = 148 * 8;
  permute_rows_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4 *)d_x, d_src_row, n_rows, row_vec,
                                                                (uint4 *)d_xp);
  VMM_LAUNCH_CHECK("permute_rows_kernel");
  return VMM_OK;
}

extern "C" int vmm_combine(const void *d_y, const int32_t *d_pos, const float *d_gates, const void *d_resid, int N,
                           int k, int H, void *d_out, void *stream) {
  if (N <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  int row_vec = H * 2 / 16;
  long long total = (long long)N * row_vec;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  combine_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4 *)d_y, d_pos, d_gates,
                                                           (const uint4 *)d_resid, N, k, row_vec, (uint4 *)d_out,
                                                           nullptr, 0);
  VMM_LAUNCH_CHECK("combine_kernel");
  return VMM_OK;
}

extern "C" int vmm_combine_shared(const void *d_y, const int32_t *d_pos, const float *d_gates, const void *d_resid,
                                  int N, int k, int H, const void *d_ys, int S, void *d_out, void *stream) {
  if (N <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  int row_vec = H * 2 / 16;
  long long total = (long long)N * row_vec;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  combine_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4 *)d_y, d_pos, d_gates,
                                                           (const uint4 *)d_resid, N, k, row_vec, (uint4 *)d_out,
                                                           (const uint4 *)d_ys, S);
  VMM_LAUNCH_CHECK("combine_kernel");
  return VMM_OK;
}

namespace {
// shared-expert "routing": every token goes to each of the S shared experts:
// src[s*N + t] = t, offsets[s] = s*N
__global__ void shared_plan_kernel(int N, int S, int32_t *__restrict__ src, int32_t *__restrict__ offs) {
  long long total = (long long)N * S;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    src[i] = (int32_t)(i % N);
  if (blockIdx.x == 0 && threadIdx.x <= S) offs[threadIdx.x] = threadIdx.x * N;
}
}  // namespace

extern "C" int vmm_shared_plan(int N, int S, int32_t *d_src, int32_t *d_offsets, void *stream) {
  if (S <= 0 || N <= 0) return VMM_OK;
  if (S > 255) return vmm::fail(VMM_EVALIDATION, "too many shared experts");
  long long total = (long long)N * S;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  shared_plan_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(N, S, d_src, d_offsets);
  VMM_LAUNCH_CHECK("shared_plan_kernel");
  return VMM_OK;
}

namespace {
template <class T>
__global__ void gather_elems_kernel(const T *__restrict__ src, const int32_t *__restrict__ rows, int n, int width,
                                    T *__restrict__ dst) {
  long long total = (long long)n * width;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int r = (int)(i / width), c = (int)(i % width);
    dst[i] = src[(long long)rows[r] * width + c];
  }
}
}  // namespace

extern "C" int vmm_gather_i32(const int32_t *d_src, const int32_t *d_rows, int n, int width, int32_t *d_dst,
                              void *stream) {
  if (n <= 0) return VMM_OK;
  long long total = (long long)n * width;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  gather_elems_kernel<int32_t><<<blocks, 256, 0, (cudaStream_t)stream>>>(d_src, d_rows, n, width, d_dst);
  VMM_LAUNCH_CHECK("gather_elems_kernel<i32>");
  return VMM_OK;
}

extern "C" int vmm_gather_f32(const float *d_src, const int32_t *d_rows, int n, int width, float *d_dst,
                              void *stream) {
  if (n <= 0) return VMM_OK;
  long long total = (long long)n * width;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  gather_elems_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(d_src, d_rows, n, width, d_dst);
  VMM_LAUNCH_CHECK("gather_elems_kernel<f32>");
  return VMM_OK;
}

namespace {
}  // namespace

extern "C" int vmm_combine_norm(const void *d_y, const int32_t *d_pos, const float *d_gates, const void *d_resid,
                                int N, int k, int H, const void *d_ys, int S, float eps, void *d_out, void *d_xn,
                                void *stream) {
  // Two passes, measured faster than one fused kernel at every batch size on B200
  // (R=256 cached layer: 2.51 + 0.42 ms vs 3.64 ms CTA-per-row / 4.22 ms warp-per-row
  // fused; after the combine's register trim 1.97 + 0.41 = 2.37 ms vs 2.92 ms for a
  // warp-per-row version built on the same combine_chunk): the combine keeps one thread
  // per (token, 16-byte chunk) with its row loads in flight and no barrier; the norm
  // re-reads the rounded rows from L2/HBM.
  // Bit-identical to vmm_combine_shared followed by vmm_rmsnorm by construction.
  int st = vmm_combine_shared(d_y, d_pos, d_gates, d_resid, N, k, H, d_ys, S, d_out, stream);
  if (st) return st;
  return vmm_rmsnorm(d_out, nullptr, N, H, eps, d_xn, stream);
}

// ---- decode glue: one CTA per decode layer ----------------------------------
// For a decode token (n <= 2 rows, n*k <= 16 picks) the per-layer glue is six
// tiny launches (combine, RMSNorm, two trace gathers, plan, row copy), each a
// few microseconds of launch/dependency latency for a few KB of work.  This
// kernel does all of it in one CTA with the same arithmetic as those kernels
// (combine_chunk, warp_row_ss / warp_row_norm_store, the stable (expert, pick)
// order of the plan), so the results are bit-identical:
//   A (warp per row): out = resid + sum_j g_j Y[pos_j]  (skipped when y == NULL:
//                     the layer's input is already `resid`), xn = RMSNorm(out)
//   B (thread 0):     ids/gates of layer l from the trace rows, stable counting
//                     sort by expert -> offsets, src_row, pos
//   C (warp per pick): xp[p] = xn[src_row[p]]
namespace {
constexpr int kGlueMaxRows = 4, kGlueMaxPicks = 32;

template <int CH>
__global__ void __launch_bounds__(256)
decode_glue_kernel(const uint4 *__restrict__ y, const int32_t *pos_prev, const float *gates_prev,
                   const uint4 *__restrict__ resid, int n, int k, int row_vec, uint4 *out, uint4 *xn,
                   const int32_t *tr_l,
                   const float *tg_l, const int32_t *__restrict__ rows, int E, int32_t *ids, float *gates,
                   int32_t *offsets, int32_t *src_row, int32_t *pos, uint4 *xp, float eps) {
  __shared__ uint4 s_xn[kGlueMaxRows][kMaxRowVec];
  __shared__ int s_src[kGlueMaxPicks], s_ids[kGlueMaxPicks];
  __shared__ float s_gts[kGlueMaxPicks];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = n * k;
  // B, part 1: the last warp stages this layer's trace ids/gates (consumed after the barrier)
  if (warp == (int)(blockDim.x >> 5) - 1 && lane < M) {
    const int t = lane / k, j = lane - t * k;
    const long long src = (long long)rows[t] * k + j;
    s_ids[lane] = tr_l[src];
    s_gts[lane] = tg_l[src];
  }
  // A, part 1: every thread combines (row, 16-byte chunk) items -- the whole block gathers the
  // k expert rows at once (one warp per row left this latency-bound) -- into out and s_xn
  for (int it = threadIdx.x; it < n * row_vec; it += blockDim.x) {
    const int t = it / row_vec, c = it - t * row_vec;
    uint4 v;
    if (y == nullptr) {
      v = resid[(long long)t * row_vec + c];
    } else {
      float acc[8];
      combine_chunk(y, pos_prev, gates_prev, t, k, row_vec, c, nullptr, 0, n, acc);
      const uint4 rv = resid[(long long)t * row_vec + c];
      const __nv_bfloat16 *rh = reinterpret_cast<const __nv_bfloat16 *>(&rv);
      __nv_bfloat16 *oh = reinterpret_cast<__nv_bfloat16 *>(&v);
#pragma unroll
      for (int q = 0; q < 8; ++q) oh[q] = __float2bfloat16(__bfloat162float(rh[q]) + acc[q]);
      out[(long long)t * row_vec + c] = v;
    }
    s_xn[t][c] = v;
  }
  __syncthreads();  // phase A has read pos/gates of the previous layer before B overwrites them
  // A, part 2: warp t normalises row t from shared memory with the warp-per-row kernel's exact
  // arithmetic (lane L: chunks L + 32 i in i order, then the xor tree), in place
  if (warp < n) {
    const int t = warp;
    uint4 v[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = lane + 32 * i;
      if (c < row_vec) v[i] = s_xn[t][c];
    }
    const float inv = rsqrtf(warp_row_ss<CH>(v, row_vec) / (float)(row_vec * 8) + eps);
    __syncwarp();
    warp_row_norm_store<CH>(v, row_vec, inv, nullptr, s_xn[t]);
    __syncwarp();
    for (int c = lane; c < row_vec; c += 32) xn[(long long)t * row_vec + c] = s_xn[t][c];
  }
  // B, part 2 in parallel (it was one thread: ~20 us of dependent loads and local-memory counts
  // per decode layer): lane i of warp 0 owns pick i; the stable (expert, pick) order of the plan
  // is offsets[e] = #picks with a smaller expert, plus the pick's rank among the earlier picks
  // of its expert (__match_any_sync)
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    int below = 0;
    for (int i = 0; i < M; ++i) below += s_ids[i] < e;
    offsets[e] = below;
  }
  if (warp == 0 && lane < M) {
    const unsigned act = M >= 32 ? 0xffffffffu : ((1u << M) - 1u);
    const int e = s_ids[lane];
    ids[lane] = e;
    gates[lane] = s_gts[lane];
    const unsigned peers = __match_any_sync(act, e);
    int below = 0;
    for (int i = 0; i < M; ++i) below += s_ids[i] < e;
    const int p = below + __popc(peers & ((1u << lane) - 1u));
    pos[lane] = p;
    src_row[p] = lane / k;
    s_src[p] = lane / k;
  }
  __syncthreads();
  for (int p = warp; p < M; p += 8) {
    const uint4 *s = s_xn[s_src[p]];
    for (int c = lane; c < row_vec; c += 32) xp[(long long)p * row_vec + c] = s[c];
  }
}
}  // namespace

extern "C" int vmm_decode_glue(const void *d_y, const int32_t *d_pos_prev, const float *d_gates_prev,
                               const void *d_resid, int n, int k, int H, void *d_out, void *d_xn,
                               const int32_t *d_tr_l,
                               const float *d_tg_l, const int32_t *d_rows, int E, int32_t *d_ids, float *d_gates,
                               int32_t *d_offsets, int32_t *d_src_row, int32_t *d_pos, void *d_xp, void *stream) {
  if (n <= 0) return VMM_OK;
  if (n > kGlueMaxRows || n * k > kGlueMaxPicks)
    return vmm::fail(VMM_EVALIDATION, "decode glue: at most 4 rows and 32 picks");
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  const int row_vec = H * 2 / 16;
  if (row_vec > kMaxRowVec) return vmm::fail(VMM_EVALIDATION, "hidden size above 4096");
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  cudaStream_t st = (cudaStream_t)stream;
#define VMM_GLUE(CH)                                                                                            \
  decode_glue_kernel<CH><<<1, 256, 0, st>>>((const uint4 *)d_y, d_pos_prev, d_gates_prev, (const uint4 *)d_resid, \
                                            n, k, row_vec, (uint4 *)d_out, (uint4 *)d_xn, d_tr_l, d_tg_l, d_rows, \
                                            E, d_ids,                                                             \
                                            d_gates, d_offsets, d_src_row, d_pos, (uint4 *)d_xp, 1e-6f)
  if (row_vec <= 64) VMM_GLUE(2);
  else if (row_vec <= 256) VMM_GLUE(8);
  else VMM_GLUE(16);
#undef VMM_GLUE
  VMM_LAUNCH_CHECK("decode_glue_kernel");
  return VMM_OK;
}

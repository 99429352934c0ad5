// Affinity-aware visual-token compression ("prune") -- one CTA per request.
//
// Restates compress() (pkg/src/moesim/compress.py:142-185) on the device,
// bit-exact in fp64:
//   s_norm = (s - lo) / (hi - lo), constant -> 0.5        compress.py:104-114
//   core   = top floor(alpha n) by (-s_norm, id)            compress.py:156-157
//   target = OR of core tokens' prefix-layer expert masks   compress.py:159-161
//   delta  = popc(m & ~target) / popc(m)                    compress.py:135-139
//   score  = s_norm - lam * delta   (separately rounded)    compress.py:172
//   extras = top (k_keep - k_core) by (-score, -s_norm, id) compress.py:174
//   retained = keep U text ids, ascending                   compress.py:63-65
// Both selections are a shared-memory bitonic sort of (key1, key2, id) with
// exact lexicographic tie keys; stream compaction uses block-wide ballot scans.
#include <math.h>

#include "common.cuh"

namespace {

constexpr int kThreads = 1024;
constexpr int kMaxVisual = 8192;
constexpr int kWords = VMM_MAX_EXPERTS / 64;

struct SortBuf {
  uint64_t *k1;
  uint64_t *k2;
  uint32_t *id;
};

__device__ __forceinline__ bool before(uint64_t a1, uint64_t a2, uint32_t ai, uint64_t b1, uint64_t b2,
                                       uint32_t bi) {
  if (a1 != b1) return a1 < b1;
  if (a2 != b2) return a2 < b2;
  return ai < bi;
}

// ascending bitonic sort of npad (power of two) entries
__device__ void bitonic_sort(SortBuf s, int npad) {
  for (int size = 2; size <= npad; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (npad >> 1); i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        uint64_t a1 = s.k1[lo], a2 = s.k2[lo], b1 = s.k1[hi], b2 = s.k2[hi];
        uint32_t ai = s.id[lo], bi = s.id[hi];
        bool swap = up ? before(b1, b2, bi, a1, a2, ai) : before(a1, a2, ai, b1, b2, bi);
        if (swap) {
          s.k1[lo] = b1; s.k2[lo] = b2; s.id[lo] = bi;
          s.k1[hi] = a1; s.k2[hi] = a2; s.id[hi] = ai;
        }
      }
      __syncthreads();
    }
  }
}

// block-wide exclusive scan of a 0/1 flag; returns prefix, writes total to *total
__device__ __forceinline__ int block_scan_flag(int flag, int *warp_tot, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned bal = __ballot_sync(0xffffffffu, flag);
  int in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    int v = (lane < (blockDim.x >> 5)) ? warp_tot[lane] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    warp_tot[32 + lane] = x - v;  // exclusive
    if (lane == 31) *total = x;
  }
  __syncthreads();
  int r = warp_tot[32 + warp] + in_warp;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void token_mask(const int32_t *routes, int P, long long T, int k, long long tok,
                                           uint64_t m[kWords]) {
#pragma unroll
  for (int w = 0; w < kWords; ++w) m[w] = 0;
  for (int p = 0; p < P; ++p) {
    const int32_t *r = routes + ((long long)p * T + tok) * k;
    for (int j = 0; j < k; ++j) {
      int e = r[j];
      m[e >> 6] |= 1ull << (e & 63);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
prune_kernel(const double *__restrict__ sal, const uint8_t *__restrict__ mod, const int32_t *__restrict__ routes,
             const int32_t *__restrict__ req_off, const int32_t *__restrict__ kcore_arr,
             const int32_t *__restrict__ kkeep_arr, long long T, int P, int k, double lam, int npad,
             double *__restrict__ s_norm_out, double *__restrict__ delta_out, double *__restrict__ score_out,
             uint8_t *__restrict__ flags_out, int32_t *__restrict__ retained, int32_t *__restrict__ n_retained,
             uint64_t *__restrict__ target_out, int32_t *__restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  SortBuf sb;
  sb.k1 = reinterpret_cast<uint64_t *>(smem);
  sb.k2 = sb.k1 + npad;
  sb.id = reinterpret_cast<uint32_t *>(sb.k2 + npad);
  int32_t *vis_tok = reinterpret_cast<int32_t *>(sb.id + npad);  // [npad]
  uint8_t *vflag = reinterpret_cast<uint8_t *>(vis_tok + npad);  // [npad] bit0 core bit1 keep
  __shared__ int warp_tot[64];
  __shared__ int s_total, s_nvis, s_bad;
  __shared__ double s_lo[32], s_hi[32];
  __shared__ unsigned long long s_target[kWords];

  const int r = blockIdx.x;
  const long long base = req_off[r];
  const int n_tok = req_off[r + 1] - req_off[r];
  const int k_core = kcore_arr[r], k_keep = kkeep_arr[r];
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);

  if (threadIdx.x == 0) { s_nvis = 0; s_bad = 0; }
  if (threadIdx.x < kWords) s_target[threadIdx.x] = 0ull;
  for (int t = threadIdx.x; t < n_tok; t += blockDim.x) {
    s_norm_out[base + t] = qnan;
    delta_out[base + t] = qnan;
    score_out[base + t] = qnan;
    flags_out[base + t] = 0;
  }
  __syncthreads();

  // 1. visual positions in id order
  for (int c0 = 0; c0 < n_tok; c0 += blockDim.x) {
    int t = c0 + threadIdx.x;
    int f = (t < n_tok) && mod[base + t] == 0;
    int pre = block_scan_flag(f, warp_tot, &s_total);
    int nv = s_nvis;
    if (f && nv + pre < npad) vis_tok[nv + pre] = t;
    __syncthreads();
    if (threadIdx.x == 0) s_nvis = nv + s_total;
    __syncthreads();
  }
  const int n = s_nvis;
  if (n > kMaxVisual || n > npad) {
    if (threadIdx.x == 0) status[r] = 2;
    return;
  }

  // 2. validation + min/max
  double lo = INFINITY, hi = -INFINITY;
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = sal[base + vis_tok[i]];
    if (!isfinite(v) || v < 0.0) bad = 1;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) status[r] = 1;
    return;
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { s_lo[threadIdx.x >> 5] = lo; s_hi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    lo = threadIdx.x < (blockDim.x >> 5) ? s_lo[threadIdx.x] : INFINITY;
    hi = threadIdx.x < (blockDim.x >> 5) ? s_hi[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (threadIdx.x == 0) { s_lo[0] = lo; s_hi[0] = hi; }
  }
  __syncthreads();
  lo = s_lo[0];
  hi = s_hi[0];
  const double span = __dsub_rn(hi, lo);

  // 3. normalised saliency + core sort keys
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    if (i < n) {
      double v = sal[base + vis_tok[i]];
      double s = (hi == lo) ? 0.5 : __ddiv_rn(__dsub_rn(v, lo), span);
      s_norm_out[base + vis_tok[i]] = s;
      sb.k1[i] = ~vmm::ord_key(s);
      sb.k2[i] = 0;
      sb.id[i] = (uint32_t)i;
      vflag[i] = 0;
    } else {
      sb.k1[i] = ~0ull; sb.k2[i] = ~0ull; sb.id[i] = 0xffffffffu;
    }
  }
  __syncthreads();
  bitonic_sort(sb, npad);
  for (int i = threadIdx.x; i < k_core; i += blockDim.x) vflag[sb.id[i]] = 1;
  __syncthreads();

  // 4. target expert set of the core
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (vflag[i] & 1) {
      uint64_t m[kWords];
      token_mask(routes, P, T, k, base + vis_tok[i], m);
#pragma unroll
      for (int w = 0; w < kWords; ++w)
        if (m[w]) atomicOr(&s_target[w], (unsigned long long)m[w]);
    }
  }
  __syncthreads();
  uint64_t tg[kWords];
#pragma unroll
  for (int w = 0; w < kWords; ++w) tg[w] = s_target[w];

  // 5. marginal expansion + score; extras sort keys
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    if (i < n && !(vflag[i] & 1)) {
      long long tok = base + vis_tok[i];
      uint64_t m[kWords];
      token_mask(routes, P, T, k, tok, m);
      int sz = 0, out = 0;
#pragma unroll
      for (int w = 0; w < kWords; ++w) { sz += __popcll(m[w]); out += __popcll(m[w] & ~tg[w]); }
      double d = __ddiv_rn((double)out, (double)sz);
      double s = s_norm_out[tok];
      double p = __dsub_rn(s, __dmul_rn(lam, d));
      delta_out[tok] = d;
      score_out[tok] = p;
      sb.k1[i] = ~vmm::ord_key(p);
      sb.k2[i] = ~vmm::ord_key(s);
      sb.id[i] = (uint32_t)i;
    } else {
      sb.k1[i] = ~0ull; sb.k2[i] = ~0ull; sb.id[i] = 0xffffffffu;
    }
  }
  __syncthreads();
  bitonic_sort(sb, npad);
  for (int i = threadIdx.x; i < k_keep - k_core; i += blockDim.x) vflag[sb.id[i]] |= 2;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (vflag[i] & 1) vflag[i] |= 2;
  if (threadIdx.x < kWords) target_out[(long long)r * kWords + threadIdx.x] = tg[threadIdx.x];
  __syncthreads();

  // 6. retained = keep U text, ascending ids (recompute visual positions in the same order)
  if (threadIdx.x == 0) { s_nvis = 0; s_bad = 0; }
  __syncthreads();
  int n_ret = 0;
  for (int c0 = 0; c0 < n_tok; c0 += blockDim.x) {
    int t = c0 + threadIdx.x;
    int m = (t < n_tok) ? mod[base + t] : 3;
    int isv = (m == 0);
    int vpre = block_scan_flag(isv, warp_tot, &s_total);
    int vbase = s_nvis;
    int vt = s_total;
    int keepv = isv ? ((vflag[vbase + vpre] >> 1) & 1) : 0;
    int f = (m == 1) || keepv;
    int pre = block_scan_flag(f, warp_tot, &s_total);
    if (f) retained[base + n_ret + pre] = t;
    if (t < n_tok) {
      uint8_t fl = 0;
      if (isv) fl = vflag[vbase + vpre] & 3;
      if (f) fl |= 4;
      flags_out[base + t] = fl;
    }
    n_ret += s_total;
    __syncthreads();
    if (threadIdx.x == 0) s_nvis = vbase + vt;
    __syncthreads();
  }
  if (threadIdx.x == 0) { n_retained[r] = n_ret; status[r] = 0; }
}

__global__ void gather_rows_kernel(const uint4 *__restrict__ src, const int32_t *__restrict__ idx, int n,
                                   int row_vec, uint4 *__restrict__ dst) {
  // one warp per row, 16-byte vectors
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < n; row += nwarps) {
    const uint4 *s = src + (long long)idx[row] * row_vec;
    uint4 *d = dst + (long long)row * row_vec;
    for (int c = lane; c < row_vec; c += 32) d[c] = __ldg(s + c);
  }
}

}  // namespace

extern "C" int vmm_prune(const double *d_saliency, const uint8_t *d_modality, const int32_t *d_routes,
                         const int32_t *d_req_off, const int32_t *d_k_core, const int32_t *d_k_keep, int R,
                         int T, int P, int k, int experts, double lam, double *d_s_norm, double *d_delta,
                         double *d_score, uint8_t *d_flags, int32_t *d_retained, int32_t *d_n_retained,
                         uint64_t *d_target, int32_t *d_status, void *stream) {
  if (R <= 0) return VMM_OK;
  if (experts < 1 || experts > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  if (P < 1 || k < 1) return vmm::fail(VMM_EVALIDATION, "prefix_layers must be non-empty and k >= 1");
  int npad = 2;
  while (npad < kMaxVisual && npad < T) npad <<= 1;
  size_t smem = (size_t)npad * (8 + 8 + 4 + 4 + 1);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((size_t)kMaxVisual * 25));
    if (e != cudaSuccess) return vmm::cuda_status(e, "prune attr");
    attr_set = true;
  }
  prune_kernel<<<R, kThreads, smem, (cudaStream_t)stream>>>(
      d_saliency, d_modality, d_routes, d_req_off, d_k_core, d_k_keep, (long long)T, P, k, lam, npad, d_s_norm,
      d_delta, d_score, d_flags, d_retained, d_n_retained, d_target, d_status);
  VMM_LAUNCH_CHECK("prune_kernel");
  return VMM_OK;
}

extern "C" int vmm_gather_rows(const void *d_src, const int32_t *d_idx, int n, int H, void *d_dst, void *stream) {
  if (n <= 0) return VMM_OK;
  if ((H * 2) % 16) return vmm::fail(VMM_EVALIDATION, "hidden size must be a multiple of 8");
  int row_vec = H * 2 / 16;
  int warps = n < 148 * 16 ? n : 148 * 16;
  int blocks = (warps * 32 + 255) / 256;
  gather_rows_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4 *)d_src, d_idx, n, row_vec,
                                                                 (uint4 *)d_dst);
  VMM_LAUNCH_CHECK("gather_rows_kernel");
  return VMM_OK;
}

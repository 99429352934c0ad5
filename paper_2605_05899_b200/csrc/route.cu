// Router: gate projection + per-token top-k + softmax over the selected logits.
//
// The reference has no router; its output contract is the RoutingTrace
// layout (pkg/src/moesim/trace.py:80-81; gates > 0 summing to 1, :375-382).
// Tie-break on equal logits: lower expert id first (as predictor.py:439).
// Also used for the gate-reuse lookahead predictor (layer l+1's gate on h_l).
//
// v1 contraction: shared-memory tiled fp32 FMA, one fixed accumulation order
// per (token, expert) so integer-valued inputs give exact logits.
#include <math.h>

#include "common.cuh"

namespace {

constexpr int kTok = 16;    // tokens per CTA
constexpr int kKc = 64;     // K chunk
constexpr int kThreads = 256;
constexpr int kMaxE = 256;
constexpr int kMaxK = 16;

__global__ void __launch_bounds__(kThreads)
route_kernel(const __nv_bfloat16 *__restrict__ x, const __nv_bfloat16 *__restrict__ wg, int N, int H, int E,
             int k, int32_t *__restrict__ ids, float *__restrict__ gates, float *__restrict__ logits_out,
             uint32_t *__restrict__ counts) {
  extern __shared__ __align__(16) float sm[];
  float *xs = sm;                      // [kTok][kKc+1]
  float *ws = xs + kTok * (kKc + 1);   // [E][kKc+1]
  float *lg = ws + E * (kKc + 1);      // [kTok][E]
  const int t0 = blockIdx.x * kTok;
  const int tx = threadIdx.x & 31;     // expert lane
  const int ty = threadIdx.x >> 5;     // token group (8 groups x 2 tokens)
  const int ej = (E + 31) / 32;
  float acc[2][kMaxE / 32];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < kMaxE / 32; ++j) acc[a][j] = 0.f;

  for (int k0 = 0; k0 < H; k0 += kKc) {
    for (int i = threadIdx.x; i < kTok * kKc; i += kThreads) {
      int r = i / kKc, c = i % kKc;
      int t = t0 + r;
      xs[r * (kKc + 1) + c] = (t < N && k0 + c < H) ? __bfloat162float(x[(long long)t * H + k0 + c]) : 0.f;
    }
    for (int i = threadIdx.x; i < E * kKc; i += kThreads) {
      int r = i / kKc, c = i % kKc;
      ws[r * (kKc + 1) + c] = (k0 + c < H) ? __bfloat162float(wg[(long long)r * H + k0 + c]) : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < kKc; ++c) {
      float xa = xs[(2 * ty) * (kKc + 1) + c];
      float xb = xs[(2 * ty + 1) * (kKc + 1) + c];
#pragma unroll
      for (int j = 0; j < kMaxE / 32; ++j) {
        if (j < ej) {
          int e = tx + 32 * j;
          float w = (e < E) ? ws[e * (kKc + 1) + c] : 0.f;
          acc[0][j] = fmaf(xa, w, acc[0][j]);
          acc[1][j] = fmaf(xb, w, acc[1][j]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < kMaxE / 32; ++j) {
      int e = tx + 32 * j;
      if (j < ej && e < E) lg[(2 * ty + a) * E + e] = acc[a][j];
    }
  __syncthreads();

  // top-k per token: one warp per token
  for (int r = ty; r < kTok; r += kThreads / 32) {
    int t = t0 + r;
    if (t >= N) break;
    const float *row = lg + r * E;
    if (logits_out)
      for (int e = tx; e < E; e += 32) logits_out[(long long)t * E + e] = row[e];
    unsigned taken[kMaxE / 32];
#pragma unroll
    for (int j = 0; j < kMaxE / 32; ++j) taken[j] = 0;
    float vals[kMaxK];
    int sel[kMaxK];
    for (int s = 0; s < k; ++s) {
      float best = -INFINITY;
      int bi = 0x7fffffff;
      for (int j = 0; j < ej; ++j) {
        int e = tx + 32 * j;
        if (e < E && !((taken[j] >> tx) & 1u)) {
          float v = row[e];
          if (v != v) v = -INFINITY;  // NaN ranks below every number
          if (v > best || (v == best && e < bi) || bi == 0x7fffffff) { best = v; bi = e; }
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi != 0x7fffffff && (bi == 0x7fffffff || ov > best || (ov == best && oi < bi))) { best = ov; bi = oi; }
      }
      if (bi == 0x7fffffff) bi = 0;  // unreachable for k <= E; keeps indices in range
      vals[s] = best;
      sel[s] = bi;
      if ((bi & 31) == tx) taken[bi >> 5] |= 1u << tx;
    }
    if (tx == 0) {
      float m = vals[0];
      float ex[kMaxK];
      float sum = 0.f;
      for (int s = 0; s < k; ++s) { ex[s] = expf(vals[s] - m); sum += ex[s]; }
      for (int s = 0; s < k; ++s) {
        if (ids) ids[(long long)t * k + s] = sel[s];
        if (gates) gates[(long long)t * k + s] = ex[s] / sum;
        if (counts) atomicAdd(&counts[sel[s]], 1u);
      }
    }
  }
}

// ---- skinny path (decode-sized N): spread the gate rows over many CTAs ----
constexpr int kSkinnyMaxN = 32;

// logits[n][g] = x[n] . W[g] for g in [0, G): one warp per gate row, all N tokens.
// The warp's whole gate row (CPL 16-byte chunks per lane) is loaded up front, so a
// launch is one DRAM round trip for W plus the token rows from L2 -- not CPL of
// them in sequence.  Lane sums run over its chunks c = lane + 32 j in j order,
// then an xor tree: the same arithmetic as the generic loop below.
template <int CPL>
__global__ void __launch_bounds__(64) skinny_logits_reg_kernel(const __nv_bfloat16 *__restrict__ x,
                                                               const __nv_bfloat16 *__restrict__ w, int N, int H,
                                                               int G, float *__restrict__ logits) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= G) return;
  const uint4 *wr = reinterpret_cast<const uint4 *>(w + (long long)warp * H);
  const int nv = H / 8;
  uint4 wv[CPL];
#pragma unroll
  for (int j = 0; j < CPL; ++j) {
    const int c = lane + 32 * j;
    wv[j] = c < nv ? __ldg(wr + c) : make_uint4(0u, 0u, 0u, 0u);
  }
  for (int n0 = 0; n0 < N; n0 += 2) {
    float acc[2] = {0.f, 0.f};
    uint4 xv[2][CPL];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int c = lane + 32 * j;
        xv[r][j] = (n0 + r < N && c < nv) ? __ldg(reinterpret_cast<const uint4 *>(x + (long long)(n0 + r) * H) + c)
                                          : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        if (lane + 32 * j < nv) {
          const __nv_bfloat16 *wh = reinterpret_cast<const __nv_bfloat16 *>(&wv[j]);
          const __nv_bfloat16 *xh = reinterpret_cast<const __nv_bfloat16 *>(&xv[r][j]);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[r] = fmaf(__bfloat162float(xh[q]), __bfloat162float(wh[q]), acc[r]);
        }
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float v = acc[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && n0 + r < N) logits[(long long)(n0 + r) * G + warp] = v;
    }
  }
}

// generic H (more than 16 chunks per lane): the same sums, one chunk at a time
__global__ void skinny_logits_kernel(const __nv_bfloat16 *__restrict__ x, const __nv_bfloat16 *__restrict__ w,
                                     int N, int H, int G, float *__restrict__ logits) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= G) return;
  const uint4 *wr = reinterpret_cast<const uint4 *>(w + (long long)warp * H);
  const int nv = H / 8;
  float acc[kSkinnyMaxN];
#pragma unroll
  for (int n = 0; n < kSkinnyMaxN; ++n) acc[n] = 0.f;
  for (int c = lane; c < nv; c += 32) {
    uint4 wv = __ldg(wr + c);
    const __nv_bfloat16 *wh = reinterpret_cast<const __nv_bfloat16 *>(&wv);
    float wf[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) wf[q] = __bfloat162float(wh[q]);
#pragma unroll
    for (int n = 0; n < kSkinnyMaxN; ++n) {
      if (n < N) {
        uint4 xv = __ldg(reinterpret_cast<const uint4 *>(x + (long long)n * H) + c);
        const __nv_bfloat16 *xh = reinterpret_cast<const __nv_bfloat16 *>(&xv);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[n] = fmaf(__bfloat162float(xh[q]), wf[q], acc[n]);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < kSkinnyMaxN; ++n) {
    if (n < N) {
      float v = acc[n];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) logits[(long long)n * G + warp] = v;
    }
  }
}

// per (token, gate group): top-k by (logit desc, id asc; NaN ranks last) -- order-preserving
// u32 keys, one warp max + one warp min (the lowest id among the equal keys) per pick (REDUX);
// taken / padding columns carry key 0, below every real key (-inf maps to 0x007fffff)
__global__ void skinny_topk_kernel(const float *__restrict__ logits, int N, int E, int NG, int k,
                                   int32_t *__restrict__ ids, float *__restrict__ gates,
                                   float *__restrict__ logits_out, uint32_t *__restrict__ counts,
                                   uint32_t *__restrict__ la_counts) {
  const int t = blockIdx.x;
  const int g = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= N || g >= NG) return;
  const float *row = logits + (long long)t * NG * E + (long long)g * E;
  uint32_t key[kMaxE / 32];
#pragma unroll
  for (int j = 0; j < kMaxE / 32; ++j) {
    const int e = lane + 32 * j;
    float f = e < E ? row[e] : -INFINITY;
    if (f != f) f = -INFINITY;
    if (g == 0 && logits_out && e < E) logits_out[(long long)t * E + e] = f;
    const uint32_t u = __float_as_uint(f);
    key[j] = e < E ? ((u & 0x80000000u) ? ~u : (u | 0x80000000u)) : 0u;
  }
  float vals[kMaxK];
  int sel[kMaxK];
  for (int s = 0; s < k; ++s) {
    uint32_t bk = 0u;
    int bj = 0;
#pragma unroll
    for (int j = 0; j < kMaxE / 32; ++j)
      if (key[j] > bk) { bk = key[j]; bj = j; }  // strict: the lower column wins in-lane ties
    const uint32_t m = __reduce_max_sync(0xffffffffu, bk);
    const uint32_t cand = (bk == m) ? (uint32_t)(lane + 32 * bj) : 0xffffffffu;
    int e = (int)__reduce_min_sync(0xffffffffu, cand);
    if (e >= E) e = 0;  // unreachable for k <= E; keeps indices in range
    sel[s] = e;
    vals[s] = __uint_as_float((m & 0x80000000u) ? (m & 0x7fffffffu) : ~m);
    if ((e & 31) == lane) {
#pragma unroll
      for (int j = 0; j < kMaxE / 32; ++j)
        if (j == (e >> 5)) key[j] = 0u;
    }
  }
  if (lane == 0) {
    if (g == 0) {
      float ex[kMaxK], sum = 0.f;
      for (int s = 0; s < k; ++s) { ex[s] = expf(vals[s] - vals[0]); sum += ex[s]; }
      for (int s = 0; s < k; ++s) {
        if (ids) ids[(long long)t * k + s] = sel[s];
        if (gates) gates[(long long)t * k + s] = ex[s] / sum;
        if (counts) atomicAdd(&counts[sel[s]], 1u);
      }
    } else if (la_counts) {
      for (int s = 0; s < k; ++s) atomicAdd(&la_counts[sel[s]], 1u);
    }
  }
}

int route_skinny(const void *x, const void *w, int N, int H, int E, int NG, int k, int32_t *ids, float *gates,
                 float *logits_out, uint32_t *counts, uint32_t *la_counts, cudaStream_t s) {
  static float *scratch = nullptr;  // [kSkinnyMaxN][2*kMaxE] fp32 logits
  if (!scratch) {
    cudaError_t e = cudaMalloc(&scratch, sizeof(float) * kSkinnyMaxN * 2 * kMaxE);
    if (e != cudaSuccess) return vmm::cuda_status(e, "skinny scratch");
  }
  const int G = NG * E;
  const int cpl = (H / 8 + 31) / 32;  // 16-byte chunks of a gate row per lane
  const __nv_bfloat16 *xb = (const __nv_bfloat16 *)x, *wb = (const __nv_bfloat16 *)w;
  const int grid2 = (G + 1) / 2;       // two warps (gate rows) per CTA: G/2 SMs stream W at once
  switch (cpl) {
#define VMM_CPL(C) \
  case C: skinny_logits_reg_kernel<C><<<grid2, 64, 0, s>>>(xb, wb, N, H, G, scratch); break;
    VMM_CPL(1) VMM_CPL(2) VMM_CPL(3) VMM_CPL(4) VMM_CPL(5) VMM_CPL(6) VMM_CPL(7) VMM_CPL(8)
    VMM_CPL(9) VMM_CPL(10) VMM_CPL(11) VMM_CPL(12) VMM_CPL(13) VMM_CPL(14) VMM_CPL(15) VMM_CPL(16)
#undef VMM_CPL
    default: skinny_logits_kernel<<<(G * 32 + 255) / 256, 256, 0, s>>>(xb, wb, N, H, G, scratch);
  }
  VMM_LAUNCH_CHECK("skinny_logits_kernel");
  skinny_topk_kernel<<<N, 32 * NG, 0, s>>>(scratch, N, E, NG, k, ids, gates, logits_out, counts, la_counts);
  VMM_LAUNCH_CHECK("skinny_topk_kernel");
  return VMM_OK;
}

}  // namespace

namespace vmm {
int route_sm100(const void *x, const void *wg_base, int w_row0, long long w_rows, int N, int H, int E, int k,
                int32_t *ids, float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, bool fused,
                int batch_rows, cudaStream_t s);
}

extern "C" int vmm_route_lookahead_ex(const void *d_x, const void *d_router, int layer, int L, int N, int H, int E,
                                      int k, int32_t *d_ids, float *d_gates, uint32_t *d_counts, uint32_t *d_la_counts,
                                      int batch_rows, void *stream) {
  if (N <= 0) return VMM_OK;
  if (layer < 0 || layer + 1 >= L) return vmm::fail(VMM_ECONTRACT, "lookahead needs a next layer");
  if (batch_rows < N) batch_rows = N;
  if (batch_rows <= kSkinnyMaxN && H % 8 == 0 && E <= kMaxE && k <= kMaxK)  // decode-sized: gate rows over many CTAs
    return route_skinny(d_x, (const __nv_bfloat16 *)d_router + (long long)layer * E * H, N, H, E, 2, k, d_ids,
                        d_gates, nullptr, d_counts, d_la_counts, (cudaStream_t)stream);
  int st = vmm::route_sm100(d_x, d_router, layer * E, (long long)L * E, N, H, E, k, d_ids, d_gates, nullptr,
                            d_counts, d_la_counts, true, batch_rows, (cudaStream_t)stream);
  if (st == -1) return vmm::fail(VMM_EVALIDATION, "fused route+lookahead needs E in {16,32,64,128}, H % 64 == 0");
  return st;
}

extern "C" int vmm_route_lookahead(const void *d_x, const void *d_router, int layer, int L, int N, int H, int E, int k,
                                   int32_t *d_ids, float *d_gates, uint32_t *d_counts, uint32_t *d_la_counts,
                                   void *stream) {
  return vmm_route_lookahead_ex(d_x, d_router, layer, L, N, H, E, k, d_ids, d_gates, d_counts, d_la_counts, N,
                                stream);
}

extern "C" int vmm_route_topk_ex(const void *d_x, const void *d_wg, int N, int H, int E, int k, int32_t *d_ids,
                                 float *d_gates, float *d_logits, uint32_t *d_counts, int batch_rows, void *stream) {
  if (N <= 0) return VMM_OK;
  if (E < 1 || E > kMaxE) return vmm::fail(VMM_EVALIDATION, "router: experts must lie in [1, 256]");
  if (k < 1 || k > kMaxK || k > E) return vmm::fail(VMM_EVALIDATION, "router: k must lie in [1, min(16, E)]");
  if (batch_rows < N) batch_rows = N;
  if (batch_rows <= kSkinnyMaxN && H % 8 == 0)  // decode-sized: gate rows over many CTAs
    return route_skinny(d_x, d_wg, N, H, E, 1, k, d_ids, d_gates, d_logits, d_counts, nullptr, (cudaStream_t)stream);
  int st = vmm::route_sm100(d_x, d_wg, 0, E, N, H, E, k, d_ids, d_gates, d_logits, d_counts, nullptr, false,
                            batch_rows, (cudaStream_t)stream);
  if (st != -1) return st;
  // shapes the tcgen05 tile does not cover (E > 128 or H % 64): CUDA-core kernel
  size_t smem = sizeof(float) * ((size_t)kTok * (kKc + 1) + (size_t)E * (kKc + 1) + (size_t)kTok * E);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return vmm::cuda_status(e, "route attr");
    attr = true;
  }
  int grid = (N + kTok - 1) / kTok;
  route_kernel<<<grid, kThreads, smem, (cudaStream_t)stream>>>((const __nv_bfloat16 *)d_x,
                                                              (const __nv_bfloat16 *)d_wg, N, H, E, k, d_ids,
                                                              d_gates, d_logits, d_counts);
  VMM_LAUNCH_CHECK("route_kernel");
  return VMM_OK;
}

extern "C" int vmm_route_topk(const void *d_x, const void *d_wg, int N, int H, int E, int k, int32_t *d_ids,
                              float *d_gates, float *d_logits, uint32_t *d_counts, void *stream) {
  return vmm_route_topk_ex(d_x, d_wg, N, H, E, k, d_ids, d_gates, d_logits, d_counts, N, stream);
}

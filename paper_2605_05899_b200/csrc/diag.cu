// Attention-derived visual-token saliency and GPU routing diagnostics.
//
// Saliency (Alg. 1 line "s <- Mean_h(A^h)",
// PAPER.md:231,260-264): the head-averaged attention each token receives from
// the query set (a CLS query, or the text tokens), computed from the vision
// encoder's Q/K without materialising the attention maps, or from given maps.
// It feeds vmm_prune exactly where the reference reads the trace's saliency
// (compress.py:145-148, trace.py:49).
//
// Diagnostics (row 4; metrics.py:25-67): per-layer working set, top-K
// coverage, inter-layer cosine similarity and Jaccard index of a token
// subset's routing, from the per-layer expert histograms vmm_demand_counts
// already builds.  Counts are integers, so every dot product / sum below is
// exact in fp64 regardless of order, and the remaining sqrt / mul / div are
// single IEEE roundings: the results are bit-identical to the reference's
// numpy/Python arithmetic (compiled with -fmad=false, IEEE div/sqrt).
#include "common.cuh"

namespace {

constexpr int kSalThreads = 256;

__device__ __forceinline__ float block_reduce(float v, float *sh, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  float r = sh[0];
  for (int w = 1; w < kSalThreads / 32; ++w) r = is_max ? fmaxf(r, sh[w]) : r + sh[w];
  return r;
}

// logits: one CTA per (request*head, chunk of 32 keys) stages the chunk's key
// rows and (64 at a time) the head's query rows in smem, then every thread
// computes (query, key) dot products: each K row is read from HBM once.
constexpr int kKeyChunk = 32, kQChunk = 64;
__global__ void __launch_bounds__(kSalThreads)
attn_logits_kernel(const __nv_bfloat16 *__restrict__ q, const __nv_bfloat16 *__restrict__ k, int Q, int N, int D,
                   float scale, float *__restrict__ P) {
  extern __shared__ float sm[];  // keys [kKeyChunk][D], queries [kQChunk][D]
  float *s_k = sm, *s_q = sm + kKeyChunk * D;
  const int rh = blockIdx.x, k0 = blockIdx.y * kKeyChunk;
  const int nk = min(kKeyChunk, N - k0);
  const __nv_bfloat16 *kb = k + ((long long)rh * N + k0) * D;
  for (int i = threadIdx.x; i < nk * D; i += kSalThreads) s_k[i] = __bfloat162float(kb[i]);
  for (int q0 = 0; q0 < Q; q0 += kQChunk) {
    const int nq = min(kQChunk, Q - q0);
    const __nv_bfloat16 *qb = q + ((long long)rh * Q + q0) * D;
    __syncthreads();
    for (int i = threadIdx.x; i < nq * D; i += kSalThreads) s_q[i] = __bfloat162float(qb[i]);
    __syncthreads();
    for (int pidx = threadIdx.x; pidx < nq * nk; pidx += kSalThreads) {
      const int qi = pidx / nk, ki = pidx % nk;
      const float *qr = s_q + qi * D, *kr = s_k + ki * D;
      float acc = 0.f;
      for (int d = 0; d < D; ++d) acc = fmaf(qr[d], kr[d], acc);
      P[((long long)rh * Q + q0 + qi) * N + k0 + ki] = acc * scale;
    }
  }
}

// in-place row softmax over the N keys, one CTA per (request, head, query) row
__global__ void __launch_bounds__(kSalThreads) attn_softmax_kernel(float *__restrict__ P, int N) {
  __shared__ float red[kSalThreads / 32];
  float *prow = P + (long long)blockIdx.x * N;
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < N; i += kSalThreads) mx = fmaxf(mx, prow[i]);
  mx = block_reduce(mx, red, true);
  float sum = 0.f;
  for (int i = threadIdx.x; i < N; i += kSalThreads) {
    const float e = __expf(prow[i] - mx);
    prow[i] = e;
    sum += e;
  }
  sum = block_reduce(sum, red, false);
  const float inv = 1.f / sum;
  for (int i = threadIdx.x; i < N; i += kSalThreads) prow[i] *= inv;
}

// s[r*N + i] = (1 / (Hh*Q)) * sum_{j ascending} P[r*Hh*Q + j][i]  (fp64, fixed order)
__global__ void head_mean_kernel(const float *__restrict__ P, int R, int HQ, int N, double *__restrict__ s) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)R * N) return;
  const int r = (int)(idx / N), i = (int)(idx % N);
  const float *base = P + (long long)r * HQ * N + i;
  double acc = 0.0;
  for (int j = 0; j < HQ; ++j) acc += (double)base[(long long)j * N];
  s[idx] = acc / (double)HQ;
}

// per layer l: out[l] = {working set, top-K coverage, cosine(l, l+1), jaccard(l, l+1)}
// (the last layer's similarity entries are NaN: the reference defines them for l < L-1)
__global__ void routing_diag_kernel(const uint32_t *__restrict__ counts, int L, int E, double n_sub_k, int top,
                                    double *__restrict__ out) {
  const int l = blockIdx.x;
  if (l >= L || threadIdx.x != 0) return;
  const uint32_t *a = counts + (long long)l * E;
  int ws = 0;
  for (int e = 0; e < E; ++e) ws += a[e] != 0;
  // top-K coverage: the sum of the `top` largest counts (order of ties is irrelevant to the sum)
  uint32_t sorted[VMM_MAX_EXPERTS];
  for (int e = 0; e < E; ++e) sorted[e] = a[e];
  for (int i = 1; i < E; ++i) {  // insertion sort, descending (E <= 256, one thread per layer)
    const uint32_t v = sorted[i];
    int j = i - 1;
    while (j >= 0 && sorted[j] < v) { sorted[j + 1] = sorted[j]; --j; }
    sorted[j + 1] = v;
  }
  double covered = 0.0;
  for (int i = 0; i < top && i < E; ++i) covered += (double)sorted[i];
  double cosv = nan(""), jac = nan("");
  if (l + 1 < L) {
    const uint32_t *b = counts + (long long)(l + 1) * E;
    double dot = 0.0, aa = 0.0, bb = 0.0;
    int inter = 0, uni = 0;
    for (int e = 0; e < E; ++e) {
      const double x = (double)a[e], y = (double)b[e];
      dot += x * y;
      aa += x * x;
      bb += y * y;
      inter += (a[e] != 0) && (b[e] != 0);
      uni += (a[e] != 0) || (b[e] != 0);
    }
    const double na = sqrt(aa), nb = sqrt(bb);
    if (na == 0.0 && nb == 0.0) cosv = 1.0;
    else if (na == 0.0 || nb == 0.0) cosv = 0.0;
    else cosv = dot / (na * nb);
    jac = uni == 0 ? 1.0 : (double)inter / (double)uni;
  }
  out[(long long)l * 4 + 0] = (double)ws;
  out[(long long)l * 4 + 1] = covered / n_sub_k;
  out[(long long)l * 4 + 2] = cosv;
  out[(long long)l * 4 + 3] = jac;
}

}  // namespace

extern "C" int vmm_attn_saliency(const void *d_q, const void *d_k, int R, int Hh, int Q, int N, int D, float scale,
                                 float *d_probs, double *d_s, void *stream) {
  if (R <= 0 || Hh <= 0 || Q <= 0 || N <= 0 || D <= 0) return vmm::fail(VMM_EVALIDATION, "empty attention shape");
  if (D > 128) return vmm::fail(VMM_EVALIDATION, "head dim must be <= 128");
  cudaStream_t st = (cudaStream_t)stream;
  dim3 g1(R * Hh, (N + kKeyChunk - 1) / kKeyChunk);
  attn_logits_kernel<<<g1, kSalThreads, sizeof(float) * (kKeyChunk + kQChunk) * D, st>>>(
      (const __nv_bfloat16 *)d_q, (const __nv_bfloat16 *)d_k, Q, N, D, scale, d_probs);
  VMM_LAUNCH_CHECK("attn_logits_kernel");
  attn_softmax_kernel<<<R * Hh * Q, kSalThreads, 0, st>>>(d_probs, N);
  VMM_LAUNCH_CHECK("attn_softmax_kernel");
  const long long n = (long long)R * N;
  head_mean_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_probs, R, Hh * Q, N, d_s);
  VMM_LAUNCH_CHECK("head_mean_kernel");
  return VMM_OK;
}

extern "C" int vmm_attn_map_saliency(const float *d_maps, int R, int HQ, int N, double *d_s, void *stream) {
  if (R <= 0 || HQ <= 0 || N <= 0) return vmm::fail(VMM_EVALIDATION, "empty attention map");
  const long long n = (long long)R * N;
  head_mean_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_maps, R, HQ, N, d_s);
  VMM_LAUNCH_CHECK("head_mean_kernel");
  return VMM_OK;
}

extern "C" int vmm_routing_diagnostics(const uint32_t *d_counts, int L, int E, int n_subset, int k, int top,
                                       double *d_out, void *stream) {
  if (n_subset <= 0) return vmm::fail(VMM_EVALIDATION, "subset must be non-empty");
  if (top < 0 || top > E) return vmm::fail(VMM_EVALIDATION, "top must lie in [0, experts]");
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  routing_diag_kernel<<<L, 32, 0, (cudaStream_t)stream>>>(d_counts, L, E, (double)n_subset * (double)k, top, d_out);
  VMM_LAUNCH_CHECK("routing_diag_kernel");
  return VMM_OK;
}

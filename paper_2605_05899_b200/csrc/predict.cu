// Demand sets and lookahead predictors (pkg/src/moesim/predictor.py).
//
//   vmm_demand_counts  : per-(layer, expert) pick counts over a token subset
//                        (active_union trace.py:102-107; demand_set :115-117)
//   vmm_oracle_targets : decayed-max targets (build_targets :120-148), exact
//   vmm_history        : decayed routing histogram (routing_histogram :63-75),
//                        bit-exact incl. numpy's pairwise normalising sum
//   vmm_mlp_predict    : features (:86-112) + bottleneck MLP (:196-202) + sigmoid (:547)
//   vmm_gate_lookahead : layer l+1 gate applied to h_l (new; no reference)
#include <math.h>

#include "common.cuh"

namespace {

__global__ void demand_counts_kernel(const int32_t *__restrict__ routes, int T, int k, int E,
                                     const int32_t *__restrict__ layers, const int32_t *__restrict__ ids, int n_ids,
                                     uint32_t *__restrict__ counts) {
  extern __shared__ uint32_t hist[];
  const int li = blockIdx.y;
  const int layer = layers[li];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int32_t *base = routes + (long long)layer * T * k;
  const long long total = (long long)n_ids * k;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int t = ids[i / k];
    int e = base[(long long)t * k + (i % k)];
    atomicAdd(&hist[e], 1u);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (hist[e]) atomicAdd(&counts[(long long)li * E + e], hist[e]);
}

__global__ void oracle_targets_kernel(const uint32_t *__restrict__ counts, int L, int E,
                                      const int32_t *__restrict__ ctx, int window, const double *__restrict__ decay,
                                      double *__restrict__ y) {
  const int c = blockIdx.x;
  const int layer = ctx[c];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double g = 0.0;
    for (int d = 1; d <= window; ++d) {
      int fut = layer + d;
      if (fut > L - 1) break;
      double w = decay[d - 1];
      if (counts[(long long)fut * E + e] > 0 && w > g) g = w;
    }
    y[(long long)c * E + e] = g;
  }
}

// numpy pairwise summation of a contiguous float64 vector (loops_utils.h.src)
__device__ double np_pairwise_sum(const double *a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  // n <= 256 (VMM_MAX_EXPERTS): one split level suffices
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

__global__ void history_kernel(const uint32_t *__restrict__ counts, int L, int E, const int32_t *__restrict__ ctx,
                               const double *__restrict__ pw, double *__restrict__ y) {
  __shared__ double acc[VMM_MAX_EXPERTS];
  __shared__ double s_total;
  const int c = blockIdx.x;
  const int layer = ctx[c];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double x = 0.0;
    for (int past = 0; past <= layer; ++past) {
      double w = pw[layer - past];
      if (w == 0.0 && past < layer) continue;
      uint32_t n = counts[(long long)past * E + e];
      for (uint32_t i = 0; i < n; ++i) x = __dadd_rn(x, w);
    }
    acc[e] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) s_total = np_pairwise_sum(acc, E);
  __syncthreads();
  const double tot = s_total;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    y[(long long)c * E + e] = tot > 0.0 ? __ddiv_rn(acc[e], tot) : acc[e];
}

// one CTA per context layer: features then three dense layers, fp64
__global__ void mlp_kernel(const double *__restrict__ hist, const double *__restrict__ emb, int D,
                           const double *__restrict__ drift, const int32_t *__restrict__ ids, int n_ids,
                           const double *__restrict__ hv, const int32_t *__restrict__ ctx, int E,
                           const double *__restrict__ w1, const double *__restrict__ b1, int dh,
                           const double *__restrict__ w2, const double *__restrict__ b2, int db,
                           const double *__restrict__ wo, const double *__restrict__ bo,
                           double *__restrict__ feat_out, double *__restrict__ y) {
  extern __shared__ double sm[];
  const int din = E + 2 * D;
  double *x = sm;            // [din]
  double *a1 = x + din;      // [dh]
  double *a2 = a1 + dh;      // [db]
  const int c = blockIdx.x;
  const int layer = ctx[c];
  for (int e = threadIdx.x; e < E; e += blockDim.x) x[e] = hist[(long long)c * E + e];
  // mean over rows of (emb[ids] + drift[layer]); numpy reduces axis 0 row by row
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double s = 0.0;
    double dr = drift[(long long)layer * D + d];
    for (int i = 0; i < n_ids; ++i) s = __dadd_rn(s, __dadd_rn(emb[(long long)ids[i] * D + d], dr));
    x[E + d] = __ddiv_rn(s, (double)n_ids);
    x[E + D + d] = hv[d];
  }
  __syncthreads();
  if (feat_out)
    for (int i = threadIdx.x; i < din; i += blockDim.x) feat_out[(long long)c * din + i] = x[i];
  for (int o = threadIdx.x; o < dh; o += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < din; ++i) s = fma(x[i], w1[(long long)o * din + i], s);
    s += b1[o];
    a1[o] = s > 0.0 ? s : 0.0;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < db; o += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < dh; ++i) s = fma(a1[i], w2[(long long)o * dh + i], s);
    s += b2[o];
    a2[o] = s > 0.0 ? s : 0.0;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < E; o += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < db; ++i) s = fma(a2[i], wo[(long long)o * db + i], s);
    s += bo[o];
    y[(long long)c * E + o] = 1.0 / (1.0 + exp(-s));
  }
}

// column means of the selected rows (ids in the given order, rows with mod != 0
// skipped when mod is given), accumulated row by row then divided by the count:
// numpy's `emb[rows].mean(axis=0)` order (visual_summary, predictor.py:78-83)
__global__ void row_mean_kernel(const double *__restrict__ emb, int D, const int32_t *__restrict__ ids, int n,
                                const uint8_t *__restrict__ mod, double *__restrict__ out) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x) {
    double s = 0.0;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      const int r = ids[i];
      if (mod && mod[r] != 0) continue;
      s = __dadd_rn(s, emb[(long long)r * D + d]);
      ++cnt;
    }
    out[d] = cnt ? __ddiv_rn(s, (double)cnt) : 0.0;
  }
}

__global__ void normalize_counts_kernel(const uint32_t *__restrict__ counts, int E, double denom,
                                        double *__restrict__ y) {
  for (int e = threadIdx.x; e < E; e += blockDim.x) y[e] = denom > 0 ? (double)counts[e] / denom : 0.0;
}

}  // namespace

extern "C" int vmm_demand_counts(const int32_t *d_routes, int L, int T, int k, int E, const int32_t *d_layers,
                                 int n_layers, const int32_t *d_ids, int n_ids, uint32_t *d_counts, void *stream) {
  if (n_layers <= 0) return VMM_OK;
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(d_counts, 0, sizeof(uint32_t) * (size_t)n_layers * E, s);
  if (e != cudaSuccess) return vmm::cuda_status(e, "demand memset");
  if (n_ids <= 0) return VMM_OK;
  long long total = (long long)n_ids * k;
  int gx = (int)((total + 1023) / 1024);
  if (gx > 16) gx = 16;
  dim3 grid(gx, n_layers);
  demand_counts_kernel<<<grid, 256, sizeof(uint32_t) * E, s>>>(d_routes, T, k, E, d_layers, d_ids, n_ids, d_counts);
  VMM_LAUNCH_CHECK("demand_counts_kernel");
  return VMM_OK;
}

extern "C" int vmm_oracle_targets(const uint32_t *d_counts, int L, int E, const int32_t *d_ctx, int n_ctx,
                                  int window, const double *d_decay, double *d_y, void *stream) {
  if (n_ctx <= 0) return VMM_OK;
  if (window < 1) return vmm::fail(VMM_EVALIDATION, "window must be >= 1");
  oracle_targets_kernel<<<n_ctx, 128, 0, (cudaStream_t)stream>>>(d_counts, L, E, d_ctx, window, d_decay, d_y);
  VMM_LAUNCH_CHECK("oracle_targets_kernel");
  return VMM_OK;
}

extern "C" int vmm_history(const uint32_t *d_counts, int L, int E, const int32_t *d_ctx, int n_ctx,
                           const double *d_pow, double *d_y, void *stream) {
  if (n_ctx <= 0) return VMM_OK;
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  history_kernel<<<n_ctx, 128, 0, (cudaStream_t)stream>>>(d_counts, L, E, d_ctx, d_pow, d_y);
  VMM_LAUNCH_CHECK("history_kernel");
  return VMM_OK;
}

extern "C" int vmm_mlp_predict(const double *d_hist, const double *d_emb, int D, const double *d_drift,
                               const int32_t *d_ids, int n_ids, const double *d_hv, const int32_t *d_ctx, int n_ctx,
                               int E, const double *d_w1, const double *d_b1, int d_hidden, const double *d_w2,
                               const double *d_b2, int d_bottleneck, const double *d_wo, const double *d_bo,
                               double *d_feat, double *d_y, void *stream) {
  if (n_ctx <= 0) return VMM_OK;
  if (n_ids <= 0) return vmm::fail(VMM_ECONTRACT, "retained token set must be non-empty");
  size_t smem = sizeof(double) * ((size_t)E + 2 * D + d_hidden + d_bottleneck);
  if (smem > 200 * 1024) return vmm::fail(VMM_EVALIDATION, "mlp predictor too wide for one CTA");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return vmm::cuda_status(e, "mlp attr");
    attr = true;
  }
  mlp_kernel<<<n_ctx, 256, smem, (cudaStream_t)stream>>>(d_hist, d_emb, D, d_drift, d_ids, n_ids, d_hv, d_ctx, E,
                                                         d_w1, d_b1, d_hidden, d_w2, d_b2, d_bottleneck, d_wo,
                                                         d_bo, d_feat, d_y);
  VMM_LAUNCH_CHECK("mlp_kernel");
  return VMM_OK;
}

extern "C" int vmm_row_mean(const double *d_emb, int D, const int32_t *d_ids, int n, const uint8_t *d_mod,
                            double *d_out, void *stream) {
  if (D <= 0) return VMM_OK;
  row_mean_kernel<<<(D + 127) / 128, 128, 0, (cudaStream_t)stream>>>(d_emb, D, d_ids, n, d_mod, d_out);
  VMM_LAUNCH_CHECK("row_mean_kernel");
  return VMM_OK;
}

extern "C" int vmm_normalize_counts(const uint32_t *d_counts, int E, double denom, double *d_y, void *stream) {
  normalize_counts_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_counts, E, denom, d_y);
  VMM_LAUNCH_CHECK("normalize_counts_kernel");
  return VMM_OK;
}

extern "C" int vmm_gate_lookahead(const void *d_x, const void *d_wnext, int N, int H, int E, int k,
                                  uint32_t *d_scratch_counts, double *d_y, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(d_scratch_counts, 0, sizeof(uint32_t) * (size_t)E, s);
  if (e != cudaSuccess) return vmm::cuda_status(e, "lookahead memset");
  int st = vmm_route_topk(d_x, d_wnext, N, H, E, k, nullptr, nullptr, nullptr, d_scratch_counts, stream);
  if (st) return st;
  normalize_counts_kernel<<<1, 256, 0, s>>>(d_scratch_counts, E, (double)N * (double)k, d_y);
  VMM_LAUNCH_CHECK("normalize_counts_kernel");
  return VMM_OK;
}

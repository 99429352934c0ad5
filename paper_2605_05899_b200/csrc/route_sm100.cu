// Router on 5th-gen tensor cores: logits = X . W_g^T in TMEM, top-k + softmax
// epilogue straight from TMEM, optionally fused with the gate-reuse lookahead
// (layer l+1's gate on the same rows: counts only).
//
// One CTA = 128 token rows (UMMA M=128).  B = the gate rows [EG x K] (or the
// two adjacent gates of layers l and l+1, [2E x K], one TMA box since the
// router weights are stored [L, E, H]).  Warp roles: 0 TMA, 1 TMEM alloc + MMA,
// then one 4-warp epilogue group PER GATE (warps 2..5 gate 0, 6..9 gate 1), so
// the two top-k selections run concurrently.  Epilogue thread t owns row t:
// it pulls its EG logits from TMEM (tcgen05.ld 32x32b.x16) and keeps a
// register-resident sorted top-K list (single pass, insertion only when a
// logit beats the current K-th; strict > keeps the lower expert id first on
// ties), softmaxes the selected logits, writes ids/gates and adds the picks to
// a shared histogram (demand set / lookahead counts).
// Contract as vmm_route_topk (trace.py:80-81; gates sum to 1, :375-382).
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "sm100.cuh"

namespace {

namespace cg = cooperative_groups;

using namespace sm100;

constexpr int BM = 128, BK = 64;
constexpr int kMaxSplit = 16;
// Stages sized so two CTAs share an SM (one's epilogue overlaps the other's loads): plain
// router (NG = 1) 3 x 32 KB, 0.44 -> 0.32 ms at 311k rows; fused lookahead (NG = 2) 2 x 48 KB,
// 0.43 -> 0.39 ms (4 stages at one CTA per SM before)
#ifndef VMM_ROUTE_LA_STAGES
#define VMM_ROUTE_LA_STAGES 2
#endif
template <int NG>
struct RouteStages {
  static constexpr int value = NG == 1 ? 3 : VMM_ROUTE_LA_STAGES;
};
constexpr int kMaxK = 8;

template <int EG, int NG>
struct RouteCfg {
  static constexpr int N = EG * NG;                          // UMMA N
  static constexpr int kThreads = 64 + 128 * NG;
  static constexpr uint32_t kA = BM * BK * 2;                // 16 KB
  static constexpr uint32_t kB = N * BK * 2;
  static constexpr uint32_t kStage = kA + kB;
  static constexpr int kCols = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
  static constexpr int kStages = RouteStages<NG>::value;
  static constexpr size_t kSmem = (size_t)kStages * kStage + 1024 + 256 + 2 * EG * 4;
};

// one row's top-K by (logit desc, id asc): single pass over TMEM columns
template <int EG, int K>
__device__ __forceinline__ void topk_from_tmem(uint32_t taddr, int E, float (&tv)[K], int (&ti)[K],
                                               float *logits_row) {
#pragma unroll
  for (int j = 0; j < K; ++j) { tv[j] = -INFINITY; ti[j] = -1; }
#pragma unroll
  for (int c = 0; c < EG / 16; ++c) {
    uint32_t r[16];
    tmem_ld16_nowait(taddr + c * 16, r);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = c * 16 + i;
      float x = __uint_as_float(r[i]);
      if (x != x) x = -INFINITY;  // NaN ranks below every number
      if (e < E) {
        if (logits_row) logits_row[e] = x;
        if (x > tv[K - 1] || ti[K - 1] < 0) {
          tv[K - 1] = x;
          ti[K - 1] = e;
#pragma unroll
          for (int j = K - 1; j > 0; --j) {
            if (tv[j] > tv[j - 1] || (ti[j - 1] < 0)) {  // strict: earlier (lower id) wins ties
              float fv = tv[j]; tv[j] = tv[j - 1]; tv[j - 1] = fv;
              int fi = ti[j]; ti[j] = ti[j - 1]; ti[j - 1] = fi;
            }
          }
        }
      }
    }
  }
}

template <int EG, int NG, int K>
__device__ __forceinline__ void epilogue(uint32_t t_base, int gate, int row, bool valid, int E,
                                         int32_t *__restrict__ ids, float *__restrict__ gates,
                                         float *__restrict__ logits_out, uint32_t *hist) {
  float tv[K];
  int ti[K];
  float *lrow = (gate == 0 && valid && logits_out) ? logits_out + (long long)row * E : nullptr;
  topk_from_tmem<EG, K>(t_base + gate * EG, E, tv, ti, lrow);
  if (!valid) return;
  if (gate == 0) {
    float ex[K], sum = 0.f;
#pragma unroll
    for (int s = 0; s < K; ++s) { ex[s] = expf(tv[s] - tv[0]); sum += ex[s]; }
#pragma unroll
    for (int s = 0; s < K; ++s) {
      if (ids) ids[(long long)row * K + s] = ti[s];
      if (gates) gates[(long long)row * K + s] = ex[s] / sum;
    }
  }
#pragma unroll
  for (int s = 0; s < K; ++s) atomicAdd(&hist[gate * EG + ti[s]], 1u);
}

template <int EG, int NG, int K>
__global__ void __launch_bounds__(RouteCfg<EG, NG>::kThreads, RouteCfg<EG, NG>::kStages <= 2 || NG == 1 ? 2 : 1)
route_sm100_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, int w_row0,
                   int N, int Kdim, int E, int32_t *__restrict__ ids, float *__restrict__ gates,
                   float *__restrict__ logits_out, uint32_t *__restrict__ counts, uint32_t *__restrict__ la_counts) {
  constexpr int kStages = RouteCfg<EG, NG>::kStages;
  using Cfg = RouteCfg<EG, NG>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem =
      reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * Cfg::kStage);
  uint64_t *empty = full + kStages;
  uint64_t *tmem_full = empty + kStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);
  uint32_t *hist = reinterpret_cast<uint32_t *>(smem + kStages * Cfg::kStage + 256);  // [NG][EG]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * BM;
  const int nk = Kdim / BK;

  for (int i = threadIdx.x; i < NG * EG; i += blockDim.x) hist[i] = 0;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_x);
    prefetch_tmap(&map_w);
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        if (kb >= kStages) mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
        unsigned char *a_dst = smem + s * Cfg::kStage;
        mbar_expect_tx(&full[s], Cfg::kStage);
        tma_load_2d(&map_x, &full[s], a_dst, kb * BK, row0);
        tma_load_2d(&map_w, &full[s], a_dst + Cfg::kA, kb * BK, w_row0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, Cfg::N);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&full[s], (kb / kStages) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * Cfg::kStage);
        const uint32_t b_addr = a_addr + Cfg::kA;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_bf16(tmem, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32), idesc, (kb | kk) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // warp w may only touch TMEM lanes [32*(w%4), +32); gate group = (w-2)/4
    const int q = warp & 3;
    const int gate = (warp - 2) >> 2;
    const int row = row0 + q * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const uint32_t t_base = tmem + ((uint32_t)(q * 32) << 16);
    epilogue<EG, NG, K>(t_base, gate, row, row < N, E, ids, gates, logits_out, hist);
  }
  tc_fence_before();
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    if (counts && hist[e]) atomicAdd(&counts[e], hist[e]);
    if (NG == 2 && la_counts && hist[EG + e]) atomicAdd(&la_counts[e], hist[EG + e]);
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kCols));
  }
}

// ---------------------------------------------------------------------------
// Split-K router for few row tiles (a single request's 1216-2368 rows are 10-19
// tiles: 19 CTAs would stream 9.7 MB through 19 SMs).  One thread-block
// CLUSTER per 128-row tile, S CTAs along K (S a power of two, S * tiles <= #SMs):
// CTA s runs the tcgen05 mainloop over its K slice, spills its fp32 partial
// logits to its own shared memory (the drained stage ring), and after one
// cluster barrier reduces rows [s*128/S, (s+1)*128/S): one warp per (row,
// gate), partials summed over the cluster in rank order (deterministic), then
// the same top-k (logit desc, id asc; NaN ranks last), softmax and demand
// counts as the one-CTA kernel.
// VMM_PRUNE_PROF dev build also stamps the split-K router (tools/route_prof.py):
// %globaltimer of CTA 0 at entry, mainloop done, partial spilled, reduced
#ifdef VMM_PRUNE_PROF
__device__ unsigned long long g_route_ts[8];
#define ROUTE_TS(i)                                                                     \
  do {                                                                                  \
    if (blockIdx.x == 0) {                                                              \
      unsigned long long t_;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      g_route_ts[i] = t_;                                                               \
    }                                                                                   \
  } while (0)
#else
#define ROUTE_TS(i) \
  do {              \
  } while (0)
#endif

template <int EG, int NG>
struct SplitCfg {
  static constexpr int N = EG * NG;
  // warps 0 (TMA) and 1 (MMA), 4 * NG spill warps; all 16 warps share the reduce + top-k,
  // one (row, gate) item per warp at a time: the item's DSMEM loads and REDUX rounds are
  // latency chains, so more warps in flight is what shortens that phase
  static constexpr int kSpillWarps = 4 * NG;
  static constexpr int kThreads = 512;
  static constexpr uint32_t kA = BM * BK * 2;
  static constexpr uint32_t kB = N * BK * 2;
  static constexpr uint32_t kStage = kA + kB;
  static constexpr int kCols = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
  static constexpr int kStages = 4;  // a whole K slice (<= 4 blocks at S >= 8) in flight at once
  static constexpr int kLd = N + 4;  // partial row stride (floats): float4 stores conflict-free
  static constexpr uint32_t kPart = BM * kLd * 4;
  static constexpr uint32_t kBody = (kStages * kStage > kPart) ? kStages * kStage : kPart;
  static constexpr size_t kSmem = (size_t)kBody + 1024 + 256;
};

template <int EG, int NG, int K>
__global__ void __launch_bounds__(SplitCfg<EG, NG>::kThreads, 1)
route_splitk_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, int w_row0,
                    int N, int Kdim, int E, int32_t *__restrict__ ids, float *__restrict__ gates,
                    float *__restrict__ logits_out, uint32_t *__restrict__ counts, uint32_t *__restrict__ la_counts) {
  using Cfg = SplitCfg<EG, NG>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kJ = (EG + 31) / 32;  // columns per lane
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem =
      reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Cfg::kBody);
  uint64_t *empty = full + kStages;
  uint64_t *tmem_full = empty + kStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);
  float *part = reinterpret_cast<float *>(smem);  // [BM][kLd], aliases the drained stage ring

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = (int)(gridDim.x / ((N + BM - 1) / BM)) ;  // cluster size = K splits
  const int s = (int)cluster_ctarank();
  const int row0 = (blockIdx.x / S) * BM;
  const int nk = Kdim / BK;
  const int kb0 = (nk * s) / S, kb1 = (nk * (s + 1)) / S;
  if (threadIdx.x == 0) ROUTE_TS(0);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_x);
    prefetch_tmap(&map_w);
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int st = i % kStages;
        if (i >= kStages) mbar_wait(&empty[st], ((i / kStages) - 1) & 1);
        unsigned char *a_dst = smem + st * Cfg::kStage;
        mbar_expect_tx(&full[st], Cfg::kStage);
        tma_load_2d(&map_x, &full[st], a_dst, kb * BK, row0);
        tma_load_2d(&map_w, &full[st], a_dst + Cfg::kA, kb * BK, w_row0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, Cfg::N);
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int st = i % kStages;
        mbar_wait(&full[st], (i / kStages) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + st * Cfg::kStage);
        const uint32_t b_addr = a_addr + Cfg::kA;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_bf16(tmem, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32), idesc, (i | kk) != 0);
        umma_commit(&empty[st]);
      }
      umma_commit(tmem_full);  // every MMA (and its smem reads) done: the ring may be overwritten
    }
    __syncwarp();
  } else if (warp < 2 + Cfg::kSpillWarps) {
    // spill this CTA's partial: thread owns TMEM lane (= tile row) 32*(w%4)+lane, gate (w-2)/4
    const int q = warp & 3;
    const int gate = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    mbar_wait(tmem_full, 0);
    if (warp == 2 && lane == 0) ROUTE_TS(1);
    tc_fence_after();
    const uint32_t t_base = tmem + ((uint32_t)(q * 32) << 16) + gate * EG;
    float *dst = part + r * Cfg::kLd + gate * EG;
#pragma unroll
    for (int c = 0; c < EG / 16; ++c) {
      uint32_t v[16];
      tmem_ld16_nowait(t_base + c * 16, v);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4 *>(dst + c * 16 + i) =
            make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                        __uint_as_float(v[i + 3]));
    }
  }
  if (warp == 2 && lane == 0) ROUTE_TS(2);
  tc_fence_before();
  cluster_sync_all();  // every CTA's partial is in its shared memory
  if (threadIdx.x == 0) ROUTE_TS(3);
  // reduction: rows [s*BM/S, (s+1)*BM/S) of the tile, one warp per (row, gate)
  const int rows_per = BM / S;
  const int nwarps = Cfg::kThreads / 32;
  cg::cluster_group cl = cg::this_cluster();
  for (int item = warp; item < rows_per * NG; item += nwarps) {
    const int rr = s * rows_per + item / NG, g = item % NG;
    const int row = row0 + rr;
    if (row >= N) continue;  // warp-uniform
    // every rank's loads are issued before any is summed (one DSMEM round trip)
    float pv[kMaxSplit][kJ];
#pragma unroll
    for (int qr = 0; qr < kMaxSplit; ++qr) {
      const float *src = cl.map_shared_rank(part, qr < S ? qr : 0) + rr * Cfg::kLd + g * EG;
#pragma unroll
      for (int j = 0; j < kJ; ++j) pv[qr][j] = (qr < S && lane + 32 * j < EG) ? src[lane + 32 * j] : 0.f;
    }
    float v[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      float acc = pv[0][j];
#pragma unroll
      for (int qr = 1; qr < kMaxSplit; ++qr)
        if (qr < S) acc += pv[qr][j];  // rank order: the same sum in every run
      v[j] = acc;
    }
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int e = lane + 32 * j;
      float x = v[j];
      if (x != x) x = -INFINITY;
      if (e >= E) x = -INFINITY;
      v[j] = x;
      if (g == 0 && logits_out && e < E) logits_out[(long long)row * E + e] = x;
    }
    // top-K by (logit desc, id asc): order-preserving u32 keys, one warp max + one warp
    // min (ids among the equal keys) per pick; taken / padding columns carry key 0,
    // below every real key (-inf maps to 0x007fffff)
    uint32_t key[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const uint32_t u = __float_as_uint(v[j]);
      key[j] = (lane + 32 * j < E) ? ((u & 0x80000000u) ? ~u : (u | 0x80000000u)) : 0u;
    }
    float vals[K];
    int sel[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      uint32_t bk = 0u;
      int bj = 0;
#pragma unroll
      for (int j = 0; j < kJ; ++j)
        if (key[j] > bk) { bk = key[j]; bj = j; }  // strict: the lower column wins in-lane ties
      const uint32_t m = __reduce_max_sync(0xffffffffu, bk);
      const uint32_t cand = (bk == m) ? (uint32_t)(lane + 32 * bj) : 0xffffffffu;
      const int e = (int)__reduce_min_sync(0xffffffffu, cand);
      sel[p] = e;
      vals[p] = __uint_as_float((m & 0x80000000u) ? (m & 0x7fffffffu) : ~m);
      if ((e & 31) == lane) {
#pragma unroll
        for (int j = 0; j < kJ; ++j)
          if (j == (e >> 5)) key[j] = 0u;
      }
    }
    if (lane == 0) {
      if (g == 0) {
        float ex[K], sum = 0.f;
#pragma unroll
        for (int p = 0; p < K; ++p) { ex[p] = expf(vals[p] - vals[0]); sum += ex[p]; }
#pragma unroll
        for (int p = 0; p < K; ++p) {
          if (ids) ids[(long long)row * K + p] = sel[p];
          if (gates) gates[(long long)row * K + p] = ex[p] / sum;
          if (counts) atomicAdd(&counts[sel[p]], 1u);
        }
      } else if (la_counts) {
#pragma unroll
        for (int p = 0; p < K; ++p) atomicAdd(&la_counts[sel[p]], 1u);
      }
    }
  }
  if (threadIdx.x == 0) ROUTE_TS(4);
  cluster_sync_all();  // DSMEM lifetime: no CTA leaves while a peer may read its partial
  if (threadIdx.x == 0) ROUTE_TS(5);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kCols));
  }
}

template <int EG, int NG, int K>
int launch_splitk(int S, const void *x, const void *wg, int w_row0, long long w_rows, int N, int H, int E,
                  int32_t *ids, float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, cudaStream_t st) {
  using Cfg = SplitCfg<EG, NG>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(route_splitk_kernel<EG, NG, K>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(route_splitk_kernel<EG, NG, K>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return vmm::cuda_status(e, "route_splitk attr");
    attr = true;
  }
  CUtensorMap mx, mw;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)N};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, BM};
    if ((rc = make_map(&mx, x, 2, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)w_rows};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, (uint32_t)Cfg::N};
    if ((rc = make_map(&mw, wg, 2, dims, str, box))) return rc;
  }
  const int tiles = (N + BM - 1) / BM;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(tiles * S);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, route_splitk_kernel<EG, NG, K>, mx, mw, w_row0, N, H, E, ids, gates,
                                     logits, counts, la_counts);
  if (e != cudaSuccess) return vmm::cuda_status(e, "route_splitk_kernel launch");
  VMM_LAUNCH_CHECK("route_splitk_kernel");
  return VMM_OK;
}

// K splits for a launch of N rows: the largest power of two S <= 16 with tiles * S <= #SMs
// and at least two 64-wide K blocks per split; 1 = the one-CTA-per-tile kernel
inline int split_k(int N, int H) {
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static int off = -1;  // VMM_ROUTE_NO_SPLITK=1: always the one-CTA kernel
  if (off < 0) off = getenv("VMM_ROUTE_NO_SPLITK") ? 1 : 0;
  if (off) return 1;
  static int forced = -1;  // VMM_ROUTE_SPLIT=S: S splits at every N (measurement knob)
  if (forced < 0) forced = getenv("VMM_ROUTE_SPLIT") ? atoi(getenv("VMM_ROUTE_SPLIT")) : 0;
  if (forced > 0) return forced;
  const int tiles = (N + BM - 1) / BM, nk = H / BK;
  int S = 1;
  while (S < kMaxSplit && tiles * S * 2 <= num_sms && nk >= 4 * S) S <<= 1;
  return S;
}

template <int EG, int NG, int K>
int launch(const void *x, const void *wg, int w_row0, long long w_rows, int N, int H, int E, int32_t *ids,
           float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, int batch_rows, cudaStream_t s) {
  using Cfg = RouteCfg<EG, NG>;
  // the split count (and so the fp32 summation order of every logit) follows the logical
  // batch, not this launch: rows routed in chunks get the bits of one launch over the batch
  const int S = split_k(batch_rows > N ? batch_rows : N, H);
  if (S > 1)
    return launch_splitk<EG, NG, K>(S, x, wg, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, s);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(route_sm100_kernel<EG, NG, K>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
    if (e != cudaSuccess) return vmm::cuda_status(e, "route_sm100 attr");
    attr = true;
  }
  CUtensorMap mx, mw;
  int st;
  {
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)N};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, BM};
    if ((st = make_map(&mx, x, 2, dims, str, box))) return st;
  }
  {
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)w_rows};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, (uint32_t)Cfg::N};
    if ((st = make_map(&mw, wg, 2, dims, str, box))) return st;
  }
  int grid = (N + BM - 1) / BM;
  route_sm100_kernel<EG, NG, K><<<grid, Cfg::kThreads, Cfg::kSmem, s>>>(mx, mw, w_row0, N, H, E, ids, gates, logits,
                                                                       counts, la_counts);
  VMM_LAUNCH_CHECK("route_sm100_kernel");
  return VMM_OK;
}

template <int EG, int NG>
int launch_k(int k, const void *x, const void *wg, int w_row0, long long w_rows, int N, int H, int E, int32_t *ids,
             float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, int batch_rows, cudaStream_t s) {
  switch (k) {
#define VMM_K(KK) \
  case KK: \
    return launch<EG, NG, KK>(x, wg, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, batch_rows, s);
    VMM_K(1) VMM_K(2) VMM_K(3) VMM_K(4) VMM_K(5) VMM_K(6) VMM_K(7) VMM_K(8)
#undef VMM_K
    default: return -1;
  }
}

}  // namespace

namespace vmm {
// tcgen05 router; returns -1 if the shape is not tileable (caller uses the SIMT kernel)
int route_sm100(const void *x, const void *wg_base, int w_row0, long long w_rows, int N, int H, int E, int k,
                int32_t *ids, float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, bool fused,
                int batch_rows, cudaStream_t s) {
  if (H % BK || k > kMaxK || k < 1 || E > 128 || N <= 0) return -1;
  if (fused) {
    switch (E) {
      case 16: return launch_k<16, 2>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, batch_rows, s);
      case 32: return launch_k<32, 2>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, batch_rows, s);
      case 64: return launch_k<64, 2>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, batch_rows, s);
      case 128:
        return launch_k<128, 2>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, batch_rows, s);
      default: return -1;
    }
  }
  if (E <= 16) return launch_k<16, 1>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, batch_rows, s);
  if (E <= 32) return launch_k<32, 1>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, batch_rows, s);
  if (E <= 64) return launch_k<64, 1>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, batch_rows, s);
  return launch_k<128, 1>(
          k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, batch_rows, s);
}
}  // namespace vmm

#ifdef VMM_PRUNE_PROF
extern "C" int vmm_route_prof_read(unsigned long long *out8) {
  return cudaMemcpyFromSymbol(out8, g_route_ts, sizeof(g_route_ts)) == cudaSuccess ? VMM_OK : VMM_ECUDA;
}
#endif

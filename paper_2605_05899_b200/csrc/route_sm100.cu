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
#include <math.h>

#include "sm100.cuh"

namespace {

using namespace sm100;

constexpr int BM = 128, BK = 64;
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

template <int EG, int NG, int K>
int launch(const void *x, const void *wg, int w_row0, long long w_rows, int N, int H, int E, int32_t *ids,
           float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, cudaStream_t s) {
  using Cfg = RouteCfg<EG, NG>;
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
             float *gates, float *logits, uint32_t *counts, uint32_t *la_counts, cudaStream_t s) {
  switch (k) {
#define VMM_K(KK) \
  case KK: return launch<EG, NG, KK>(x, wg, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, s);
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
                cudaStream_t s) {
  if (H % BK || k > kMaxK || k < 1 || E > 128 || N <= 0) return -1;
  if (fused) {
    switch (E) {
      case 16: return launch_k<16, 2>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, s);
      case 32: return launch_k<32, 2>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, s);
      case 64: return launch_k<64, 2>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, s);
      case 128:
        return launch_k<128, 2>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, la_counts, s);
      default: return -1;
    }
  }
  if (E <= 16) return launch_k<16, 1>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, s);
  if (E <= 32) return launch_k<32, 1>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, s);
  if (E <= 64) return launch_k<64, 1>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, s);
  return launch_k<128, 1>(k, x, wg_base, w_row0, w_rows, N, H, E, ids, gates, logits, counts, nullptr, s);
}
}  // namespace vmm

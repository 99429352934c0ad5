// Grouped bf16 SwiGLU expert FFN on 5th-gen tensor cores (sm_100a).
//
//   H1[m, :] = SiLU(Xp[m] . Wg^T) * (Xp[m] . Wu^T)      (GEMM1, fused epilogue)
//   Y [m, :] = H1[m] . Wd^T                              (GEMM2)
// for the rows m of each expert (contiguous after vmm_permute_plan), with the
// expert's weights read from an HBM arena slot chosen by the expert cache
// (slot table).  No reference numerics exist (the reference models expert
// compute as a constant, pkg/src/moesim/pipeline.py:546-552).
//
// Kernel anatomy (one 128x128 output tile per CTA, 6 warps):
//   warp 0      : TMA producer  -- A tile [128 x 64] of Xp/H1 and B tile
//                 [128 x 64] of the weight slot, SWIZZLE_128B, mbarrier tx
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer
//                 (M=128, N=128, K=16 per instruction, fp32 accumulate in TMEM)
//   warps 2..5  : epilogue -- tcgen05.ld 32x32b, SwiGLU / bf16 pack, stores
// A kStages-deep smem ring (full/empty mbarriers) overlaps TMA with MMA.
#include <math.h>

#include <cstdlib>
#include <atomic>
#include <mutex>

#include "sm100.cuh"

// VMM_FFN_PROF (a separate dev build, see tools/ffn_prof.py): per-CTA cycle
// counters of the pair kernel's waits, read back with vmm_ffn_prof_read.
#ifdef VMM_FFN_PROF
__device__ unsigned long long g_ffn_prof[256][24];
__device__ int g_ffn_prof_mode;  // bit 0: skip the H1 dependency waits, bit 1: skip the epilogue stores (wrong results)
#define PROF_T0() const long long _pt0 = clock64()
#define PROF_ADD(slot) (_pacc[slot] += (unsigned long long)(clock64() - _pt0))
#else
#define PROF_T0()
#define PROF_ADD(slot)
#endif

namespace {

using namespace sm100;

constexpr int BM = 128, BN = 128, BK = 64;
constexpr int kStages = 6;
constexpr int kThreads = 192;
constexpr uint32_t kTileBytes = BM * BK * 2;  // 16 KB (A) == BN*BK*2 (B)
constexpr uint32_t kStageBytes = 2 * kTileBytes;
constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
int g_num_sms = 0;

// ---- the grouped GEMM (persistent, warp-specialised) ----------------------
// Tiles: (m_tile, n_tile) with n fastest; m_tiles are ceil(M_e / BM) per expert.
// Roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer, warps 2..5
// epilogue.  The smem ring runs continuously across tiles and the accumulator
// is double-buffered in TMEM (2 x BN columns), so the epilogue of tile i
// overlaps the TMA/MMA of tile i+1 and HBM streaming never drains between tiles.
struct TileInfo {
  int expert, row0, row_end, slot, n_tile;
};

__device__ __forceinline__ TileInfo tile_info(int t, int n_tiles, const int *tile_base, const int *offs,
                                              const int *slots, int E) {
  TileInfo ti;
  const int m_tile = t / n_tiles;
  ti.n_tile = t - m_tile * n_tiles;
  int lo = 0, hi = E - 1;  // last expert with tile_base[e] <= m_tile
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_base[mid] <= m_tile) lo = mid; else hi = mid - 1;
  }
  // skip experts with zero tiles (tile_base[e] == tile_base[e+1])
  while (lo + 1 < E && tile_base[lo + 1] <= m_tile) ++lo;
  ti.expert = lo;
  ti.row0 = offs[lo] + (m_tile - tile_base[lo]) * BM;
  ti.row_end = offs[lo + 1];
  ti.slot = slots[lo];
  return ti;
}

template <bool kSwiGLU>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const int32_t *__restrict__ offsets, const int32_t *__restrict__ slot_of, int E, int K,
                    int n_tiles, __nv_bfloat16 *__restrict__ out, int ld_out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  uint64_t *tmem_full = empty + kStages;   // [2]
  uint64_t *tmem_empty = tmem_full + 2;    // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);
  __shared__ int s_offs[VMM_MAX_EXPERTS + 1], s_tile_base[VMM_MAX_EXPERTS + 1], s_slots[VMM_MAX_EXPERTS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e <= E; e += blockDim.x) s_offs[e] = offsets[e];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_slots[e] = slot_of[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      s_tile_base[e] = acc;
      acc += (s_offs[e + 1] - s_offs[e] + BM - 1) / BM;
    }
    s_tile_base[E] = acc;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tmem_full[b], 1); mbar_init(&tmem_empty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = s_tile_base[E] * n_tiles;
  const int nk = K / BK;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileInfo ti = tile_info(t, n_tiles, s_tile_base, s_offs, s_slots, E);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
          unsigned char *a_dst = smem + s * kStageBytes;
          mbar_expect_tx(&full[s], kStageBytes);
          tma_load_2d(&map_a, &full[s], a_dst, kb * BK, ti.row0);
          tma_load_3d(&map_b, &full[s], a_dst + kTileBytes, kb * BK, ti.n_tile * BN, ti.slot);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int b = local & 1, use = local >> 1;
        if (use > 0) mbar_wait(&tmem_empty[b], (use - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + b * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * kStageBytes);
          const uint32_t b_addr = a_addr + kTileBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)  // 16 bf16 = 32 B steps inside the 128 B swizzle atom
            umma_bf16(acc, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32), idesc_bf16(BM, BN),
                      (kb | kk) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[b]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warp w reads TMEM lanes [32*(w%4), +32)
    const int q = warp & 3;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const TileInfo ti = tile_info(t, n_tiles, s_tile_base, s_offs, s_slots, E);
      const int b = local & 1, use = local >> 1;
      const int row = ti.row0 + q * 32 + lane;
      mbar_wait(&tmem_full[b], use & 1);
      tc_fence_after();
      const uint32_t t_base = tmem + b * BN + ((uint32_t)(q * 32) << 16);
      if constexpr (kSwiGLU) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float g[32], u[32];
          tmem_ld32(t_base + half * 32, g);
          tmem_ld32(t_base + 64 + half * 32, u);
          if (half == 1) {  // accumulator fully read: hand the buffer back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tmem_empty[b]);
          }
          if (row < ti.row_end) {
            uint4 *dst = reinterpret_cast<uint4 *>(out + (long long)row * ld_out + ti.n_tile * (BN / 2) + half * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 o;
              o.x = pack_bf16(silu(g[8 * v + 0]) * u[8 * v + 0], silu(g[8 * v + 1]) * u[8 * v + 1]);
              o.y = pack_bf16(silu(g[8 * v + 2]) * u[8 * v + 2], silu(g[8 * v + 3]) * u[8 * v + 3]);
              o.z = pack_bf16(silu(g[8 * v + 4]) * u[8 * v + 4], silu(g[8 * v + 5]) * u[8 * v + 5]);
              o.w = pack_bf16(silu(g[8 * v + 6]) * u[8 * v + 6], silu(g[8 * v + 7]) * u[8 * v + 7]);
              dst[v] = o;
            }
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float a[32];
          tmem_ld32(t_base + c * 32, a);
          if (c == BN / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tmem_empty[b]);
          }
          if (row < ti.row_end) {
            uint4 *dst = reinterpret_cast<uint4 *>(out + (long long)row * ld_out + ti.n_tile * BN + c * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 o;
              o.x = pack_bf16(a[8 * v + 0], a[8 * v + 1]);
              o.y = pack_bf16(a[8 * v + 2], a[8 * v + 3]);
              o.z = pack_bf16(a[8 * v + 4], a[8 * v + 5]);
              o.w = pack_bf16(a[8 * v + 6], a[8 * v + 7]);
              dst[v] = o;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}


// ---- fused GEMM1 + GEMM2, expert-granular overlap with the copy stream -------
// One persistent launch runs both contractions of a layer.  The tile space is a
// sequence of blocks of (n1 + n2) tiles: block b holds the n1 GEMM1 tiles of
// m-tile b and the n2 GEMM2 tiles of m-tile b - kLag, so a GEMM2 tile comes
// ~2 waves after the GEMM1 tiles whose H1 rows it consumes.  Dependencies are
// resolved with flags instead of kernel boundaries:
//   * GEMM1 tile of expert e waits until the copy stream's fill of e's slot
//     has landed (ready[slot - ready_base] >= need[e]; the copy stream writes
//     the fill sequence number with a stream memory op after each copy), so
//     the FFN of a layer starts on resident experts while misses stream in;
//   * GEMM2 tile of m-tile r waits until all n1 GEMM1 tiles of r stored their
//     H1 columns (done[r] == 4 * n1 epilogue-warp arrivals, release/acquire).
// Tiles are assigned round-robin (static), every CTA is resident (grid <= SMs,
// 1 CTA/SM) and a tile only waits on lower-index tiles or on copies, so the
// lowest unfinished tile can always progress: no deadlock.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t *p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_acq_rel_add(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= want (wrap-safe u32 sequence compare); a wait beyond 30 s
// means a lost copy or a broken dependency: trap (error) instead of hanging the GPU
__device__ __forceinline__ void wait_at_least(const uint32_t *p, uint32_t want, int sleep_ns) {
  if ((int)(ld_acquire_u32(p) - want) >= 0) return;
  const uint64_t t0 = global_ns();
  while ((int)(ld_acquire_u32(p) - want) < 0) {
    __nanosleep(sleep_ns);
    if (global_ns() - t0 > 30ull * 1000000000ull) {
      printf("vmm watchdog: block %d thread %d stuck on flag %p (%u < %u)\n", blockIdx.x, threadIdx.x, p,
             ld_acquire_u32(p), want);
      __trap();
    }
  }
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct FusedTile {
  bool valid, gemm2;
  int m_tile, n_tile;
};
__device__ __forceinline__ FusedTile fused_tile(int t, int n1, int n2, int MT, int lag) {
  FusedTile f;
  const int per = n1 + n2;
  const int b = t / per, j = t - b * per;
  f.gemm2 = j >= n1;
  f.m_tile = f.gemm2 ? b - lag : b;
  f.n_tile = f.gemm2 ? j - n1 : j;
  f.valid = f.m_tile >= 0 && f.m_tile < MT;
  return f;
}

// TN = N tile width (128 or 256): a 128x256 tile halves the A re-reads per FLOP
// (L2->SMEM traffic is the limiter of a 128x128 tcgen05 tile).
template <int TN>
struct FusedCfg {
  static constexpr int kStages = TN == 256 ? 4 : 6;
  static constexpr uint32_t kATile = BM * BK * 2, kBTile = TN * BK * 2;
  static constexpr uint32_t kStage = kATile + kBTile;
  static constexpr size_t kSmem = (size_t)kStages * kStage + 1024 + 256;
};

template <int TN>
__global__ void __launch_bounds__(kThreads, 1)
ffn_fused_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w13,
                 const __grid_constant__ CUtensorMap map_h1, const __grid_constant__ CUtensorMap map_w2,
                 const int32_t *__restrict__ offsets, const int32_t *__restrict__ slot_of,
                 const uint32_t *__restrict__ need, const uint32_t *ready, int ready_base, uint32_t *done, int E,
                 int H, int I, int lag, const int32_t *__restrict__ src_row, int M_total,
                 __nv_bfloat16 *__restrict__ h1, __nv_bfloat16 *__restrict__ y) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + FusedCfg<TN>::kStages * FusedCfg<TN>::kStage);
  uint64_t *empty = full + FusedCfg<TN>::kStages;
  uint64_t *tmem_full = empty + FusedCfg<TN>::kStages;   // [2]
  uint64_t *tmem_empty = tmem_full + 2;    // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);
  __shared__ int s_offs[VMM_MAX_EXPERTS + 1], s_tile_base[VMM_MAX_EXPERTS + 1], s_slots[VMM_MAX_EXPERTS];
  __shared__ uint32_t s_need[VMM_MAX_EXPERTS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e <= E; e += blockDim.x) s_offs[e] = offsets[e];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    s_slots[e] = slot_of[e];
    s_need[e] = need ? need[e] : 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      s_tile_base[e] = acc;
      acc += (s_offs[e + 1] - s_offs[e] + BM - 1) / BM;
    }
    s_tile_base[E] = acc;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_x);
    prefetch_tmap(&map_w13);
    prefetch_tmap(&map_h1);
    prefetch_tmap(&map_w2);
    for (int s = 0; s < FusedCfg<TN>::kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tmem_full[b], 1); mbar_init(&tmem_empty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int MT = s_tile_base[E];
  const int n1 = (2 * I) / TN, n2 = H / TN;
  const int total = (MT + lag) * (n1 + n2);
  const int nk1 = H / BK, nk2 = I / BK;

  if (warp == 0) {
    // TMA producer.  GEMM1 A rows come either from the permuted copy Xp (one
    // box load) or -- src_row != NULL -- straight from the token rows X through
    // tile::gather4 (each lane fetches 4 of the tile's 128 rows), which removes
    // the permute_rows pass (Xp write + re-read) entirely.
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const FusedTile f = fused_tile(t, n1, n2, MT, lag);
      if (!f.valid) continue;
      const TileInfo ti = tile_info(f.m_tile * n1, n1, s_tile_base, s_offs, s_slots, E);
      if (lane == 0) {
        const uint32_t nd = s_need[ti.expert];
        // the expert's slot fill must have landed (copy stream -> ready flag); once seen, the
        // expert's later tiles skip the flag load (only this thread reads s_need)
        if (nd) {
          wait_at_least(ready + (ti.slot - ready_base), nd, 256);
          s_need[ti.expert] = 0u;
        }
        // GEMM2: H1 rows of this m-tile complete (all GEMM1 n-tiles stored)
        if (f.gemm2) wait_at_least(done + f.m_tile, 4u * (uint32_t)n1, 64);
        if (nd || f.gemm2) fence_proxy_async_global();
      }
      const bool gather = src_row != nullptr && !f.gemm2;
      int g[4];
      if (gather) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int p = ti.row0 + 4 * lane + j;  // rows past the layer end: any valid row (masked later)
          g[j] = __ldg(src_row + (p < M_total ? p : M_total - 1));
        }
      }
      __syncwarp();
      const CUtensorMap *ma = f.gemm2 ? &map_h1 : &map_x;
      const CUtensorMap *mb = f.gemm2 ? &map_w2 : &map_w13;
      const int nk = f.gemm2 ? nk2 : nk1;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % FusedCfg<TN>::kStages;
        unsigned char *a_dst = smem + s * FusedCfg<TN>::kStage;
        if (lane == 0) {
          if (it >= FusedCfg<TN>::kStages) mbar_wait(&empty[s], ((it / FusedCfg<TN>::kStages) - 1) & 1);
          mbar_expect_tx(&full[s], FusedCfg<TN>::kStage);
          tma_load_3d(mb, &full[s], a_dst + FusedCfg<TN>::kATile, kb * BK, f.n_tile * TN, ti.slot);
          if (!gather) tma_load_2d(ma, &full[s], a_dst, kb * BK, ti.row0);
        }
        if (gather) {
          __syncwarp();  // stage free + expect_tx posted before the gathers complete bytes
          tma_gather4(ma, &full[s], a_dst + lane * 4 * BK * 2, kb * BK, g[0], g[1], g[2], g[3]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const FusedTile f = fused_tile(t, n1, n2, MT, lag);
        if (!f.valid) continue;
        const int nk = f.gemm2 ? nk2 : nk1;
        const int b = local & 1, use = local >> 1;
        if (use > 0) mbar_wait(&tmem_empty[b], (use - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + b * TN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % FusedCfg<TN>::kStages;
          mbar_wait(&full[s], (it / FusedCfg<TN>::kStages) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * FusedCfg<TN>::kStage);
          const uint32_t b_addr = a_addr + FusedCfg<TN>::kATile;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(acc, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32), idesc_bf16(BM, TN),
                      (kb | kk) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[b]);
        ++local;
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const FusedTile f = fused_tile(t, n1, n2, MT, lag);
      if (!f.valid) continue;
      const TileInfo ti = tile_info(f.m_tile * n1, n1, s_tile_base, s_offs, s_slots, E);
      const int b = local & 1, use = local >> 1;
      ++local;
      const int row = ti.row0 + q * 32 + lane;
      mbar_wait(&tmem_full[b], use & 1);
      tc_fence_after();
      const uint32_t t_base = tmem + b * TN + ((uint32_t)(q * 32) << 16);
      if (!f.gemm2) {
        // accumulator columns: TN/128 pairs of [64 gate | 64 up] -> 64 H1 columns each
#pragma unroll
        for (int hc = 0; hc < TN / 64; ++hc) {
          const int pair = hc >> 1, half = hc & 1;
          float g[32], u[32];
          tmem_ld32(t_base + pair * 128 + half * 32, g);
          tmem_ld32(t_base + pair * 128 + 64 + half * 32, u);
          if (hc == TN / 64 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tmem_empty[b]);
          }
          if (row < ti.row_end) {
            uint4 *dst = reinterpret_cast<uint4 *>(h1 + (long long)row * I + f.n_tile * (TN / 2) + pair * 64 +
                                                   half * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 o;
              o.x = pack_bf16(silu(g[8 * v + 0]) * u[8 * v + 0], silu(g[8 * v + 1]) * u[8 * v + 1]);
              o.y = pack_bf16(silu(g[8 * v + 2]) * u[8 * v + 2], silu(g[8 * v + 3]) * u[8 * v + 3]);
              o.z = pack_bf16(silu(g[8 * v + 4]) * u[8 * v + 4], silu(g[8 * v + 5]) * u[8 * v + 5]);
              o.w = pack_bf16(silu(g[8 * v + 6]) * u[8 * v + 6], silu(g[8 * v + 7]) * u[8 * v + 7]);
              dst[v] = o;
            }
          }
        }
        // publish this warp's 32 H1 rows of the tile to the GEMM2 TMA readers
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) red_release_add(done + f.m_tile, 1u);
      } else {
#pragma unroll
        for (int c = 0; c < TN / 32; ++c) {
          float a[32];
          tmem_ld32(t_base + c * 32, a);
          if (c == TN / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tmem_empty[b]);
          }
          if (row < ti.row_end) {
            uint4 *dst = reinterpret_cast<uint4 *>(y + (long long)row * H + f.n_tile * TN + c * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 o;
              o.x = pack_bf16(a[8 * v + 0], a[8 * v + 1]);
              o.y = pack_bf16(a[8 * v + 2], a[8 * v + 3]);
              o.z = pack_bf16(a[8 * v + 4], a[8 * v + 5]);
              o.w = pack_bf16(a[8 * v + 6], a[8 * v + 7]);
              dst[v] = o;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TN));
  }
}

// ---- CTA-pair variant: 256 x 256 tiles with tcgen05 cta_group::2 ------------
// A cluster of 2 CTAs (one TPC) owns a 256-row x 256-column tile: each CTA
// stages its own 128 A rows and half (128 rows) of the B tile, the leader CTA
// issues M=256 N=256 pair MMAs over both CTAs' smem, and each CTA's TMEM
// receives its 128 accumulator rows.  Per FLOP this moves 1/3 less L2->SMEM
// data than the 128x256 single-CTA tile.  Same fused GEMM1/GEMM2 tile order,
// copy ready flags and H1 block counters as ffn_fused_kernel.
constexpr int BM2 = 256, TN2 = 256, kStages2 = 6;
constexpr uint32_t kHalf2 = 128 * BK * 2;  // 16 KB: 128 rows x 64 K of A or of B
constexpr uint32_t kStage2 = 2 * kHalf2;
// epilogue staging for the TMA stores: per epilogue warp two 2 KB buffers of
// 32 rows x 32 bf16 columns (SWIZZLE_64B), after the stage ring
constexpr uint32_t kStg2 = 4 * 2 * 2048;
constexpr size_t kSmem2 = (size_t)kStages2 * kStage2 + kStg2 + 1024 + 256;

// Static persistent schedule: wave w hands tiles [w*ncl, (w+1)*ncl) to the ncl
// clusters, rotated by one cluster per wave.  Without the rotation cluster c
// would see only the N-tiles j = (c + w*ncl) mod (n1+n2) -- with ncl = 74 and
// n1+n2 = 14 only 7 of the 14 (one parity) -- so half of every M-tile's GEMM1
// tiles ran on one group of clusters and the GEMM2 tiles waited on the slower
// group.  With the rotation every cluster cycles through all N-tiles.
__device__ __forceinline__ int pair_sched(int w, int cid, int ncl) { return w * ncl + (cid + w) % ncl; }

// tile_base[i] = first m-tile of the i-th expert in walk order (order[i]; identity by default)
__device__ __forceinline__ TileInfo pair_tile_info(int m_tile, const int *tile_base, const int *offs, const int *slots,
                                                   const int *order, int E) {
  TileInfo ti;
  int lo = 0, hi = E - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_base[mid] <= m_tile) lo = mid; else hi = mid - 1;
  }
  while (lo + 1 < E && tile_base[lo + 1] <= m_tile) ++lo;
  const int e = order[lo];
  ti.expert = e;
  ti.row0 = offs[e] + (m_tile - tile_base[lo]) * BM2;
  ti.row_end = offs[e + 1];
  ti.slot = slots[e];
  ti.n_tile = 0;
  return ti;
}

// GATHER: GEMM1's A rows are gathered straight from the token rows x (one row
// per gather thread, 8 x 16-byte cp.async per k-block into the SW128 layout)
// instead of TMA box loads of a permuted copy -- no permute pass over HBM.
// Bit-identical, but measured 2.6x slower than permute + TMA on B200 (25.6 vs
// 9.9 ms at 1.25M rows: scattered 128-byte row pieces, ~3 stages in flight per
// thread), so it is opt-in (VMM_FFN_GATHER=1) and kept as the measured
// alternative.
// Warps 6..9 gather and publish each stage to the leader's full barrier.
template <bool GATHER>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GATHER ? kThreads + 128 : kThreads, 1)
ffn_pair_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w13,
                const __grid_constant__ CUtensorMap map_h1, const __grid_constant__ CUtensorMap map_w2,
                const __grid_constant__ CUtensorMap map_h1s, const __grid_constant__ CUtensorMap map_ys,
                const int32_t *__restrict__ offsets, const int32_t *__restrict__ slot_of,
                const uint32_t *__restrict__ need, const uint32_t *ready, int ready_base, uint32_t *done, int E, int H,
                int I, int lag, const __nv_bfloat16 *__restrict__ xg, const int32_t *__restrict__ src_row,
                int M_total, __nv_bfloat16 *__restrict__ h1, __nv_bfloat16 *__restrict__ y, int discard_h1,
                int l2_hints, const int32_t *__restrict__ walk_order) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *stg = smem + kStages2 * kStage2;
  uint64_t *full = reinterpret_cast<uint64_t *>(stg + kStg2);
  uint64_t *empty = full + kStages2;
  uint64_t *tmem_full = empty + kStages2;  // [2]
  uint64_t *tmem_empty = tmem_full + 2;    // [2] (the leader's counts 8 epilogue warps of the pair)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);
  __shared__ int s_offs[VMM_MAX_EXPERTS + 1], s_tile_base[VMM_MAX_EXPERTS + 1], s_slots[VMM_MAX_EXPERTS];
  __shared__ int s_order[VMM_MAX_EXPERTS];
  __shared__ uint32_t s_need[VMM_MAX_EXPERTS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  for (int e = threadIdx.x; e <= E; e += blockDim.x) s_offs[e] = offsets[e];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    s_slots[e] = slot_of[e];
    s_need[e] = need ? need[e] : 0u;
    s_order[e] = walk_order ? walk_order[e] : e;  // expert walk order (a permutation of [0, E))
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < E; ++i) {
      const int e = s_order[i];
      s_tile_base[i] = acc;
      acc += (s_offs[e + 1] - s_offs[e] + BM2 - 1) / BM2;
    }
    s_tile_base[E] = acc;
  }
  if (warp == 0 && lane == 0) {
    if (!GATHER) prefetch_tmap(&map_x);  // (gather mode passes no A map for GEMM1)
    prefetch_tmap(&map_w13);
    prefetch_tmap(&map_h1);
    prefetch_tmap(&map_w2);
    // full: the leader producer's expect_tx arrival (+ the two CTAs' gather relays)
    for (int s = 0; s < kStages2; ++s) { mbar_init(&full[s], GATHER ? 9 : 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tmem_full[b], 1); mbar_init(&tmem_empty[b], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // both CTAs: the pair allocation (same columns in each CTA's TMEM)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * TN2));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated before any cross-CTA use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int MT = s_tile_base[E];
  const int n1 = (2 * I) / TN2, n2 = H / TN2;
  const int total = (MT + lag) * (n1 + n2);
  const int nk1 = H / BK, nk2 = I / BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
#ifdef VMM_FFN_PROF
  unsigned long long _pacc[24] = {};
  const long long _prof_k0 = clock64();
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][10] = global_ns();
#endif

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int wv = 0, t = pair_sched(0, cid, ncl); wv * ncl < total; t = pair_sched(++wv, cid, ncl)) {
        if (t >= total) continue;
        const FusedTile f = fused_tile(t, n1, n2, MT, lag);
        if (!f.valid) continue;
        const TileInfo ti = pair_tile_info(f.m_tile, s_tile_base, s_offs, s_slots, s_order, E);
        const uint32_t nd = s_need[ti.expert];
        {
          PROF_T0();
          if (nd) {  // once seen, the expert's later tiles skip the flag load (only this thread reads s_need)
            wait_at_least(ready + (ti.slot - ready_base), nd, 256);
            s_need[ti.expert] = 0u;
          }
#ifdef VMM_FFN_PROF
          if (f.gemm2) {
            const uint32_t v0 = ld_acquire_u32(done + f.m_tile);
            if ((int)(v0 - 8u * (uint32_t)n1) < 0) _pacc[6] += 1;
          }
#endif
#ifdef VMM_FFN_PROF
          if (f.gemm2 && !(g_ffn_prof_mode & 1)) wait_at_least(done + f.m_tile, 8u * (uint32_t)n1, 64);
#else
          if (f.gemm2) wait_at_least(done + f.m_tile, 8u * (uint32_t)n1, 64);
#endif
          PROF_ADD(0);
        }
        if (nd || f.gemm2) fence_proxy_async_global();
        const CUtensorMap *ma = f.gemm2 ? &map_h1 : &map_x;
        const CUtensorMap *mb = f.gemm2 ? &map_w2 : &map_w13;
        const int nk = f.gemm2 ? nk2 : nk1;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages2;
          if (it >= kStages2) {
            PROF_T0();
            mbar_wait_watchdog(&empty[s], ((it / kStages2) - 1) & 1);
            PROF_ADD(1);
          }
          unsigned char *a_dst = smem + s * kStage2;
          const bool a_tma = !GATHER || f.gemm2;
          // both CTAs' TMA bytes land on the leader's barrier
          if (leader) mbar_expect_tx(&full[s], a_tma ? 2 * kStage2 : 2 * kHalf2);
          const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
          if (a_tma) tma_load_2d_cg2(ma, fb, a_dst, kb * BK, ti.row0 + 128 * (int)rank);
          tma_load_3d_cg2(mb, fb, a_dst + kHalf2, kb * BK, f.n_tile * TN2 + 128 * (int)rank, ti.slot);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int it = 0, local = 0;
      for (int wv = 0, t = pair_sched(0, cid, ncl); wv * ncl < total; t = pair_sched(++wv, cid, ncl)) {
        if (t >= total) continue;
        const FusedTile f = fused_tile(t, n1, n2, MT, lag);
        if (!f.valid) continue;
        const int nk = f.gemm2 ? nk2 : nk1;
        const int b = local & 1, use = local >> 1;
        if (use > 0) {
          PROF_T0();
          mbar_wait_watchdog(&tmem_empty[b], (use - 1) & 1);
          PROF_ADD(2);
        }
        tc_fence_after();
        const uint32_t acc = tmem + b * TN2;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages2;
          {
            PROF_T0();
            mbar_wait_watchdog(&full[s], (it / kStages2) & 1);
            PROF_ADD(f.gemm2 ? 4 : 3);
#ifdef VMM_FFN_PROF
            _pacc[f.gemm2 ? 9 : 8] += 1;
#endif
          }
          if (GATHER) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * kStage2);
          const uint32_t b_addr = a_addr + kHalf2;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_cg2(acc, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32), idesc_bf16(BM2, TN2),
                          (kb | kk) != 0);
          umma_commit_mc2(&empty[s]);
        }
        umma_commit_mc2(&tmem_full[b]);
        ++local;
      }
    }
    __syncwarp();
  } else if (GATHER && warp >= 6 && warp < 10) {
    // gather: thread t owns row t of this CTA's 128-row A half (8 x 16 B per k-block) via cp.async
    // groups; a stage's completion is published per warp (wait_group, proxy fence, lane 0 arrives on
    // the leader's full barrier: 4 warps x 2 CTAs + the producer's expect_tx arrival).  kGD stages
    // stay in flight per thread (kGD < kStages2, so a blocking empty wait never waits on a stage
    // this warp has not published yet).
    constexpr int kGD = 4;
    const int t = threadIdx.x - 192;
    int it = 0, pend[kGD + 1], np = 0;
    auto publish = [&](int ps) {
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&full[ps]), 0));
    };
    auto flush_to = [&](int keep) {  // publish all but the newest `keep` pending stages
      while (np > keep) {
        if (keep == 4) asm volatile("cp.async.wait_group 4;" ::: "memory");
        else if (keep == 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
        else if (keep == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
        else if (keep == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        publish(pend[0]);
        for (int i = 1; i < np; ++i) pend[i - 1] = pend[i];
        --np;
      }
    };
    for (int wv = 0, tt = pair_sched(0, cid, ncl); wv * ncl < total; tt = pair_sched(++wv, cid, ncl)) {
      if (tt >= total) continue;
      const FusedTile f = fused_tile(tt, n1, n2, MT, lag);
      if (!f.valid) continue;
      if (f.gemm2) {  // no gather: publish the stages after their previous round was consumed
        for (int kb = 0; kb < nk2; ++kb, ++it) {
          const int s = it % kStages2;
          if (it >= kStages2) mbar_wait_watchdog(&empty[s], ((it / kStages2) - 1) & 1);
          if (np == kGD) flush_to(kGD - 1);
          pend[np++] = s;
          asm volatile("cp.async.commit_group;" ::: "memory");  // empty group keeps the group count aligned
        }
        continue;
      }
      const TileInfo ti = pair_tile_info(f.m_tile, s_tile_base, s_offs, s_slots, s_order, E);
      // warp gw4 owns local rows [32 gw4, +32); each cp.async instruction covers 4 rows x 128 B
      // (8 lanes per row: coalesced 128-byte pieces, 4 L1 wavefronts instead of 32)
      const int gw4 = t >> 5;
      const int r = ti.row0 + 128 * (int)rank + gw4 * 32 + lane;
      const int tok_lane = src_row[r < M_total ? r : M_total - 1];
      const int c = lane & 7;
      long long src_off[8];
      uint32_t dst_off[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rl = gw4 * 32 + 4 * i + (lane >> 3);  // local row 0..127 of this CTA's half
        const int tok = __shfl_sync(0xffffffffu, tok_lane, 4 * i + (lane >> 3));
        src_off[i] = (long long)tok * H * 2 + c * 16;
        dst_off[i] = rl * 128 + ((c ^ (rl & 7)) << 4);
      }
      const char *xb = reinterpret_cast<const char *>(xg);
      for (int kb = 0; kb < nk1; ++kb, ++it) {
        const int s = it % kStages2;
        if (it >= kStages2) mbar_wait_watchdog(&empty[s], ((it / kStages2) - 1) & 1);
        const uint32_t dst = smem_u32(smem + s * kStage2);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + dst_off[i]),
                       "l"(xb + src_off[i] + (size_t)kb * BK * 2)
                       : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (np == kGD) flush_to(kGD - 1);
        pend[np++] = s;
      }
    }
    flush_to(0);
  } else if (warp >= 2 && warp < 6) {
    // epilogue: TMEM -> registers -> bf16 -> swizzled staging -> TMA store (32 rows x 32 columns per
    // store; a warp's rows that straddle the tile's expert boundary use direct stores instead)
    const int q = warp & 3;
    int local = 0;
#ifdef VMM_FFN_PROF
    const bool _nostore = (g_ffn_prof_mode & 2) != 0;
#else
    constexpr bool _nostore = false;
#endif
    uint32_t nst = 0;  // this warp's TMA stores so far (staging buffer nst & 1)
    unsigned char *stg_w = stg + q * 4096;
    // L2 priorities of the epilogue stores (hints & 1: H1 evict_last -- it is re-read by the GEMM2
    // tiles a few waves later, then discarded; hints & 2: Y evict_first -- streamed out, read by
    // the next kernel): keeps H1 resident so its lines are dropped before any write-back
    const uint64_t pol_h1 = l2_policy_evict_last(), pol_y = l2_policy_evict_first();
    auto stage_store = [&](const uint32_t (&w)[16], const CUtensorMap *map, int c0, int r0, int hint) {
      unsigned char *buf = stg_w + (nst & 1) * 2048;
      if (nst >= 2) {
        PROF_T0();
        if (lane == 0) bulk_wait_read<1>();  // the store that last read this buffer is done with it
        __syncwarp();
        if (q == 0 && lane == 0) PROF_ADD(14);
      }
      PROF_T0();
      uint4 *rowp = reinterpret_cast<uint4 *>(buf + lane * 64);
      const int sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16 B chunk ^= address bits 7..8
#pragma unroll
      for (int v = 0; v < 4; ++v) rowp[v ^ sw] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (hint == 1) tma_store_2d_hint(map, buf, c0, r0, pol_h1);
        else if (hint == 2) tma_store_2d_hint(map, buf, c0, r0, pol_y);
        else tma_store_2d(map, buf, c0, r0);
        bulk_commit();
      }
      if (q == 0 && lane == 0) PROF_ADD(13);
      ++nst;
    };
    const uint32_t te_leader[2] = {mapa_shared(smem_u32(&tmem_empty[0]), 0), mapa_shared(smem_u32(&tmem_empty[1]), 0)};
    for (int wv = 0, t = pair_sched(0, cid, ncl); wv * ncl < total; t = pair_sched(++wv, cid, ncl)) {
      if (t >= total) continue;
      const FusedTile f = fused_tile(t, n1, n2, MT, lag);
      if (!f.valid) continue;
      const TileInfo ti = pair_tile_info(f.m_tile, s_tile_base, s_offs, s_slots, s_order, E);
      const int b = local & 1, use = local >> 1;
      ++local;
      const int r_w0 = ti.row0 + 128 * (int)rank + q * 32;
      const int row = r_w0 + lane;
      const bool tma_rows = r_w0 + 32 <= ti.row_end;  // all 32 rows of this warp inside the tile's expert
      {
        PROF_T0();
        mbar_wait_watchdog(&tmem_full[b], use & 1);
        if (q == 0 && lane == 0) PROF_ADD(5);
      }
      tc_fence_after();
#ifdef VMM_FFN_PROF
      const long long _tile_t0 = clock64();
#endif
      const uint32_t t_base = tmem + b * TN2 + ((uint32_t)(q * 32) << 16);
      if (!f.gemm2) {
#pragma unroll
        for (int hc = 0; hc < TN2 / 64; ++hc) {
          const int pair = hc >> 1, half = hc & 1;
          uint32_t g[32], u[32];
          tmem_ld32_nowait(t_base + pair * 128 + half * 32, g);
          tmem_ld32_nowait(t_base + pair * 128 + 64 + half * 32, u);
          {
            PROF_T0();
            tmem_wait_ld();
            if (q == 0 && lane == 0) PROF_ADD(15);
          }
          if (hc == TN2 / 64 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed_cluster(te_leader[b]);
          }
          uint32_t w[16];
#pragma unroll
          for (int e2 = 0; e2 < 16; ++e2) {
            const float g0 = __uint_as_float(g[2 * e2]), g1 = __uint_as_float(g[2 * e2 + 1]);
            w[e2] = pack_bf16(silu(g0) * __uint_as_float(u[2 * e2]), silu(g1) * __uint_as_float(u[2 * e2 + 1]));
          }
          const int c0 = f.n_tile * (TN2 / 2) + pair * 64 + half * 32;
          if (_nostore) {
          } else if (tma_rows) {
            stage_store(w, &map_h1s, c0, r_w0, l2_hints & 1);
          } else if (row < ti.row_end) {
            uint4 *dst = reinterpret_cast<uint4 *>(h1 + (long long)row * I + c0);
#pragma unroll
            for (int v = 0; v < 4; ++v) dst[v] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
          }
        }
        // H1 block counter: this warp's rows are written (TMA stores complete, generic stores fenced)
        {
          PROF_T0();
          if (tma_rows && lane == 0) bulk_wait<0>();
          fence_proxy_async_global();
          if (!tma_rows) __threadfence();
          __syncwarp();
          if (lane == 0) red_release_add(done + f.m_tile, 1u);
          if (q == 0 && lane == 0) PROF_ADD(12);
        }
      } else {
#pragma unroll
        for (int c2 = 0; c2 < TN2 / 32; c2 += 2) {  // two 32-column loads per TMEM wait
          uint32_t a[2][32];
          tmem_ld32_nowait(t_base + c2 * 32, a[0]);
          tmem_ld32_nowait(t_base + c2 * 32 + 32, a[1]);
          {
            PROF_T0();
            tmem_wait_ld();
            if (q == 0 && lane == 0) PROF_ADD(15);
          }
          if (c2 == TN2 / 32 - 2) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed_cluster(te_leader[b]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t w[16];
#pragma unroll
            for (int e2 = 0; e2 < 16; ++e2)
              w[e2] = pack_bf16(__uint_as_float(a[h][2 * e2]), __uint_as_float(a[h][2 * e2 + 1]));
            const int c0 = f.n_tile * TN2 + (c2 + h) * 32;
            if (_nostore) {
            } else if (tma_rows) {
              stage_store(w, &map_ys, c0, r_w0, l2_hints & 2);
            } else if (row < ti.row_end) {
              uint4 *dst = reinterpret_cast<uint4 *>(y + (long long)row * H + c0);
#pragma unroll
              for (int v = 0; v < 4; ++v) dst[v] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
            }
          }
        }
        // H1 is dead once every GEMM2 tile of this m-tile has consumed it (its accumulator is
        // complete, so its TMA loads of H1 landed): the last of the 8 * n2 epilogue warps drops
        // the m-tile's H1 rows from L2 without a write-back (discard.global.L2), so the dirty
        // H1 lines never reach DRAM.  The arrivals share the m-tile's GEMM1 counter in its high
        // half (GEMM2 tiles only run once the low half reached 8 * n1).  Only the tile's own
        // rows [row0, row_end) are dropped: rows past row_end belong to the next expert.
        if (discard_h1) {
          __syncwarp();
          uint32_t old = 0;
          if (lane == 0) old = atom_acq_rel_add(done + f.m_tile, 1u << 16);
          old = __shfl_sync(0xffffffffu, old, 0);
          if ((old >> 16) == 8u * (uint32_t)n2 - 1u) {
            const int r_end = ti.row_end < ti.row0 + BM2 ? ti.row_end : ti.row0 + BM2;
            const char *b0 = reinterpret_cast<const char *>(h1 + (long long)ti.row0 * I);
            const long long n_lines = (long long)(r_end - ti.row0) * I * 2 / 128;
            for (long long i = lane; i < n_lines; i += 32)
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(b0 + i * 128) : "memory");
          }
        }
      }
#ifdef VMM_FFN_PROF
      if (q == 0 && lane == 0) _pacc[f.gemm2 ? 17 : 16] += (unsigned long long)(clock64() - _tile_t0);
      if (q == 0 && lane == 0) _pacc[f.gemm2 ? 19 : 18] += 1;
#endif
    }
    if (lane == 0) bulk_wait<0>();  // staging reads and Y writes complete before the CTA exits
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
#ifdef VMM_FFN_PROF
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][7] = (unsigned long long)(clock64() - _prof_k0);
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][11] = global_ns();
  for (int j = 0; j < 24; ++j)
    if (_pacc[j] && j != 10 && j != 11) atomicAdd(&g_ffn_prof[blockIdx.x][j], _pacc[j]);
#endif
  cluster_sync_all();  // every pair MMA into either CTA has been consumed before TMEM is freed
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TN2));
  }
}

// ---- decode-sized batches: weight-streaming SwiGLU on CUDA cores -----------
// With <= kSkinnyRows rows in the whole layer (one decode token: k rows) the
// tensor-core tiles would be >90% padding and a 128x128 tile loop per expert is
// latency-bound.  Instead every warp owns one output feature of one expert and
// streams that feature's weight rows once (16-byte vector loads, coalesced),
// dotting them with the expert's few token rows held in L1/L2.  HBM-bound on
// the demanded experts' weights, spread over all SMs.
constexpr int kSkinnyRows = 16;

// One persistent launch (one 512-thread CTA per SM, all co-resident) runs both
// phases, separated by a grid-wide barrier:
//   phase 1: work item = (active expert, output feature f): its gate and up
//            rows of W13 (2 x 4 KB at H=2048), dotted with the expert's token
//            rows -> H1 = SiLU(g) * u;
//   phase 2: work item = (active expert, 4 output columns): 4 rows of W2
//            (4 x 1.5 KB), dotted with the expert's H1 rows -> Y.
// Each lane issues all of its 16-byte loads of an item (NW rows x SEG chunks)
// before touching any, so every warp keeps 6-8 KB of weights in flight and 16
// warps per SM cover the HBM latency; the items of a phase stream through the
// active experts' weights exactly once.
constexpr int kRC = 4;  // token rows per pass (an expert has one row per decode token)

__device__ __forceinline__ void bf16x8_fma(const uint4 &w, const uint4 &x, float &acc) {
  const __nv_bfloat16 *wh = reinterpret_cast<const __nv_bfloat16 *>(&w);
  const __nv_bfloat16 *xh = reinterpret_cast<const __nv_bfloat16 *>(&x);
#pragma unroll
  for (int q = 0; q < 8; ++q) acc = fmaf(__bfloat162float(xh[q]), __bfloat162float(wh[q]), acc);
}

// acc[r][i] = <x row r, weight row i> (lane partials reduced over the warp) for
// NW weight rows of row_vec uint4; x rows read coherently (phase 2 reads H1
// written earlier in the same launch)
template <int NW, int SEG>
__device__ __forceinline__ void warp_dot(const uint4 *const (&w)[NW], int row_vec, const uint4 *x, int x_stride,
                                         int nrows, float (&acc)[kRC][NW]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < kRC; ++r)
#pragma unroll
    for (int i = 0; i < NW; ++i) acc[r][i] = 0.f;
  for (int s0 = 0; s0 < row_vec; s0 += 32 * SEG) {
    uint4 a[NW][SEG];
#pragma unroll
    for (int i = 0; i < NW; ++i)
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        const int c = s0 + lane + 32 * u;
        if (c < row_vec) a[i][u] = __ldg(w[i] + c);
      }
#pragma unroll
    for (int r = 0; r < kRC; ++r) {
      if (r < nrows) {
#pragma unroll
        for (int u = 0; u < SEG; ++u) {
          const int c = s0 + lane + 32 * u;
          if (c < row_vec) {
            const uint4 xv = __ldcg(x + (long long)r * x_stride + c);
#pragma unroll
            for (int i = 0; i < NW; ++i) bf16x8_fma(a[i][u], xv, acc[r][i]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kRC; ++r)
#pragma unroll
    for (int i = 0; i < NW; ++i)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[r][i] += __shfl_xor_sync(0xffffffffu, acc[r][i], o);
}

constexpr int kSkinnyThreads = 512;

// A decode layer's slot table and fill sequences passed BY VALUE (2 KB of kernel parameters,
// captured at launch): no per-layer upload in the compute stream
struct SkinnyRows {
  int32_t slot[VMM_MAX_EXPERTS];
  uint32_t need[VMM_MAX_EXPERTS];
  int by_value, has_need;
};

__global__ void __launch_bounds__(kSkinnyThreads, 1)
skinny_ffn_kernel(const __nv_bfloat16 *__restrict__ xp, const int32_t *__restrict__ offsets, int E,
                  const int32_t *__restrict__ slot_of, const __nv_bfloat16 *__restrict__ w13,
                  const __nv_bfloat16 *__restrict__ w2, long long stride, int H, int I, const uint32_t *need,
                  const uint32_t *ready, int ready_base, unsigned int *grid_bar, unsigned int bar_target,
                  __nv_bfloat16 *h1, __nv_bfloat16 *__restrict__ y, const __grid_constant__ SkinnyRows rows) {
  __shared__ int s_act[kSkinnyRows], s_r0[kSkinnyRows], s_r1[kSkinnyRows], s_slot[kSkinnyRows];
  __shared__ uint32_t s_need[kSkinnyRows];
  __shared__ int s_nact;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef VMM_FFN_PROF
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][20] = global_ns();
#endif
  if (warp == 0) {  // active experts in ascending id order (at most M_total <= 16 of them)
    int seen = 0;
    for (int c0 = 0; c0 < E; c0 += 32) {
      const int e = c0 + lane;
      const bool act = e < E && offsets[e + 1] > offsets[e];
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      if (act) {
        const int j = seen + __popc(bal & ((1u << lane) - 1u));
        if (j < kSkinnyRows) {
          s_act[j] = e;
          s_r0[j] = offsets[e];
          s_r1[j] = offsets[e + 1];
        }
      }
      seen += __popc(bal);
    }
    if (lane == 0) s_nact = seen < kSkinnyRows ? seen : kSkinnyRows;
    __syncwarp();
    // the active experts' slots and fill sequences, read once per CTA (from the by-value
    // parameter block when the executor passes the host rows, else from device rows)
    if (lane < (seen < kSkinnyRows ? seen : kSkinnyRows)) {
      const int e = s_act[lane];
      s_slot[lane] = rows.by_value ? rows.slot[e] : slot_of[e];
      s_need[lane] = rows.by_value ? (rows.has_need ? rows.need[e] : 0u) : (need ? need[e] : 0u);
    }
  }
  __syncthreads();
  const int nact = s_nact;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp, nwarps = gridDim.x * (blockDim.x >> 5);
  // phase 1: gate/up
  const int rv1 = H / 8;
  for (int it = gw; it < nact * I; it += nwarps) {
    const int j = it / I, f = it - j * I;
    if (s_need[j] && lane == 0) wait_at_least(ready + (s_slot[j] - ready_base), s_need[j], 128);
    __syncwarp();
    const __nv_bfloat16 *w = w13 + (long long)s_slot[j] * stride;
    const int grow = (f >> 6) * 128 + (f & 63);  // interleaved 64|64 gate/up blocks
    const uint4 *rows[2] = {reinterpret_cast<const uint4 *>(w + (long long)grow * H),
                            reinterpret_cast<const uint4 *>(w + (long long)(grow + 64) * H)};
    for (int m0 = s_r0[j]; m0 < s_r1[j]; m0 += kRC) {
      float acc[kRC][2];
      warp_dot<2, 8>(rows, rv1, reinterpret_cast<const uint4 *>(xp + (long long)m0 * H), rv1,
                     min(kRC, s_r1[j] - m0), acc);
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < kRC; ++r)
          if (m0 + r < s_r1[j]) h1[(long long)(m0 + r) * I + f] = __float2bfloat16(silu(acc[r][0]) * acc[r][1]);
    }
  }
  // grid-wide barrier (all CTAs co-resident: one per SM): H1 complete before phase 2
  __threadfence();
  __syncthreads();
#ifdef VMM_FFN_PROF
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][21] = global_ns();
#endif
  if (threadIdx.x == 0) {
    atomicAdd(grid_bar, 1u);
    wait_at_least(grid_bar, bar_target, 32);
  }
  __syncthreads();
#ifdef VMM_FFN_PROF
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][22] = global_ns();
#endif
  // phase 2: down projection, 4 output columns per item
  const int rv2 = I / 8;
  const int ncol4 = H / 4;
  for (int it = gw; it < nact * ncol4; it += nwarps) {
    const int j = it / ncol4, n = 4 * (it - j * ncol4);
    const __nv_bfloat16 *w = w2 + (long long)s_slot[j] * stride;
    const uint4 *rows[4] = {reinterpret_cast<const uint4 *>(w + (long long)(n + 0) * I),
                            reinterpret_cast<const uint4 *>(w + (long long)(n + 1) * I),
                            reinterpret_cast<const uint4 *>(w + (long long)(n + 2) * I),
                            reinterpret_cast<const uint4 *>(w + (long long)(n + 3) * I)};
    for (int m0 = s_r0[j]; m0 < s_r1[j]; m0 += kRC) {
      float acc[kRC][4];
      warp_dot<4, 4>(rows, rv2, reinterpret_cast<const uint4 *>(h1 + (long long)m0 * I), rv2,
                     min(kRC, s_r1[j] - m0), acc);
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < kRC; ++r)
          if (m0 + r < s_r1[j]) {
            __nv_bfloat162 *dst = reinterpret_cast<__nv_bfloat162 *>(y + (long long)(m0 + r) * H + n);
            dst[0] = __floats2bfloat162_rn(acc[r][0], acc[r][1]);
            dst[1] = __floats2bfloat162_rn(acc[r][2], acc[r][3]);
          }
    }
  }
#ifdef VMM_FFN_PROF
  __syncthreads();
  if (threadIdx.x == 0) g_ffn_prof[blockIdx.x][23] = global_ns();
#endif
}

// ---- decode-sized layers on the tensor cores (swap-AB) -----------------------
// A decode layer is <= 16 rows spread over <= 16 experts: the FLOPs are nothing,
// the cost is streaming the active experts' weights (75 MB at C3) from HBM.  The
// CUDA-core kernel above streams them through the LSUs and tops out near 2 TB/s
// (each SM's outstanding-load budget).  Here the weights stream by TMA -- an
// 8-stage ring of 128-row x 64-column tiles per SM -- and tcgen05 does the
// arithmetic with the roles swapped: D[128 weight rows][16 token slots] =
// W_tile . X^T, A = the weight tile (K-major, TMA SW128), B = the expert's <= 16
// token rows staged once per tile in shared memory (zero-padded to 16), the
// accumulator 16 TMEM columns.
//   work items: GEMM1 (expert j, 128 W13 rows = 64 gate + 64 up rows of 64
//   features) -> H1 = SiLU(gate) * up; GEMM2 (expert j, 128 W2 rows = 128 output
//   columns) after all of expert j's GEMM1 items (per-expert done counters,
//   release/acquire).  CTAs [0, n1) take one GEMM1 item each when n1 < grid and
//   the rest share the GEMM2 items (their TMA rings fill with GEMM2 weights while
//   the GEMM1 CTAs run); otherwise items go round-robin in list order (GEMM1
//   first), so a CTA never waits on an item queued behind its own.
// Roles: warp 0 = TMA producer (runs ahead across items), warps 1-4 = B staging,
// the MMA issuer (warp 1 lane 0) and the epilogue (TMEM lane quarter = warp % 4).
// a ring stage holds kDecKQ consecutive 64-column k-blocks of the tile's 128 rows, loaded by ONE
// 4-D TMA box so each weight row's kDecKQ x 128 B are requested together (DRAM page locality)
#ifndef VMM_DEC_KQ
#define VMM_DEC_KQ 2
#endif
constexpr int kDecKQ = VMM_DEC_KQ;
constexpr int kDecStages = 8 / kDecKQ, kDecThreads = 160, kDecN = 16;
constexpr uint32_t kDecTile = 128 * BK * 2 * kDecKQ;  // A stage: kDecKQ x 16 KB
constexpr int kDecMaxK = 2048;               // B staging: 16 rows x K <= 2048 (64 KB)
constexpr size_t kDecSmem = (size_t)kDecStages * kDecTile + (size_t)kDecN * kDecMaxK * 2 + 64 * kDecN * 4 + 1024 + 256;

struct DecItem {
  bool g2;
  int j, t;
};
__device__ __forceinline__ DecItem dec_item(int item, int n1, int per1, int per2) {
  DecItem d;
  d.g2 = item >= n1;
  const int i = d.g2 ? item - n1 : item;
  const int per = d.g2 ? per2 : per1;
  d.j = i / per;
  d.t = i - d.j * per;
  return d;
}
// k-th item of CTA b (-1 when none): split assignment when the GEMM1 items do not fill the grid
__device__ __forceinline__ int dec_cta_item(int b, int k, int G, int n1, int nt) {
  if (n1 < G && nt > n1) {
    if (b < n1) return k == 0 ? b : -1;
    const int i = n1 + (b - n1) + k * (G - n1);
    return i < nt ? i : -1;
  }
  const int i = b + k * G;
  return i < nt ? i : -1;
}

__global__ void __launch_bounds__(kDecThreads, 1)
decode_tc_kernel(const __grid_constant__ CUtensorMap map_w13, const __grid_constant__ CUtensorMap map_w2,
                 const __nv_bfloat16 *__restrict__ xp, const int32_t *__restrict__ offsets, int E,
                 const int32_t *__restrict__ slot_of, int H, int I, const uint32_t *need, const uint32_t *ready,
                 int ready_base, uint32_t *done, __nv_bfloat16 *h1, __nv_bfloat16 *__restrict__ y,
                 const __nv_bfloat16 *w13b, const __nv_bfloat16 *w2b, long long stride) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *ring = smem;
  unsigned char *bst = ring + kDecStages * kDecTile;                       // B staging (SW128 per k-block)
  float *s_gate = reinterpret_cast<float *>(bst + (size_t)kDecN * kDecMaxK * 2);  // [64][16]
  uint64_t *full = reinterpret_cast<uint64_t *>(s_gate + 64 * kDecN);
  uint64_t *empty = full + kDecStages;
  uint64_t *tfull = empty + kDecStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 1);
  __shared__ int s_act[kSkinnyRows], s_r0[kSkinnyRows], s_r1[kSkinnyRows];
  __shared__ int s_nact;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {  // active experts in ascending id order
    int seen = 0;
    for (int c0 = 0; c0 < E; c0 += 32) {
      const int e = c0 + lane;
      const bool act = e < E && offsets[e + 1] > offsets[e];
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      if (act) {
        const int j = seen + __popc(bal & ((1u << lane) - 1u));
        if (j < kSkinnyRows) {
          s_act[j] = e;
          s_r0[j] = offsets[e];
          s_r1[j] = offsets[e + 1];
        }
      }
      seen += __popc(bal);
    }
    if (lane == 0) {
      s_nact = seen < kSkinnyRows ? seen : kSkinnyRows;
      prefetch_tmap(&map_w13);
      prefetch_tmap(&map_w2);
      for (int s = 0; s < kDecStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
      mbar_init(tfull, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nact = s_nact;
  const int per1 = (2 * I) / 128, per2 = H / 128;
  const int n1 = nact * per1, nt = n1 + nact * per2;
  const int G = gridDim.x, b = blockIdx.x;
  if (warp == 0) {
    if (lane == 0) {  // producer: every item's weight tiles through the ring
      // first, bulk L2 prefetches of ALL of this CTA's weight tiles (each a contiguous range of
      // 128 weight rows): DRAM streams them in large contiguous pieces while the ring's strided
      // 128-byte box rows then mostly hit L2.  Experts still in flight are skipped.
      for (int k = 0;; ++k) {
        const int item = dec_cta_item(b, k, G, n1, nt);
        if (item < 0) break;
        const DecItem d = dec_item(item, n1, per1, per2);
        const int e = s_act[d.j];
        if (need && need[e]) continue;
        const long long K = d.g2 ? I : H;
        const char *base = reinterpret_cast<const char *>(d.g2 ? w2b : w13b) + (long long)slot_of[e] * stride * 2 +
                           (long long)d.t * 128 * K * 2;
        const long long bytes = 128 * K * 2;
        for (long long off = 0; off < bytes; off += 65536) {
          const unsigned n = (unsigned)(bytes - off < 65536 ? bytes - off : 65536);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(n) : "memory");
        }
      }
      int it = 0;
      for (int k = 0;; ++k) {
        const int item = dec_cta_item(b, k, G, n1, nt);
        if (item < 0) break;
        const DecItem d = dec_item(item, n1, per1, per2);
        const int e = s_act[d.j];
        if (need && need[e]) {
          wait_at_least(ready + (slot_of[e] - ready_base), need[e], 128);
          fence_proxy_async_global();
        }
        const CUtensorMap *map = d.g2 ? &map_w2 : &map_w13;
        const int nk = (d.g2 ? I : H) / (BK * kDecKQ);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kDecStages;
          if (it >= kDecStages) mbar_wait_watchdog(&empty[s], ((it / kDecStages) - 1) & 1);
          mbar_expect_tx(&full[s], kDecTile);
          tma_load_4d(map, &full[s], ring + s * kDecTile, 0, d.t * 128, kb * kDecKQ, slot_of[e]);
        }
      }
    }
  } else {
    const int gt = threadIdx.x - 32;  // 0..127
    const int wq = warp & 3;          // TMEM lane quarter this warp may read
    int it = 0;
    for (int k = 0;; ++k) {
      const int item = dec_cta_item(b, k, G, n1, nt);
      if (item < 0) break;
      const DecItem d = dec_item(item, n1, per1, per2);
      const int r0 = s_r0[d.j], ne = s_r1[d.j] - s_r0[d.j];
      const int K = d.g2 ? I : H, nkb = K / BK;
      if (d.g2) {  // every GEMM1 item of this expert has published its H1 columns
        if (gt == 0) wait_at_least(done + d.j, (uint32_t)per1, 64);
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      // B: the expert's rows (zero-padded to 16), one SW128 K-major 16 x 64 block per k-block
      const uint4 *src = reinterpret_cast<const uint4 *>(d.g2 ? h1 : xp);
      const int rv = K / 8;
      for (int idx = gt; idx < kDecN * rv; idx += 128) {
        const int r = idx / rv, cc = idx - r * rv;  // row, 16-byte chunk along K
        const int kb = cc >> 3, c = cc & 7;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < ne) v = d.g2 ? __ldcg(src + (long long)(r0 + r) * rv + cc) : __ldg(src + (long long)(r0 + r) * rv + cc);
        *reinterpret_cast<uint4 *>(bst + kb * (kDecN * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = v;
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (gt == 0) {  // MMA issuer
        tc_fence_after();
        for (int ks = 0; ks < nkb / kDecKQ; ++ks, ++it) {
          const int s = it % kDecStages;
          mbar_wait_watchdog(&full[s], (it / kDecStages) & 1);
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < kDecKQ; ++q) {
            const int kb = ks * kDecKQ + q;
            const uint32_t a_addr = smem_u32(ring + s * kDecTile + q * (128 * BK * 2));
            const uint32_t b_addr = smem_u32(bst + kb * (kDecN * 128));
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_bf16(tmem, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32), idesc_bf16(128, kDecN),
                        (kb | kk) != 0);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(tfull);
      }
      mbar_wait_watchdog(tfull, k & 1);
      tc_fence_after();
      uint32_t v[16];
      tmem_ld16_nowait(tmem + ((uint32_t)(32 * wq) << 16), v);
      tmem_wait_ld();
      const int row = 32 * wq + lane;  // weight row within the tile
      if (!d.g2) {
        if (row < 64)
#pragma unroll
          for (int n = 0; n < kDecN; ++n) s_gate[row * kDecN + n] = __uint_as_float(v[n]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (row >= 64) {
          const int f = d.t * 64 + row - 64;
          for (int n = 0; n < ne; ++n)
            h1[(long long)(r0 + n) * I + f] =
                __float2bfloat16(silu(s_gate[(row - 64) * kDecN + n]) * __uint_as_float(v[n]));
        }
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (gt == 0) red_release_add(done + d.j, 1u);
      } else {
        const int col = d.t * 128 + row;
        for (int n = 0; n < ne; ++n) y[(long long)(r0 + n) * H + col] = __float2bfloat16(__uint_as_float(v[n]));
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // TMEM, B staging and s_gate free for the next item
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
}

// ---- CUDA-core cross-check path -------------------------------------------
__device__ __forceinline__ int expert_of_row(const int32_t *offsets, int E, int row) {
  int lo = 0, hi = E - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (offsets[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void simt_gemm1_kernel(const __nv_bfloat16 *__restrict__ xp, const int32_t *__restrict__ offsets, int E,
                                  int M, int H, int I, const __nv_bfloat16 *__restrict__ w13, long long stride,
                                  const int32_t *__restrict__ slot_of, __nv_bfloat16 *__restrict__ h1) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)M * I) return;
  int m = (int)(idx / I), f = (int)(idx % I);
  int e = expert_of_row(offsets, E, m);
  const __nv_bfloat16 *w = w13 + (long long)slot_of[e] * stride;
  int gr = (f / 64) * 128 + (f % 64), ur = gr + 64;
  float g = 0.f, u = 0.f;
  for (int kk = 0; kk < H; ++kk) {
    float x = __bfloat162float(xp[(long long)m * H + kk]);
    g = fmaf(x, __bfloat162float(w[(long long)gr * H + kk]), g);
    u = fmaf(x, __bfloat162float(w[(long long)ur * H + kk]), u);
  }
  h1[(long long)m * I + f] = __float2bfloat16(silu(g) * u);
}

__global__ void simt_gemm2_kernel(const __nv_bfloat16 *__restrict__ h1, const int32_t *__restrict__ offsets, int E,
                                  int M, int H, int I, const __nv_bfloat16 *__restrict__ w2, long long stride,
                                  const int32_t *__restrict__ slot_of, __nv_bfloat16 *__restrict__ y) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)M * H) return;
  int m = (int)(idx / H), n = (int)(idx % H);
  int e = expert_of_row(offsets, E, m);
  const __nv_bfloat16 *w = w2 + (long long)slot_of[e] * stride;
  float a = 0.f;
  for (int kk = 0; kk < I; ++kk) a = fmaf(__bfloat162float(h1[(long long)m * I + kk]),
                                          __bfloat162float(w[(long long)n * I + kk]), a);
  y[(long long)m * H + n] = __float2bfloat16(a);
}

}  // namespace

#ifdef VMM_FFN_PROF
extern "C" int vmm_ffn_prof_mode(int mode) {
  return (int)cudaMemcpyToSymbol(g_ffn_prof_mode, &mode, sizeof(int));
}
extern "C" int vmm_ffn_prof_read(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_ffn_prof, sizeof(unsigned long long) * 256 * 24);
  if (reset) {
    static unsigned long long zero[256 * 24];
    cudaMemcpyToSymbol(g_ffn_prof, zero, sizeof(zero));
  }
  return 0;
}
#endif

// Grid barrier of the persistent decode FFN: a ring of per-device counters; each
// launch takes the next one, zeroes it on ITS stream (cudaMemsetAsync, stream-
// ordered before the kernel) and waits for target = grid.  Launches on different
// streams therefore never share a live counter (unless > kBarRing are in flight),
// a failed launch leaves no state behind, and the cooperative launch guarantees
// that all `grid` CTAs are co-resident.
static int skinny_launch(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                         const void *d_w13, const void *d_w2, long long stride, const int32_t *d_slot_of,
                         const uint32_t *d_need, const uint32_t *d_ready, int ready_base, void *d_h1, void *d_y,
                         void *stream, const int32_t *h_slot_of = nullptr, const uint32_t *h_need = nullptr) {
  if (H % 8 || I % 8 || H % 4) return vmm::fail(VMM_EVALIDATION, "decode FFN: hidden/inter must be multiples of 8");
  constexpr int kBarRing = 64;
  static unsigned int *bar[64] = {nullptr};
  static std::atomic<unsigned int> next[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return vmm::fail(VMM_ECUDA, "device index out of range");
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!bar[dev]) {
      cudaError_t e = cudaMalloc(&bar[dev], sizeof(unsigned int) * kBarRing);
      if (e == cudaSuccess) e = cudaMemset(bar[dev], 0, sizeof(unsigned int) * kBarRing);
      if (e != cudaSuccess) return vmm::cuda_status(e, "decode FFN barrier");
    }
  }
  if (!g_num_sms) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = g_num_sms;
  unsigned int *counter = bar[dev] + (next[dev].fetch_add(1u) % kBarRing);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), (cudaStream_t)stream);
  if (e != cudaSuccess) return vmm::cuda_status(e, "decode FFN barrier reset");
  const __nv_bfloat16 *xp = (const __nv_bfloat16 *)d_xp, *w13 = (const __nv_bfloat16 *)d_w13,
                      *w2 = (const __nv_bfloat16 *)d_w2;
  __nv_bfloat16 *h1 = (__nv_bfloat16 *)d_h1, *y = (__nv_bfloat16 *)d_y;
  unsigned int target = (unsigned int)grid;
  SkinnyRows rows;
  rows.by_value = h_slot_of != nullptr;
  rows.has_need = h_need != nullptr;
  if (rows.by_value) {
    for (int e = 0; e < E; ++e) {
      rows.slot[e] = h_slot_of[e];
      rows.need[e] = h_need ? h_need[e] : 0u;
    }
  }
  void *args[] = {(void *)&xp, (void *)&d_offsets, (void *)&E, (void *)&d_slot_of, (void *)&w13, (void *)&w2,
                  (void *)&stride, (void *)&H, (void *)&I, (void *)&d_need, (void *)&d_ready, (void *)&ready_base,
                  (void *)&counter, (void *)&target, (void *)&h1, (void *)&y, (void *)&rows};
  e = cudaLaunchCooperativeKernel((const void *)skinny_ffn_kernel, dim3(grid), dim3(kSkinnyThreads), args, 0,
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return vmm::cuda_status(e, "skinny_ffn_kernel (cooperative launch)");
  vmm::count_launch();
  return VMM_OK;
}

// decode-sized layer on the tensor cores; returns 1 (nothing launched) when the shape does not fit
static int decode_tc_launch(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                            const void *d_w13, const void *d_w2, long long stride, long long n_slots,
                            const int32_t *d_slot_of, const uint32_t *d_need, const uint32_t *d_ready, int ready_base,
                            void *d_h1, void *d_y, void *stream) {
  // opt-in (VMM_DECODE_TC=1, read per call): measured slower than the CUDA-core kernel at C3
  // decode sizes (43 vs 39 us for 8 experts): per-SM TMA streaming of 128-byte box rows tops
  // out near 30-40 GB/s and only the GEMM1 items' SMs stream during GEMM1
  const bool tc = std::getenv("VMM_DECODE_TC") != nullptr;
  if (!tc || H % 128 || I % 64 || H > kDecMaxK || I > kDecMaxK || M_total > kSkinnyRows || stride % 8) return 1;
  static uint32_t *done_tab[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return vmm::fail(VMM_ECUDA, "device index out of range");
  if (!done_tab[dev]) {
    cudaError_t e = cudaMalloc(&done_tab[dev], sizeof(uint32_t) * kSkinnyRows);
    if (e != cudaSuccess) return vmm::cuda_status(e, "decode FFN counters");
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem);
    if (e != cudaSuccess) return vmm::cuda_status(e, "decode FFN attr");
    attr = true;
  }
  CUtensorMap mw13, mw2;
  int st;
  // 4-D views {64 columns, rows, K / 64 column blocks, slots}: a box {64, 128, kDecKQ, 1} lands as
  // kDecKQ SW128 k-block tiles of 128 rows, one after the other
  if ((H / BK) % kDecKQ || (I / BK) % kDecKQ) return 1;
  {
    uint64_t dims[4] = {(uint64_t)BK, (uint64_t)2 * I, (uint64_t)H / BK, (uint64_t)n_slots};
    uint64_t str[3] = {(uint64_t)H * 2, (uint64_t)BK * 2, (uint64_t)stride * 2};
    uint32_t box[4] = {BK, 128, (uint32_t)kDecKQ, 1};
    if ((st = make_map(&mw13, d_w13, 4, dims, str, box))) return st;
  }
  {
    uint64_t dims[4] = {(uint64_t)BK, (uint64_t)H, (uint64_t)I / BK, (uint64_t)n_slots};
    uint64_t str[3] = {(uint64_t)I * 2, (uint64_t)BK * 2, (uint64_t)stride * 2};
    uint32_t box[4] = {BK, 128, (uint32_t)kDecKQ, 1};
    if ((st = make_map(&mw2, d_w2, 4, dims, str, box))) return st;
  }
  if (!g_num_sms) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t ce = cudaMemsetAsync(done_tab[dev], 0, sizeof(uint32_t) * kSkinnyRows, s);
  if (ce != cudaSuccess) return vmm::cuda_status(ce, "decode FFN counters memset");
  decode_tc_kernel<<<g_num_sms, kDecThreads, kDecSmem, s>>>(
      mw13, mw2, (const __nv_bfloat16 *)d_xp, d_offsets, E, d_slot_of, H, I, d_need, d_ready, ready_base,
      done_tab[dev], (__nv_bfloat16 *)d_h1, (__nv_bfloat16 *)d_y, (const __nv_bfloat16 *)d_w13,
      (const __nv_bfloat16 *)d_w2, stride);
  VMM_LAUNCH_CHECK("decode_tc_kernel");
  return VMM_OK;
}

extern "C" int vmm_grouped_swiglu(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                                  const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                                  long long n_slots, const int32_t *d_slot_of_expert, void *d_h1, void *d_y,
                                  void *stream) {
  if (M_total <= 0) return VMM_OK;
  if (H % BN || H % BK || I % 64 || I % BK || (2 * I) % BN)
    return vmm::fail(VMM_EVALIDATION, "grouped_swiglu: hidden must be a multiple of 128, inter of 64");
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  if (slot_stride % 8) return vmm::fail(VMM_EVALIDATION, "slot stride must be a multiple of 8 elements");
  if (M_total <= kSkinnyRows) {  // decode-sized layer: every expert has <= 16 rows
    const int r = decode_tc_launch(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride, n_slots,
                                   d_slot_of_expert, nullptr, nullptr, 0, d_h1, d_y, stream);
    if (r != 1) return r;
    return skinny_launch(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride, d_slot_of_expert,
                         nullptr, nullptr, 0, d_h1, d_y, stream);
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e1 = cudaFuncSetAttribute(grouped_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kSmemBytes);
    cudaError_t e2 = cudaFuncSetAttribute(grouped_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kSmemBytes);
    if (e1 != cudaSuccess) return vmm::cuda_status(e1, "ffn attr");
    if (e2 != cudaSuccess) return vmm::cuda_status(e2, "ffn attr");
    attr = true;
  }
  CUtensorMap ma1, mb1, ma2, mb2;
  int st;
  {
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)M_total};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, BM};
    if ((st = make_map(&ma1, d_xp, 2, dims, str, box))) return st;
  }
  {
    uint64_t dims[3] = {(uint64_t)H, (uint64_t)2 * I, (uint64_t)n_slots};
    uint64_t str[2] = {(uint64_t)H * 2, (uint64_t)slot_stride * 2};
    uint32_t box[3] = {BK, BN, 1};
    if ((st = make_map(&mb1, d_w13_arena, 3, dims, str, box))) return st;
  }
  {
    uint64_t dims[2] = {(uint64_t)I, (uint64_t)M_total};
    uint64_t str[1] = {(uint64_t)I * 2};
    uint32_t box[2] = {BK, BM};
    if ((st = make_map(&ma2, d_h1, 2, dims, str, box))) return st;
  }
  {
    uint64_t dims[3] = {(uint64_t)I, (uint64_t)H, (uint64_t)n_slots};
    uint64_t str[2] = {(uint64_t)I * 2, (uint64_t)slot_stride * 2};
    uint32_t box[3] = {BK, BN, 1};
    if ((st = make_map(&mb2, d_w2_arena, 3, dims, str, box))) return st;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // persistent: one CTA per SM (bounded by the largest possible tile count)
  const int max_m_tiles = (M_total + BM - 1) / BM + E;
  const int n1 = (2 * I) / BN, n2 = H / BN;
  cudaStream_t s = (cudaStream_t)stream;
  int g1 = g_num_sms < max_m_tiles * n1 ? g_num_sms : max_m_tiles * n1;
  int g2 = g_num_sms < max_m_tiles * n2 ? g_num_sms : max_m_tiles * n2;
  grouped_gemm_kernel<true><<<g1, kThreads, kSmemBytes, s>>>(ma1, mb1, d_offsets, d_slot_of_expert, E, H, n1,
                                                             (__nv_bfloat16 *)d_h1, I);
  VMM_LAUNCH_CHECK("grouped_gemm_kernel<swiglu>");
  grouped_gemm_kernel<false><<<g2, kThreads, kSmemBytes, s>>>(ma2, mb2, d_offsets, d_slot_of_expert, E, I, n2,
                                                              (__nv_bfloat16 *)d_y, H);
  VMM_LAUNCH_CHECK("grouped_gemm_kernel<down>");
  return VMM_OK;
}

// H1 is scratch: by default the CTA-pair path drops consumed H1 rows from L2 without
// writing them back, so its contents after the call are undefined.  keep != 0 keeps them
// (tests compare H1 bit for bit).
static std::atomic<int> g_keep_h1{0};
extern "C" int vmm_ffn_keep_h1(int keep) {
  g_keep_h1.store(keep ? 1 : 0, std::memory_order_relaxed);
  return VMM_OK;
}

extern "C" int vmm_grouped_swiglu_fused_ex(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H,
                                           int I, const void *d_w13_arena, const void *d_w2_arena,
                                           long long slot_stride, long long n_slots, const int32_t *d_slot_of_expert,
                                           const uint32_t *d_need, const uint32_t *d_ready, int ready_base,
                                           uint32_t *d_done, const void *d_x_rows, const int32_t *d_src_row,
                                           int n_x_rows, void *d_h1, void *d_y, const int32_t *d_order,
                                           void *stream);

// decode-sized layer (M_total <= 16) with the slot table and fill sequences given as HOST rows:
// they travel as kernel parameters, so the layer needs no upload in the compute stream
extern "C" int vmm_grouped_swiglu_decode(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                                         const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                                         const int32_t *h_slot_of_expert, const uint32_t *h_need,
                                         const uint32_t *d_ready, int ready_base, void *d_h1, void *d_y,
                                         void *stream) {
  if (M_total <= 0) return VMM_OK;
  if (M_total > kSkinnyRows) return vmm::fail(VMM_ECONTRACT, "decode FFN: at most 16 rows");
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  if (!h_slot_of_expert) return vmm::fail(VMM_ECONTRACT, "decode FFN: host slot rows required");
  if (h_need && !d_ready) return vmm::fail(VMM_ECONTRACT, "need[] without ready flags");
  return skinny_launch(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride, nullptr, nullptr,
                       d_ready, ready_base, d_h1, d_y, stream, h_slot_of_expert, h_need);
}

extern "C" int vmm_grouped_swiglu_fused(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                                        const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                                        long long n_slots, const int32_t *d_slot_of_expert, const uint32_t *d_need,
                                        const uint32_t *d_ready, int ready_base, uint32_t *d_done,
                                        const void *d_x_rows, const int32_t *d_src_row, int n_x_rows, void *d_h1,
                                        void *d_y, void *stream) {
  return vmm_grouped_swiglu_fused_ex(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride, n_slots,
                                     d_slot_of_expert, d_need, d_ready, ready_base, d_done, d_x_rows, d_src_row,
                                     n_x_rows, d_h1, d_y, nullptr, stream);
}

extern "C" int vmm_grouped_swiglu_fused_ex(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H,
                                           int I, const void *d_w13_arena, const void *d_w2_arena,
                                           long long slot_stride, long long n_slots, const int32_t *d_slot_of_expert,
                                           const uint32_t *d_need, const uint32_t *d_ready, int ready_base,
                                           uint32_t *d_done, const void *d_x_rows, const int32_t *d_src_row,
                                           int n_x_rows, void *d_h1, void *d_y, const int32_t *d_order,
                                           void *stream) {
  if (M_total <= 0) return VMM_OK;
  if (M_total <= kSkinnyRows) {  // decode-sized: persistent weight-streaming kernel (waits on flags too)
    if (d_src_row) return vmm::fail(VMM_ECONTRACT, "row gather needs the tensor-core path (M > 16)");
    if (d_need && !d_ready) return vmm::fail(VMM_ECONTRACT, "need[] without ready flags");
    const int r = decode_tc_launch(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride, n_slots,
                                   d_slot_of_expert, d_need, d_ready, ready_base, d_h1, d_y, stream);
    if (r != 1) return r;
    return skinny_launch(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride, d_slot_of_expert,
                         d_need, d_ready, ready_base, d_h1, d_y, stream);
  }
  if (d_done == nullptr)
    return d_need ? vmm::fail(VMM_ECONTRACT, "ready flags need the fused path's scratch")
         : d_src_row ? vmm::fail(VMM_ECONTRACT, "row gather needs the fused path's scratch")
                  : vmm_grouped_swiglu(d_xp, d_offsets, E, M_total, H, I, d_w13_arena, d_w2_arena, slot_stride,
                                       n_slots, d_slot_of_expert, d_h1, d_y, stream);
  if (H % BN || H % BK || I % 64 || I % BK || (2 * I) % BN)
    return vmm::fail(VMM_EVALIDATION, "grouped_swiglu: hidden must be a multiple of 128, inter of 64");
  if (E < 1 || E > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  if (slot_stride % 8) return vmm::fail(VMM_EVALIDATION, "slot stride must be a multiple of 8 elements");
  if (d_need && !d_ready) return vmm::fail(VMM_ECONTRACT, "need[] without ready flags");
  // 128x256 tiles when the widths allow (H and 2I multiples of 256), else 128x128
  static const bool force_narrow = std::getenv("VMM_FFN_TN128") != nullptr;  // A/B comparison knob
  const bool wide = !force_narrow && (H % 256 == 0) && ((2 * I) % 256 == 0);
  const int TN = wide ? 256 : 128;
  // CTA pairs (256x256 tiles) once the average expert has >= 256 rows: tensor-bound batches
  static const bool no_pair = std::getenv("VMM_FFN_NO_PAIR") != nullptr;
  const bool pair = wide && !no_pair && M_total >= 256 * E;
  const uint32_t b_rows = pair ? 128u : (uint32_t)TN;  // a pair CTA stages half of the 256-row B tile
  static bool attr = false;
  if (!attr) {
    cudaError_t e1 = cudaFuncSetAttribute(ffn_fused_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)FusedCfg<256>::kSmem);
    if (e1 == cudaSuccess)
      e1 = cudaFuncSetAttribute(ffn_fused_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)FusedCfg<128>::kSmem);
    if (e1 != cudaSuccess) return vmm::cuda_status(e1, "ffn fused attr");
    attr = true;
  }
  CUtensorMap mx, mw13, mh1, mw2;
  int st;
  if (d_src_row && !pair) {  // A rows gathered from the token rows (tile::gather4: box of one row)
    if (!d_x_rows || n_x_rows <= 0) return vmm::fail(VMM_ECONTRACT, "row gather needs the token rows");
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)n_x_rows};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, 1};
    if ((st = make_map(&mx, d_x_rows, 2, dims, str, box))) return st;
  } else if (d_src_row) {  // pair + gather: GEMM1 rows come from cp.async; the map is never used
    mx = CUtensorMap{};
  } else {
    uint64_t dims[2] = {(uint64_t)H, (uint64_t)M_total};
    uint64_t str[1] = {(uint64_t)H * 2};
    uint32_t box[2] = {BK, BM};
    if ((st = make_map(&mx, d_xp, 2, dims, str, box))) return st;
  }
  {
    uint64_t dims[3] = {(uint64_t)H, (uint64_t)2 * I, (uint64_t)n_slots};
    uint64_t str[2] = {(uint64_t)H * 2, (uint64_t)slot_stride * 2};
    uint32_t box[3] = {BK, b_rows, 1};
    if ((st = make_map(&mw13, d_w13_arena, 3, dims, str, box))) return st;
  }
  {
    uint64_t dims[2] = {(uint64_t)I, (uint64_t)M_total};
    uint64_t str[1] = {(uint64_t)I * 2};
    uint32_t box[2] = {BK, BM};
    if ((st = make_map(&mh1, d_h1, 2, dims, str, box))) return st;
  }
  {
    uint64_t dims[3] = {(uint64_t)I, (uint64_t)H, (uint64_t)n_slots};
    uint64_t str[2] = {(uint64_t)I * 2, (uint64_t)slot_stride * 2};
    uint32_t box[3] = {BK, b_rows, 1};
    if ((st = make_map(&mw2, d_w2_arena, 3, dims, str, box))) return st;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int max_m_tiles = (M_total + BM - 1) / BM + E;
  const int n1 = (2 * I) / TN, n2 = H / TN;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t ce = cudaMemsetAsync(d_done, 0, sizeof(uint32_t) * max_m_tiles, s);
  if (ce != cudaSuccess) return vmm::cuda_status(ce, "ffn done memset");
  const int grid = g_num_sms < max_m_tiles * (n1 + n2) ? g_num_sms : max_m_tiles * (n1 + n2);
  const int lag = (2 * grid + n1 + n2 - 1) / (n1 + n2);  // GEMM2 tiles ~2 waves behind their GEMM1 tiles
  if (pair) {
    static bool attr2 = false;
    if (!attr2) {
      cudaError_t e2 = cudaFuncSetAttribute(ffn_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kSmem2);
      if (e2 == cudaSuccess)
        e2 = cudaFuncSetAttribute(ffn_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2);
      if (e2 != cudaSuccess) return vmm::cuda_status(e2, "ffn pair attr");
      attr2 = true;
    }
    const int max_pair_tiles = (M_total + BM2 - 1) / BM2 + E;
    int gridp = g_num_sms & ~1;
    if (gridp > 2 * max_pair_tiles * (n1 + n2)) gridp = 2 * max_pair_tiles * (n1 + n2);
    const int ncl = gridp / 2;
    CUtensorMap mh1s, mys;  // epilogue TMA stores: 32 x 32 boxes, SWIZZLE_64B
    {
      uint64_t dims[2] = {(uint64_t)I, (uint64_t)M_total};
      uint64_t str[1] = {(uint64_t)I * 2};
      uint32_t box[2] = {32, 32};
      if ((st = make_map_swz(&mh1s, d_h1, 2, dims, str, box, 64))) return st;
    }
    {
      uint64_t dims[2] = {(uint64_t)H, (uint64_t)M_total};
      uint64_t str[1] = {(uint64_t)H * 2};
      uint32_t box[2] = {32, 32};
      if ((st = make_map_swz(&mys, d_y, 2, dims, str, box, 64))) return st;
    }
    static const int lag_waves = std::getenv("VMM_FFN_LAG") ? std::atoi(std::getenv("VMM_FFN_LAG")) : 4;
    const int lagp = (lag_waves * ncl + n1 + n2 - 1) / (n1 + n2);
    // drop consumed H1 rows from L2 without write-back unless the caller keeps H1 (vmm_ffn_keep_h1;
    // VMM_FFN_NO_DISCARD=1 keeps it for the whole process, for A/B runs)
    static const bool no_discard_env = std::getenv("VMM_FFN_NO_DISCARD") != nullptr;
    const int discard = (no_discard_env || g_keep_h1.load(std::memory_order_relaxed)) ? 0 : 1;
    // L2 priorities of the epilogue stores (bit 0: H1 evict_last, bit 1: Y evict_first; VMM_FFN_L2HINTS=n
    // for A/B runs).  Measured at R=256 (2.49M picks, ncu): DRAM 26.3 GB without discard or hints,
    // 24.7 GB with the discard, 22.5 GB with discard + both hints = 1.04x the 21.6 GB minimum
    // (weights + Xp read + Y write), same time (profiles/r02_ffn_l2_traffic.txt)
    static const int l2_hints = std::getenv("VMM_FFN_L2HINTS") ? std::atoi(std::getenv("VMM_FFN_L2HINTS")) : 3;
    if (d_src_row)
      ffn_pair_kernel<true><<<gridp, kThreads + 128, kSmem2, s>>>(
          mx, mw13, mh1, mw2, mh1s, mys, d_offsets, d_slot_of_expert, d_need, d_ready, ready_base, d_done, E, H, I,
          lagp, (const __nv_bfloat16 *)d_x_rows, d_src_row, M_total, (__nv_bfloat16 *)d_h1, (__nv_bfloat16 *)d_y,
          discard, l2_hints, d_order);
    else
      ffn_pair_kernel<false><<<gridp, kThreads, kSmem2, s>>>(
          mx, mw13, mh1, mw2, mh1s, mys, d_offsets, d_slot_of_expert, d_need, d_ready, ready_base, d_done, E, H, I,
          lagp, nullptr, nullptr, M_total, (__nv_bfloat16 *)d_h1, (__nv_bfloat16 *)d_y, discard, l2_hints, d_order);
    VMM_LAUNCH_CHECK("ffn_pair_kernel");
    return VMM_OK;
  }
  if (wide)
    ffn_fused_kernel<256><<<grid, kThreads, FusedCfg<256>::kSmem, s>>>(
        mx, mw13, mh1, mw2, d_offsets, d_slot_of_expert, d_need, d_ready, ready_base, d_done, E, H, I, lag,
        d_src_row, M_total, (__nv_bfloat16 *)d_h1, (__nv_bfloat16 *)d_y);
  else
    ffn_fused_kernel<128><<<grid, kThreads, FusedCfg<128>::kSmem, s>>>(
        mx, mw13, mh1, mw2, d_offsets, d_slot_of_expert, d_need, d_ready, ready_base, d_done, E, H, I, lag,
        d_src_row, M_total, (__nv_bfloat16 *)d_h1, (__nv_bfloat16 *)d_y);
  VMM_LAUNCH_CHECK("ffn_fused_kernel");
  return VMM_OK;
}

extern "C" int vmm_grouped_swiglu_simt(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                                       const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                                       const int32_t *d_slot_of_expert, void *d_h1, void *d_y, void *stream) {
  if (M_total <= 0) return VMM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  long long n1 = (long long)M_total * I, n2 = (long long)M_total * H;
  simt_gemm1_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, s>>>((const __nv_bfloat16 *)d_xp, d_offsets, E, M_total,
                                                                  H, I, (const __nv_bfloat16 *)d_w13_arena,
                                                                  slot_stride, d_slot_of_expert, (__nv_bfloat16 *)d_h1);
  VMM_LAUNCH_CHECK("simt_gemm1_kernel");
  simt_gemm2_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, s>>>((const __nv_bfloat16 *)d_h1, d_offsets, E, M_total,
                                                                  H, I, (const __nv_bfloat16 *)d_w2_arena,
                                                                  slot_stride, d_slot_of_expert, (__nv_bfloat16 *)d_y);
  VMM_LAUNCH_CHECK("simt_gemm2_kernel");
  return VMM_OK;
}

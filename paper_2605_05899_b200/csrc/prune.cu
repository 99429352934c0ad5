// Affinity-aware visual-token compression ("prune") -- one thread-block
// CLUSTER per request: a single CTA for batches of requests, up to 16 CTAs
// (one token slice each, distributed shared memory) for a single request.
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
//
// Selection without sorting.  Both selections only need the SET of winners
// (the outputs are id-sorted), so each is a threshold search: a radix select
// over the 64-bit order-preserving keys of the doubles (eight 8-bit digit
// passes; each CTA histograms its slice, warp-aggregated for the skewed top
// digits, and every CTA sums the cluster's histograms over DSMEM and takes
// the same digit), then the tie at the threshold is broken by id: each CTA
// counts its slice's ties, takes its quota after the lower-ranked slices
// (DSMEM prefix) and marks it with an ordered ballot scan.  The composite
// extras key (-score, -s_norm, id) is a select on score, a select on s_norm
// among the score ties (skipped when all of them fit) and the id quota.
// Per-token state (prefix expert mask, order keys of s_norm / score, flags:
// 33 B at E <= 128) lives in the slice's shared memory when it fits: the
// routes are read once, in the first pass, with every prefix layer's loads in
// flight, and the selections, target OR and marginal expansion run on chip.
// A slice that does not fit re-derives its state from the global outputs and
// the routes (core masks for the target set, the rest for their expansion):
// no cap on the tokens per request.
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kMaxCluster = 16;

// VMM_PRUNE_PROF (the prof dev build, tools/prune_prof.py): %globaltimer at the phase
// boundaries of CTA 0, thread 0
#ifdef VMM_PRUNE_PROF
__device__ unsigned long long g_prune_ts[16];
#define PRUNE_TS(i)                                                                     \
  do {                                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                          \
      unsigned long long t_;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      g_prune_ts[i] = t_;                                                               \
    }                                                                                   \
  } while (0)
#else
#define PRUNE_TS(i) \
  do {              \
  } while (0)
#endif

struct Shared {
  int warp_tot[64];
  int hist[2][256];  // double-buffered: remote CTAs read pass p while this CTA fills pass p+1
  int tot[256];
  double dlo[32], dhi[32];
  int wred[32][2];
  int sel_digit, sel_above, total;
  int hpass;  // radix passes run so far (histogram double-buffer parity)
  // cluster-visible per-CTA partials (one field per exchange: no reuse races)
  int part_nv, part_bad, part_tie0, part_tie1, part_ret, part_bad2;
  double part_lo, part_hi;
  unsigned long long part_mask[4];
  unsigned long long target[4];
  int g_nv, g_bad, g_prefix;
  double g_lo, g_hi;
};

template <class T>
__device__ __forceinline__ T *remote(cg::cluster_group &cl, T *p, int rank) {
  return cl.map_shared_rank(p, rank);
}

// cluster barrier; a one-CTA cluster (batches) only needs the block barrier, which
// also keeps L1 warm (barrier.cluster invalidates L1D)
__device__ __forceinline__ void csync(cg::cluster_group &cl) {
  if (cl.num_blocks() > 1) cl.sync();
  else __syncthreads();
}

// block-wide exclusive scan of a 0/1 flag; returns prefix, writes total to sh.total
__device__ __forceinline__ int block_scan_flag(int flag, Shared &sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned bal = __ballot_sync(0xffffffffu, flag);
  int in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) sh.warp_tot[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    int v = (lane < (int)(blockDim.x >> 5)) ? sh.warp_tot[lane] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    sh.warp_tot[32 + lane] = x - v;  // exclusive
    if (lane == 31) sh.total = x;
  }
  __syncthreads();
  int r = sh.warp_tot[32 + warp] + in_warp;
  __syncthreads();
  return r;
}

// sum over the cluster of an int partial (every thread gets the same value);
// `before` = sum over ranks < this CTA's rank
__device__ __forceinline__ int cluster_sum(cg::cluster_group &cl, Shared &sh, int *field, int *before) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
  if (warp == 0) {
    const int v = lane < C ? *remote(cl, field, lane) : 0;
    const int tot = __reduce_add_sync(0xffffffffu, v);
    const int pre = __reduce_add_sync(0xffffffffu, lane < me ? v : 0);
    if (lane == 0) { sh.total = tot; sh.g_prefix = pre; }
  }
  __syncthreads();
  const int tot = sh.total;
  if (before) *before = sh.g_prefix;
  __syncthreads();
  return tot;
}

// Radix select over the cluster: among candidate tokens of every slice, the
// largest key T with count(key >= T) >= need (1 <= need <= #candidates).
// Returns T, count(key > T) and count(key == T).  All threads of all CTAs call it.
// Early exit: once every key of the selected bucket is needed (the common case
// after 2-4 digits for continuous keys), the winners are exactly the
// candidates with key >= T, T = the bucket's lowest key; *ge_out = 1 then and
// the caller marks key >= T with no tie step.
template <class Cand, class Key>
__device__ void cluster_threshold(cg::cluster_group &cl, int t0s, int t1s, int need, Cand cand, Key key,
                                  Shared &sh, unsigned long long *T_out, int *gt_out, int *eq_out, int *ge_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int C = (int)cl.num_blocks();
  unsigned long long prefix = 0ull, pmask = 0ull;
  int remaining = need, above = 0, eq = 0, ge = 0;
  // histogram buffers alternate over every pass of every call (the pass count is the
  // same sequence in every CTA): a remote CTA may still read this CTA's previous pass
  int hp = sh.hpass;
  for (int shift = 56; shift >= 0; shift -= 8) {
    int *hist = sh.hist[hp & 1];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int b0 = t0s; b0 < t1s; b0 += blockDim.x) {  // warp-uniform trip count
      const int t = b0 + threadIdx.x;
      int dig = -1;
      if (t < t1s && cand(t)) {
        const unsigned long long k = key(t);
        if ((k & pmask) == prefix) dig = (int)((k >> shift) & 255ull);
      }
      // skewed digits are the common case (the top bytes of doubles in one binade):
      // a warp whose valid lanes agree adds once
      const unsigned act = __ballot_sync(0xffffffffu, dig >= 0);
      if (act) {
        const int d0 = __shfl_sync(0xffffffffu, dig, __ffs(act) - 1);
        if (__all_sync(0xffffffffu, dig < 0 || dig == d0)) {
          if (lane == __ffs(act) - 1) atomicAdd(&hist[d0], __popc(act));
        } else if (dig >= 0) {
          atomicAdd(&hist[dig], 1);
        }
      }
    }
    csync(cl);  // every slice's histogram of this pass is complete
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
      // all C remote loads issued before any is consumed (one DSMEM round trip, not C)
      int v[kMaxCluster];
#pragma unroll
      for (int r = 0; r < kMaxCluster; ++r) v[r] = r < C ? *remote(cl, hist + b, r) : 0;
      int sum = 0;
#pragma unroll
      for (int r = 0; r < kMaxCluster; ++r) sum += v[r];
      sh.tot[b] = sum;
    }
    __syncthreads();
    if (warp == 0) {  // lane l owns bins [8l, 8l + 8); suffix sums from the top bin down
      int c[8], own = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { c[i] = sh.tot[lane * 8 + i]; own += c[i]; }
      int suf = own;  // inclusive suffix sum over lanes >= lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += v;
      }
      const int beyond = suf - own;
      if (beyond < remaining && remaining <= suf) {  // exactly one lane
        int acc = beyond, d = lane * 8 + 7;
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          if (acc + c[i] >= remaining) { d = lane * 8 + i; break; }
          acc += c[i];
        }
        sh.sel_digit = d;
        sh.sel_above = acc;
      }
    }
    __syncthreads();
    const int d = sh.sel_digit, ab = sh.sel_above;
    eq = sh.tot[d];
    above += ab;
    remaining -= ab;
    prefix |= (unsigned long long)d << shift;
    pmask |= 255ull << shift;
    __syncthreads();  // sel_* / tot are rewritten by the next pass
    ++hp;
    if (shift > 0 && remaining == eq) {  // the whole bucket is needed: done
      ge = 1;
      break;
    }
  }
  if (threadIdx.x == 0) sh.hpass = hp;
  __syncthreads();
  *T_out = prefix;
  *gt_out = above;
  *eq_out = eq;
  *ge_out = ge;
}

// Mark, in global id order over the cluster, the first r candidates with tie(t):
// this slice's quota is r minus the ties of the lower-ranked slices.
template <class Tie, class Mark>
__device__ void cluster_mark_first(cg::cluster_group &cl, int t0s, int t1s, int r, int *part, Tie tie, Mark mark,
                                   Shared &sh) {
  int cnt = 0;
  for (int t = t0s + threadIdx.x; t < t1s; t += blockDim.x) cnt += tie(t) ? 1 : 0;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) sh.wred[threadIdx.x >> 5][0] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh.wred[w][0];
    *part = s;
  }
  csync(cl);
  int before = 0;
  cluster_sum(cl, sh, part, &before);
  const int quota = r - before;
  int done = 0;
  for (int c0 = t0s; c0 < t1s && done < quota; c0 += blockDim.x) {
    const int t = c0 + threadIdx.x;
    const int f = (t < t1s) && tie(t);
    const int pre = block_scan_flag(f, sh);
    if (f && done + pre < quota) mark(t);
    done += sh.total;
    __syncthreads();
  }
}

// 1 << s with PTX clamping: any s >= 32 (including the wrapped "negative" e - 32 i of a
// lower word) gives 0, so setting bit e of word i is branch- and select-free
__device__ __forceinline__ uint32_t bit_clamped(uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(1u), "r"(s));
  return r;
}

template <int NW32>
__device__ __forceinline__ void mask_add(uint32_t (&m)[NW32], uint32_t e) {
#pragma unroll
  for (int i = 0; i < NW32; ++i) m[i] |= bit_clamped(e - 32u * i);
}

// expert mask of one token over the P prefix layers; loads for 4 layers are issued
// before any is consumed (k == 8: two 16-byte loads per layer row).  Built in 32-bit
// words (about 2.5 instructions per id and word); an id outside [0, E) sets *bad
// (the caller reports it; its bit, if any, never reaches an output).
template <int NW>
__device__ __forceinline__ int token_mask(const int32_t *__restrict__ routes, int P, long long T, int k, int E,
                                          long long tok, uint64_t (&m)[NW]) {
  constexpr int NW32 = 2 * NW;
  uint32_t w[NW32];
#pragma unroll
  for (int i = 0; i < NW32; ++i) w[i] = 0u;
  uint32_t emax = 0u;  // unsigned max: a negative id wraps above E
  constexpr int kG = 8, kK = 8;
  if (k == kK) {
    for (int p0 = 0; p0 < P; p0 += kG) {
      int4 a[kG], b[kG];
#pragma unroll
      for (int q = 0; q < kG; ++q) {
        if (p0 + q < P) {
          const int4 *r = reinterpret_cast<const int4 *>(routes + ((long long)(p0 + q) * T + tok) * kK);
          a[q] = __ldg(r);
          b[q] = __ldg(r + 1);
        }
      }
#pragma unroll
      for (int q = 0; q < kG; ++q) {
        if (p0 + q < P) {
          const uint32_t v[8] = {(uint32_t)a[q].x, (uint32_t)a[q].y, (uint32_t)a[q].z, (uint32_t)a[q].w,
                                 (uint32_t)b[q].x, (uint32_t)b[q].y, (uint32_t)b[q].z, (uint32_t)b[q].w};
#pragma unroll
          for (int j = 0; j < kK; ++j) {
            emax = max(emax, v[j]);
            mask_add<NW32>(w, v[j]);
          }
        }
      }
    }
  } else {
    for (int p = 0; p < P; ++p) {
      const int32_t *r = routes + ((long long)p * T + tok) * k;
      for (int j = 0; j < k; ++j) {
        const uint32_t e = (uint32_t)__ldg(r + j);
        emax = max(emax, e);
        mask_add<NW32>(w, e);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i) m[i] = ((uint64_t)w[2 * i + 1] << 32) | w[2 * i];
  return emax >= (uint32_t)E;
}

// Per-token working state of the CTA's slice: 64-bit order keys of s_norm and
// score plus flags (bit0 core, bit1 keep, bit7 visual).  On chip (dynamic smem,
// 17 B/token, indexed t - t0) when the slice fits, else re-derived from the
// global outputs.
struct TokState {
  bool onchip;
  int t0;
  unsigned long long *mk;  // on chip: the token's prefix expert mask (NW words), built in phase 1
  unsigned long long *ks, *kp;
  uint8_t *f;
  const double *sn, *sc;
  const uint8_t *mod;
  uint8_t *fl;
  __device__ __forceinline__ bool vis(int t) const { return onchip ? (f[t - t0] & 0x80) != 0 : mod[t] == 0; }
  __device__ __forceinline__ uint8_t flags(int t) const { return onchip ? f[t - t0] : fl[t]; }
  __device__ __forceinline__ void set_flags(int t, uint8_t v) {
    if (onchip) f[t - t0] = v; else fl[t] = v;
  }
  __device__ __forceinline__ unsigned long long key_s(int t) const {
    return onchip ? ks[t - t0] : vmm::ord_key(sn[t]);
  }
  __device__ __forceinline__ unsigned long long key_p(int t) const {
    return onchip ? kp[t - t0] : vmm::ord_key(sc[t]);
  }
};

template <int NW>
__global__ void __launch_bounds__(256, 2)
prune_kernel(const double *__restrict__ sal, const uint8_t *__restrict__ mod, const int32_t *__restrict__ routes,
             const int32_t *__restrict__ req_off, const int32_t *__restrict__ kcore_arr,
             const int32_t *__restrict__ kkeep_arr, double alpha, double beta, long long T, int P, int k, int E,
             double lam, int cap, double *s_norm_out, double *delta_out, double *score_out, uint8_t *flags_out,
             int32_t *__restrict__ retained, int32_t *__restrict__ n_retained, uint64_t *__restrict__ target_out,
             int32_t *__restrict__ status) {
  __shared__ Shared sh;
  extern __shared__ __align__(16) unsigned char dyn[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x / C;
  const long long base = req_off[r];
  const int n_tok = req_off[r + 1] - req_off[r];
  const int slice = (n_tok + C - 1) / C;
  const int t0 = min(n_tok, me * slice), t1 = min(n_tok, t0 + slice);
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const double *s_req = sal + base;
  const uint8_t *m_req = mod + base;
  double *sn = s_norm_out + base, *dl = delta_out + base, *sc = score_out + base;
  uint8_t *fl = flags_out + base;
  TokState S;
  S.onchip = t1 - t0 <= cap;
  S.t0 = t0;
  S.mk = reinterpret_cast<unsigned long long *>(dyn);
  S.ks = S.mk + (S.onchip ? (t1 - t0) * NW : 0);
  S.kp = S.ks + (S.onchip ? t1 - t0 : 0);
  S.f = reinterpret_cast<uint8_t *>(S.kp + (S.onchip ? t1 - t0 : 0));
  S.sn = sn;
  S.sc = sc;
  S.mod = m_req;
  S.fl = fl;

  PRUNE_TS(0);
  // 1. outputs reset, visual count, saliency validation and min/max (compress.py:104-114)
  // On chip, every visual token's prefix expert mask is built here too, once: its route
  // loads (all P layers in flight, P <= 8) overlap the min/max and the core selection, and
  // the target OR / marginal expansion then read shared memory only.
  double lo = INFINITY, hi = -INFINITY;
  int nv = 0, bad = 0, ebad = 0;
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    dl[t] = qnan;
    sc[t] = qnan;
    const bool v = m_req[t] == 0;
    if (!v) sn[t] = qnan;
    if (S.onchip) S.f[t - t0] = v ? 0x80 : 0;
    else fl[t] = 0;
    if (v) {
      const double x = s_req[t];
      if (!isfinite(x) || x < 0.0) bad = 1;
      lo = fmin(lo, x);
      hi = fmax(hi, x);
      ++nv;
      if (S.onchip) {
        uint64_t m[NW];
        ebad |= token_mask<NW>(routes, P, T, k, E, base + t, m);
#pragma unroll
        for (int w = 0; w < NW; ++w) S.mk[(t - t0) * NW + w] = m[w];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  nv = __reduce_add_sync(0xffffffffu, nv);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0) { sh.dlo[warp] = lo; sh.dhi[warp] = hi; sh.wred[warp][0] = nv; sh.wred[warp][1] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = INFINITY, h = -INFINITY;
    int n = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      l = fmin(l, sh.dlo[w]);
      h = fmax(h, sh.dhi[w]);
      n += sh.wred[w][0];
      b |= sh.wred[w][1];
    }
    sh.part_lo = l; sh.part_hi = h; sh.part_nv = n; sh.part_bad = b;
    for (int w = 0; w < 4; ++w) sh.target[w] = 0ull;
    sh.hpass = 0;
  }
  csync(cl);
  if (warp == 0) {  // cluster totals (fmin/fmax and integer sums: order-independent, exact)
    double l = INFINITY, h = -INFINITY;
    int n = 0, b = 0;
    if (lane < C) {
      l = *remote(cl, &sh.part_lo, lane);
      h = *remote(cl, &sh.part_hi, lane);
      n = *remote(cl, &sh.part_nv, lane);
      b = *remote(cl, &sh.part_bad, lane);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
      h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    n = __reduce_add_sync(0xffffffffu, n);
    b = __reduce_or_sync(0xffffffffu, b);
    if (lane == 0) { sh.g_lo = l; sh.g_hi = h; sh.g_nv = n; sh.g_bad = b; }
  }
  __syncthreads();
  lo = sh.g_lo;
  hi = sh.g_hi;
  nv = sh.g_nv;
  bad = sh.g_bad;
  int k_core = 0, k_keep = 0, st = bad ? 1 : 0;
  if (!st) {
    if (kcore_arr) {
      k_core = kcore_arr[r];
      k_keep = kkeep_arr[r];
    } else {  // compress.py:151-152: floor(alpha * n_visual) -- one correctly rounded product
      k_core = (int)floor(__dmul_rn(alpha, (double)nv));
      k_keep = (int)floor(__dmul_rn(beta, (double)nv));
    }
    if (k_keep < k_core || k_core < 0) st = 3;  // compress.py:153-154
  }
  if (st) {
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) { sn[t] = qnan; fl[t] = 0; }
    if (me == 0 && threadIdx.x == 0) { status[r] = st; n_retained[r] = 0; }
    csync(cl);  // no CTA leaves while another may still read its shared memory
    return;
  }
  if (k_keep > nv) k_keep = nv;
  if (k_core > nv) k_core = nv;

  PRUNE_TS(1);
  // 2. normalised saliency
  const double span = __dsub_rn(hi, lo);
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
    if (m_req[t] == 0) {
      const double v = (hi == lo) ? 0.5 : __ddiv_rn(__dsub_rn(s_req[t], lo), span);
      sn[t] = v;
      if (S.onchip) S.ks[t - t0] = vmm::ord_key(v);
    }
  __syncthreads();

  auto is_vis = [&](int t) { return S.vis(t); };
  auto key_s = [&](int t) { return S.key_s(t); };

  PRUNE_TS(2);
  // 3. salient core: top k_core by (-s_norm, id)
  if (k_core > 0) {
    if (k_core >= nv) {
      for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
        if (S.vis(t)) S.set_flags(t, S.flags(t) | 1);
    } else {
      unsigned long long Ts;
      int gt, eq, ge;
      cluster_threshold(cl, t0, t1, k_core, is_vis, key_s, sh, &Ts, &gt, &eq, &ge);
      for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
        if (S.vis(t) && (S.key_s(t) > Ts || (ge && S.key_s(t) == Ts))) S.set_flags(t, S.flags(t) | 1);
      __syncthreads();
      auto tie = [&](int t) { return S.vis(t) && S.key_s(t) == Ts; };
      auto mark = [&](int t) { S.set_flags(t, S.flags(t) | 1); };
      if (ge) {
        // key >= Ts marked above
      } else if (k_core - gt == eq) {  // every tie fits
        for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
          if (tie(t)) mark(t);
      } else {
        cluster_mark_first(cl, t0, t1, k_core - gt, &sh.part_tie0, tie, mark, sh);
      }
    }
  }
  __syncthreads();

  PRUNE_TS(3);
  // 4. target expert set = OR of the core tokens' prefix masks, over the cluster
  {
    uint64_t acc[NW] = {};
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
      if (S.flags(t) & 1) {
        uint64_t m[NW];
        if (S.onchip) {
#pragma unroll
          for (int w = 0; w < NW; ++w) m[w] = S.mk[(t - t0) * NW + w];
        } else {
          ebad |= token_mask<NW>(routes, P, T, k, E, base + t, m);
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) acc[w] |= m[w];
      }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      unsigned lo32 = __reduce_or_sync(0xffffffffu, (unsigned)acc[w]);
      unsigned hi32 = __reduce_or_sync(0xffffffffu, (unsigned)(acc[w] >> 32));
      if (lane == 0 && (lo32 | hi32)) atomicOr(&sh.target[w], ((unsigned long long)hi32 << 32) | lo32);
    }
    __syncthreads();
    if (threadIdx.x < 4) sh.part_mask[threadIdx.x] = sh.target[threadIdx.x];
    csync(cl);
    if (warp == 0) {
      uint64_t m[4] = {0, 0, 0, 0};
      if (lane < C)
#pragma unroll
        for (int w = 0; w < NW; ++w) m[w] = *remote(cl, &sh.part_mask[w], lane);
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        unsigned lo32 = __reduce_or_sync(0xffffffffu, (unsigned)m[w]);
        unsigned hi32 = __reduce_or_sync(0xffffffffu, (unsigned)(m[w] >> 32));
        if (lane == 0) sh.target[w] = ((unsigned long long)hi32 << 32) | lo32;
      }
    }
    __syncthreads();
  }
  uint64_t tg[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) tg[w] = sh.target[w];

  PRUNE_TS(4);
  // 5. marginal expansion + score for the non-core visual tokens (compress.py:163-172)
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
    if (S.vis(t) && !(S.flags(t) & 1)) {
      uint64_t m[NW];
      if (S.onchip) {
#pragma unroll
        for (int w = 0; w < NW; ++w) m[w] = S.mk[(t - t0) * NW + w];
      } else {
        ebad |= token_mask<NW>(routes, P, T, k, E, base + t, m);
      }
      int sz = 0, out = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) { sz += __popcll(m[w]); out += __popcll(m[w] & ~tg[w]); }
      const double d = __ddiv_rn((double)out, (double)sz);
      const double p = __dsub_rn(sn[t], __dmul_rn(lam, d));
      dl[t] = d;
      sc[t] = p;
      if (S.onchip) S.kp[t - t0] = vmm::ord_key(p);
    }
  ebad = __syncthreads_or(ebad);
  if (threadIdx.x == 0) sh.part_bad2 = ebad;
  csync(cl);
  if (cluster_sum(cl, sh, &sh.part_bad2, nullptr)) {  // an expert id outside [0, E) (TraceError)
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) fl[t] = 0;
    if (me == 0 && threadIdx.x == 0) { status[r] = 4; n_retained[r] = 0; }
    csync(cl);
    return;
  }

  PRUNE_TS(5);
  // 6. extras: top (k_keep - k_core) non-core visual tokens by (-score, -s_norm, id)
  const int need = k_keep - k_core;
  auto is_rest = [&](int t) { return S.vis(t) && !(S.flags(t) & 1); };
  if (need > 0) {
    if (need >= nv - k_core) {
      for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
        if (is_rest(t)) S.set_flags(t, S.flags(t) | 2);
    } else {
      auto key_p = [&](int t) { return S.key_p(t); };
      auto mark = [&](int t) { S.set_flags(t, S.flags(t) | 2); };
      unsigned long long Tp, Ts = 0ull;
      int gtp, eqp, gep, gts = 0, eqs = 0, ges = 0;
      cluster_threshold(cl, t0, t1, need, is_rest, key_p, sh, &Tp, &gtp, &eqp, &gep);
      const int r1 = need - gtp;  // from the score ties, by s_norm
      auto tie_p = [&](int t) { return is_rest(t) && S.key_p(t) == Tp; };
      const bool all_p = gep || r1 == eqp;  // gep: every key >= Tp wins (Tp is a bucket bound)
      if (!all_p) {
        cluster_threshold(cl, t0, t1, r1, tie_p, key_s, sh, &Ts, &gts, &eqs, &ges);
      }
      for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
        if (is_rest(t)) {
          const unsigned long long kp = S.key_p(t);
          if (kp > Tp || (kp == Tp && (all_p || S.key_s(t) > Ts || (ges && S.key_s(t) == Ts)))) mark(t);
        }
      __syncthreads();
      if (!all_p && !ges) {
        const int r2 = r1 - gts;  // from the (score, s_norm) ties, by id
        auto tie_ps = [&](int t) { return tie_p(t) && S.key_s(t) == Ts; };
        if (r2 == eqs) {
          for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x)
            if (tie_ps(t)) mark(t);
        } else {
          cluster_mark_first(cl, t0, t1, r2, &sh.part_tie1, tie_ps, mark, sh);
        }
      }
    }
  }
  __syncthreads();
  if (me == 0 && threadIdx.x < NW) target_out[(long long)r * 4 + threadIdx.x] = tg[threadIdx.x];
  if (me == 0 && threadIdx.x >= NW && threadIdx.x < 4) target_out[(long long)r * 4 + threadIdx.x] = 0ull;

  PRUNE_TS(6);
  // 7. retained = keep U text, ascending request-local ids (compress.py:63-65); final flags.
  // Slice counts first, then each slice writes at its cluster prefix.
  int cnt = 0;
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    const uint8_t fs = S.flags(t);
    cnt += (m_req[t] == 1) || (fs & 3);
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) sh.wred[warp][0] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh.wred[w][0];
    sh.part_ret = s;
  }
  csync(cl);
  int before = 0;
  const int n_ret_all = cluster_sum(cl, sh, &sh.part_ret, &before);
  int n_ret = before;
  for (int c0 = t0; c0 < t1; c0 += blockDim.x) {
    const int t = c0 + threadIdx.x;
    int f = 0;
    uint8_t fo = 0;
    if (t < t1) {
      const uint8_t fs = S.flags(t);
      fo = (fs & 1) ? 3 : (fs & 2);  // core tokens are kept
      f = (m_req[t] == 1) || (fo & 2);
    }
    const int pre = block_scan_flag(f, sh);
    if (f) retained[base + n_ret + pre] = t;
    if (t < t1) fl[t] = fo | (f ? 4 : 0);
    n_ret += sh.total;
  }
  if (me == 0 && threadIdx.x == 0) { n_retained[r] = n_ret_all; status[r] = 0; }
  PRUNE_TS(7);
  csync(cl);  // DSMEM lifetime: every remote read of this CTA's partials is done
  PRUNE_TS(8);
}

// Pack the per-request retained lists into one ascending list of GLOBAL row ids
// (request r's ids + req_off[r]) and the per-request offsets into it.
__global__ void retained_pack_kernel(const int32_t *__restrict__ req_off, const int32_t *__restrict__ retained,
                                     const int32_t *__restrict__ n_retained, int R, int32_t *__restrict__ out,
                                     int32_t *__restrict__ out_off) {
  __shared__ int s_off;
  const int r = blockIdx.x;
  int acc = 0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) acc += n_retained[i];
  acc = __reduce_add_sync(0xffffffffu, acc);
  if (threadIdx.x == 0) s_off = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_off, acc);
  __syncthreads();
  const int off = s_off, n = n_retained[r], b = req_off[r];
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[off + i] = retained[b + i] + b;
  if (threadIdx.x == 0) {
    out_off[r] = off;
    if (r == R - 1) out_off[R] = off + n;
  }
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
                         const int32_t *d_req_off, const int32_t *d_k_core, const int32_t *d_k_keep, double alpha,
                         double beta, int R, int T, int P, int k, int experts, double lam, double *d_s_norm,
                         double *d_delta, double *d_score, uint8_t *d_flags, int32_t *d_retained,
                         int32_t *d_n_retained, uint64_t *d_target, int32_t *d_status, void *stream) {
  if (R <= 0) return VMM_OK;
  if (experts < 1 || experts > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "experts must lie in [1, 256]");
  if (P < 1 || k < 1) return vmm::fail(VMM_EVALIDATION, "prefix_layers must be non-empty and k >= 1");
  if ((d_k_core == nullptr) != (d_k_keep == nullptr))
    return vmm::fail(VMM_ECONTRACT, "k_core and k_keep must both be given or both be NULL");
  // one cluster per request: as many CTAs per request as keep ~148 SMs busy (16 for one
  // request, 1 for a batch of >= 148); each CTA keeps up to 4096 tokens' state on chip
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static int c_max = -1;  // VMM_PRUNE_CLUSTER: cap on the CTAs per request (tuning knob)
  if (c_max < 0) {
    const char *v = getenv("VMM_PRUNE_CLUSTER");
    c_max = v ? atoi(v) : kMaxCluster;
    if (c_max < 1 || c_max > kMaxCluster) c_max = kMaxCluster;
  }
  int C = 1;
  while (C < c_max && (long long)R * C * 2 <= num_sms) C <<= 1;
  // on-chip token state per slice: NW mask words + two order keys + flags (33 B/token at
  // E <= 128); a C3 request (2368 tokens) fits one CTA with two CTAs per SM
  const bool wide = experts > 128;
  const int cap = 2560;
  const size_t smem = (size_t)cap * (8 * (wide ? 4 : 2) + 17);
  static bool attr[2] = {false, false};
  if (!attr[wide]) {
    const void *fn = wide ? (const void *)prune_kernel<4> : (const void *)prune_kernel<2>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return vmm::cuda_status(e, "prune attr");
    attr[wide] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(R * C);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const long long TT = T;
  cudaError_t e = wide ? cudaLaunchKernelEx(&cfg, prune_kernel<4>, d_saliency, d_modality, d_routes, d_req_off,
                                            d_k_core, d_k_keep, alpha, beta, TT, P, k, experts, lam, cap, d_s_norm,
                                            d_delta, d_score, d_flags, d_retained, d_n_retained, d_target, d_status)
                       : cudaLaunchKernelEx(&cfg, prune_kernel<2>, d_saliency, d_modality, d_routes, d_req_off,
                                            d_k_core, d_k_keep, alpha, beta, TT, P, k, experts, lam, cap, d_s_norm,
                                            d_delta, d_score, d_flags, d_retained, d_n_retained, d_target, d_status);
  if (e != cudaSuccess) return vmm::cuda_status(e, "prune_kernel launch");
  VMM_LAUNCH_CHECK("prune_kernel");
  return VMM_OK;
}

extern "C" int vmm_retained_pack(const int32_t *d_req_off, const int32_t *d_retained, const int32_t *d_n_retained,
                                 int R, int32_t *d_out, int32_t *d_out_off, void *stream) {
  if (R <= 0) return VMM_OK;
  retained_pack_kernel<<<R, 256, 0, (cudaStream_t)stream>>>(d_req_off, d_retained, d_n_retained, R, d_out,
                                                            d_out_off);
  VMM_LAUNCH_CHECK("retained_pack_kernel");
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

#ifdef VMM_PRUNE_PROF
extern "C" int vmm_prune_prof_read(unsigned long long *out16) {
  return cudaMemcpyFromSymbol(out16, g_prune_ts, sizeof(g_prune_ts)) == cudaSuccess ? VMM_OK : VMM_ECUDA;
}
#endif

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
//
// Selection without sorting.  Both selections only need the SET of winners
// (the outputs are id-sorted), so each is a threshold search: a radix select
// over the 64-bit order-preserving keys of the doubles (eight 8-bit digit
// passes, shared-memory histograms with warp-aggregated adds for the skewed
// top digits), then the tie at the threshold is broken by id with one
// block-wide ordered ballot scan.  The composite extras key (-score, -s_norm,
// id) is two nested searches (score, then s_norm among the score ties) and
// the id scan.  No per-token state is kept on chip: the keys are re-read
// from the s_norm/score outputs the CTA itself wrote (L1/L2-resident), so
// there is no cap on the tokens per request.  Routes are read exactly once:
// the core tokens' masks for the target set, then every other visual
// token's mask for its marginal expansion.
#include <math.h>

#include "common.cuh"

namespace {

constexpr int kWords = VMM_MAX_EXPERTS / 64;

struct Shared {
  int warp_tot[64];
  int red[32][2];
  int hist[256];
  int sel_digit, sel_above;
  double dlo[32], dhi[32];
  unsigned long long target[kWords];
  int total, nvis, bad;
};

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

// Threshold search (radix select): among candidate tokens (cand(t) true) with
// 64-bit keys key(t), the largest T with count(key >= T) >= need (1 <= need <=
// #candidates).  Eight passes over 8-bit digits, most significant first: a
// shared-memory histogram of the candidates matching the digits fixed so far,
// then a suffix scan picks the digit holding the need-th largest key.
// Returns T and count(key > T).  All threads of the block must call it.
template <class Cand, class Key>
__device__ void block_threshold(int n_tok, int need, Cand cand, Key key, Shared &sh, unsigned long long *T_out,
                                int *gt_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long prefix = 0ull, pmask = 0ull;
  int remaining = need, above = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) sh.hist[b] = 0;
    __syncthreads();
    for (int t0 = 0; t0 < n_tok; t0 += blockDim.x) {  // warp-uniform trip count
      const int t = t0 + threadIdx.x;
      int dig = -1;
      if (t < n_tok && cand(t)) {
        const unsigned long long k = key(t);
        if ((k & pmask) == prefix) dig = (int)((k >> shift) & 255ull);
      }
      // skewed digits are the common case (the top bytes of doubles in one binade):
      // a warp whose valid lanes agree adds once
      const unsigned act = __ballot_sync(0xffffffffu, dig >= 0);
      if (act) {
        const int d0 = __shfl_sync(0xffffffffu, dig, __ffs(act) - 1);
        if (__all_sync(0xffffffffu, dig < 0 || dig == d0)) {
          if (lane == __ffs(act) - 1) atomicAdd(&sh.hist[d0], __popc(act));
        } else if (dig >= 0) {
          atomicAdd(&sh.hist[dig], 1);
        }
      }
    }
    __syncthreads();
    if (warp == 0) {  // lane l owns bins [8l, 8l + 8); suffix sums from the top bin down
      int c[8], own = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { c[i] = sh.hist[lane * 8 + i]; own += c[i]; }
      int suf = own;  // inclusive suffix sum over lanes >= lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += v;
      }
      const int beyond = suf - own;  // keys in bins of higher lanes
      if (beyond < remaining && remaining <= suf) {  // exactly one lane
        int acc = beyond, d = lane * 8 + 7;
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          if (acc + c[i] >= remaining) { d = lane * 8 + i; break; }
          acc += c[i];
        }
        sh.sel_digit = d;
        sh.sel_above = acc;  // candidates above the chosen digit at this level
      }
    }
    __syncthreads();
    const int d = sh.sel_digit, ab = sh.sel_above;
    above += ab;
    remaining -= ab;
    prefix |= (unsigned long long)d << shift;
    pmask |= 255ull << shift;
    __syncthreads();  // sel_* and hist are rewritten by the next pass
  }
  *T_out = prefix;
  *gt_out = above;
}

// Mark, in id order, the first r candidates with key == T (ties at the threshold).
template <class Tie, class Mark>
__device__ void block_mark_first(int n_tok, int r, Tie tie, Mark mark, Shared &sh) {
  int done = 0;
  for (int c0 = 0; c0 < n_tok && done < r; c0 += blockDim.x) {
    const int t = c0 + threadIdx.x;
    const int f = (t < n_tok) && tie(t);
    const int pre = block_scan_flag(f, sh);
    if (f && done + pre < r) mark(t);
    done += sh.total;
    __syncthreads();
  }
}

__device__ __forceinline__ void mask_set(uint64_t (&m)[kWords], int e) {
  const uint64_t bit = 1ull << (e & 63);
  const int w = e >> 6;
#pragma unroll
  for (int i = 0; i < kWords; ++i) m[i] |= (i == w) ? bit : 0ull;  // no dynamic register indexing
}

// expert mask of one token over the P prefix layers; loads for 4 layers are issued
// before any is consumed (k == 8: two 16-byte loads per layer row)
__device__ __forceinline__ int token_mask(const int32_t *__restrict__ routes, int P, long long T, int k, int E,
                                          long long tok, uint64_t (&m)[kWords]) {
#pragma unroll
  for (int w = 0; w < kWords; ++w) m[w] = 0;
  int bad = 0;
  constexpr int kG = 4, kK = 8;
  for (int p0 = 0; p0 < P; p0 += kG) {
    int v[kG][kK];
#pragma unroll
    for (int q = 0; q < kG; ++q) {
      const int32_t *r = routes + ((long long)(p0 + q) * T + tok) * k;
      if (p0 + q >= P) {
#pragma unroll
        for (int j = 0; j < kK; ++j) v[q][j] = -1;
      } else if (k == 8) {
        const int4 a = __ldg(reinterpret_cast<const int4 *>(r)), b = __ldg(reinterpret_cast<const int4 *>(r) + 1);
        v[q][0] = a.x; v[q][1] = a.y; v[q][2] = a.z; v[q][3] = a.w;
        v[q][4] = b.x; v[q][5] = b.y; v[q][6] = b.z; v[q][7] = b.w;
      } else {
#pragma unroll
        for (int j = 0; j < kK; ++j) v[q][j] = j < k ? __ldg(r + j) : -1;
      }
    }
#pragma unroll
    for (int q = 0; q < kG; ++q)
#pragma unroll
      for (int j = 0; j < kK; ++j) {
        const int e = v[q][j];
        if (p0 + q < P && j < k) {
          if ((unsigned)e >= (unsigned)E) bad = 1;
          else mask_set(m, e);
        }
      }
    if (k > kK)  // wide top-k: the rest of each row, scalar
      for (int q = 0; q < kG && p0 + q < P; ++q) {
        const int32_t *r = routes + ((long long)(p0 + q) * T + tok) * k;
        for (int j = kK; j < k; ++j) {
          const int e = __ldg(r + j);
          if ((unsigned)e >= (unsigned)E) bad = 1;
          else mask_set(m, e);
        }
      }
  }
  return bad;
}

// Per-token working state: 64-bit order keys of s_norm and score plus flags
// (bit0 core, bit1 keep, bit7 visual).  On chip (dynamic smem, 17 B/token)
// when the request fits `cap` tokens, else re-derived from the global outputs.
struct TokState {
  bool onchip;
  unsigned long long *ks, *kp;
  uint8_t *f;
  const double *sn, *sc;
  const uint8_t *mod;
  uint8_t *fl;
  __device__ __forceinline__ bool vis(int t) const { return onchip ? (f[t] & 0x80) != 0 : mod[t] == 0; }
  __device__ __forceinline__ uint8_t flags(int t) const { return onchip ? f[t] : fl[t]; }
  __device__ __forceinline__ void set_flags(int t, uint8_t v) {
    if (onchip) f[t] = v; else fl[t] = v;
  }
  __device__ __forceinline__ unsigned long long key_s(int t) const { return onchip ? ks[t] : vmm::ord_key(sn[t]); }
  __device__ __forceinline__ unsigned long long key_p(int t) const { return onchip ? kp[t] : vmm::ord_key(sc[t]); }
};

template <int kT>
__global__ void __launch_bounds__(kT, kT == 256 ? 3 : 1)
prune_kernel(const double *__restrict__ sal, const uint8_t *__restrict__ mod, const int32_t *__restrict__ routes,
             const int32_t *__restrict__ req_off, const int32_t *__restrict__ kcore_arr,
             const int32_t *__restrict__ kkeep_arr, double alpha, double beta, long long T, int P, int k, int E,
             double lam, int cap, double *s_norm_out, double *delta_out, double *score_out, uint8_t *flags_out,
             int32_t *__restrict__ retained, int32_t *__restrict__ n_retained, uint64_t *__restrict__ target_out,
             int32_t *__restrict__ status) {
  __shared__ Shared sh;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int r = blockIdx.x;
  const long long base = req_off[r];
  const int n_tok = req_off[r + 1] - req_off[r];
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const double *s_req = sal + base;
  const uint8_t *m_req = mod + base;
  double *sn = s_norm_out + base, *dl = delta_out + base, *sc = score_out + base;
  uint8_t *fl = flags_out + base;
  TokState S;
  S.onchip = n_tok <= cap;
  S.ks = reinterpret_cast<unsigned long long *>(dyn);
  S.kp = S.ks + (S.onchip ? n_tok : 0);
  S.f = reinterpret_cast<uint8_t *>(S.kp + (S.onchip ? n_tok : 0));
  S.sn = sn;
  S.sc = sc;
  S.mod = m_req;
  S.fl = fl;

  if (threadIdx.x < kWords) sh.target[threadIdx.x] = 0ull;

  // 1. outputs reset, visual count, saliency validation and min/max (compress.py:104-114)
  double lo = INFINITY, hi = -INFINITY;
  int nv = 0, bad = 0;
  for (int t = threadIdx.x; t < n_tok; t += kT) {
    dl[t] = qnan;
    sc[t] = qnan;
    const bool v = m_req[t] == 0;
    if (!v) sn[t] = qnan;
    if (S.onchip) S.f[t] = v ? 0x80 : 0;
    else fl[t] = 0;
    if (v) {
      const double x = s_req[t];
      if (!isfinite(x) || x < 0.0) bad = 1;
      lo = fmin(lo, x);
      hi = fmax(hi, x);
      ++nv;
    }
  }
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    nv = __reduce_add_sync(0xffffffffu, nv);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) { sh.dlo[warp] = lo; sh.dhi[warp] = hi; sh.red[warp][0] = nv; sh.red[warp][1] = bad; }
    __syncthreads();
    lo = INFINITY;
    hi = -INFINITY;
    nv = 0;
    bad = 0;
#pragma unroll 8
    for (int w = 0; w < kT / 32; ++w) {
      lo = fmin(lo, sh.dlo[w]);
      hi = fmax(hi, sh.dhi[w]);
      nv += sh.red[w][0];
      bad |= sh.red[w][1];
    }
    __syncthreads();
  }
  if (bad) {
    for (int t = threadIdx.x; t < n_tok; t += kT) { sn[t] = qnan; fl[t] = 0; }
    if (threadIdx.x == 0) { status[r] = 1; n_retained[r] = 0; }
    return;
  }
  int k_core, k_keep;
  if (kcore_arr) {
    k_core = kcore_arr[r];
    k_keep = kkeep_arr[r];
  } else {  // compress.py:151-152: floor(alpha * n_visual) -- one correctly rounded product
    k_core = (int)floor(__dmul_rn(alpha, (double)nv));
    k_keep = (int)floor(__dmul_rn(beta, (double)nv));
  }
  if (k_keep < k_core || k_core < 0) {  // compress.py:153-154
    for (int t = threadIdx.x; t < n_tok; t += kT) { sn[t] = qnan; fl[t] = 0; }
    if (threadIdx.x == 0) { status[r] = 3; n_retained[r] = 0; }
    return;
  }
  if (k_keep > nv) k_keep = nv;
  if (k_core > nv) k_core = nv;

  // 2. normalised saliency
  const double span = __dsub_rn(hi, lo);
  for (int t = threadIdx.x; t < n_tok; t += kT)
    if (m_req[t] == 0) {
      const double v = (hi == lo) ? 0.5 : __ddiv_rn(__dsub_rn(s_req[t], lo), span);
      sn[t] = v;
      if (S.onchip) S.ks[t] = vmm::ord_key(v);
    }
  __syncthreads();

  auto is_vis = [&](int t) { return S.vis(t); };
  auto key_s = [&](int t) { return S.key_s(t); };

  // 3. salient core: top k_core by (-s_norm, id)
  if (k_core > 0) {
    if (k_core >= nv) {
      for (int t = threadIdx.x; t < n_tok; t += kT)
        if (S.vis(t)) S.set_flags(t, S.flags(t) | 1);
    } else {
      unsigned long long Ts;
      int gt;
      block_threshold(n_tok, k_core, is_vis, key_s, sh, &Ts, &gt);
      for (int t = threadIdx.x; t < n_tok; t += kT)
        if (S.vis(t) && S.key_s(t) > Ts) S.set_flags(t, S.flags(t) | 1);
      __syncthreads();
      block_mark_first(n_tok, k_core - gt, [&](int t) { return S.vis(t) && S.key_s(t) == Ts; },
                       [&](int t) { S.set_flags(t, S.flags(t) | 1); }, sh);
    }
  }
  __syncthreads();

  // 4. target expert set = OR of the core tokens' prefix masks
  {
    uint64_t acc[kWords] = {};
    int ebad = 0;
    for (int t = threadIdx.x; t < n_tok; t += kT)
      if (S.flags(t) & 1) {
        uint64_t m[kWords];
        ebad |= token_mask(routes, P, T, k, E, base + t, m);
#pragma unroll
        for (int w = 0; w < kWords; ++w) acc[w] |= m[w];
      }
#pragma unroll
    for (int w = 0; w < kWords; ++w) {
      unsigned lo32 = __reduce_or_sync(0xffffffffu, (unsigned)acc[w]);
      unsigned hi32 = __reduce_or_sync(0xffffffffu, (unsigned)(acc[w] >> 32));
      if ((threadIdx.x & 31) == 0 && (lo32 | hi32))
        atomicOr(&sh.target[w], ((unsigned long long)hi32 << 32) | lo32);
    }
    bad = __syncthreads_or(ebad);
  }
  uint64_t tg[kWords];
#pragma unroll
  for (int w = 0; w < kWords; ++w) tg[w] = sh.target[w];

  // 5. marginal expansion + score for the non-core visual tokens (compress.py:163-172)
  {
    int ebad = 0;
    for (int t = threadIdx.x; t < n_tok; t += kT)
      if (S.vis(t) && !(S.flags(t) & 1)) {
        uint64_t m[kWords];
        ebad |= token_mask(routes, P, T, k, E, base + t, m);
        int sz = 0, out = 0;
#pragma unroll
        for (int w = 0; w < kWords; ++w) { sz += __popcll(m[w]); out += __popcll(m[w] & ~tg[w]); }
        const double d = __ddiv_rn((double)out, (double)sz);
        const double p = __dsub_rn(sn[t], __dmul_rn(lam, d));
        dl[t] = d;
        sc[t] = p;
        if (S.onchip) S.kp[t] = vmm::ord_key(p);
      }
    bad |= __syncthreads_or(ebad);
  }
  if (bad) {  // an expert id outside [0, E) in the prefix routes (TraceError)
    for (int t = threadIdx.x; t < n_tok; t += kT) fl[t] = 0;
    if (threadIdx.x == 0) { status[r] = 4; n_retained[r] = 0; }
    return;
  }

  // 6. extras: top (k_keep - k_core) non-core visual tokens by (-score, -s_norm, id)
  const int need = k_keep - k_core;
  auto is_rest = [&](int t) { return S.vis(t) && !(S.flags(t) & 1); };
  if (need > 0) {
    if (need >= nv - k_core) {
      for (int t = threadIdx.x; t < n_tok; t += kT)
        if (is_rest(t)) S.set_flags(t, S.flags(t) | 2);
    } else {
      auto key_p = [&](int t) { return S.key_p(t); };
      unsigned long long Tp, Ts;
      int gtp, gts;
      block_threshold(n_tok, need, is_rest, key_p, sh, &Tp, &gtp);
      const int r1 = need - gtp;  // from the score ties, by s_norm
      auto tie_p = [&](int t) { return is_rest(t) && S.key_p(t) == Tp; };
      block_threshold(n_tok, r1, tie_p, key_s, sh, &Ts, &gts);
      const int r2 = r1 - gts;  // from the (score, s_norm) ties, by id
      for (int t = threadIdx.x; t < n_tok; t += kT)
        if (is_rest(t)) {
          const unsigned long long kp = S.key_p(t);
          if (kp > Tp || (kp == Tp && S.key_s(t) > Ts)) S.set_flags(t, S.flags(t) | 2);
        }
      __syncthreads();
      block_mark_first(n_tok, r2, [&](int t) { return tie_p(t) && S.key_s(t) == Ts; },
                       [&](int t) { S.set_flags(t, S.flags(t) | 2); }, sh);
    }
  }
  __syncthreads();
  if (threadIdx.x < kWords) target_out[(long long)r * kWords + threadIdx.x] = tg[threadIdx.x];

  // 7. retained = keep U text, ascending request-local ids (compress.py:63-65); final flags
  int n_ret = 0;
  for (int c0 = 0; c0 < n_tok; c0 += kT) {
    const int t = c0 + threadIdx.x;
    int f = 0;
    uint8_t fo = 0;
    if (t < n_tok) {
      const uint8_t fs = S.flags(t);
      fo = (fs & 1) ? 3 : (fs & 2);  // core tokens are kept
      f = (m_req[t] == 1) || (fo & 2);
    }
    const int pre = block_scan_flag(f, sh);
    if (f) retained[base + n_ret + pre] = t;
    if (t < n_tok) fl[t] = fo | (f ? 4 : 0);
    n_ret += sh.total;
  }
  if (threadIdx.x == 0) { n_retained[r] = n_ret; status[r] = 0; }
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
  cudaStream_t st = (cudaStream_t)stream;
  // per-token state on chip (17 B/token) for requests up to `cap` tokens; larger ones
  // run from the global outputs.  A few requests: 1024 threads each (latency), up to
  // 8192 tokens on chip; a batch: 256 threads, up to 4096 tokens (~68 KB: 3 CTAs/SM)
  const bool batch = R >= 64;
  const int cap = batch ? 4096 : (T < 8192 ? T : 8192);
  const size_t smem = (size_t)cap * 17;
  static bool attr[2] = {false, false};
  if (!attr[batch]) {
    cudaError_t e = batch ? cudaFuncSetAttribute(prune_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 4096 * 17)
                          : cudaFuncSetAttribute(prune_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 8192 * 17);
    if (e != cudaSuccess) return vmm::cuda_status(e, "prune attr");
    attr[batch] = true;
  }
  if (batch) {
    prune_kernel<256><<<R, 256, smem, st>>>(d_saliency, d_modality, d_routes, d_req_off, d_k_core, d_k_keep, alpha,
                                            beta, (long long)T, P, k, experts, lam, cap, d_s_norm, d_delta, d_score,
                                            d_flags, d_retained, d_n_retained, d_target, d_status);
  } else {
    prune_kernel<1024><<<R, 1024, smem, st>>>(d_saliency, d_modality, d_routes, d_req_off, d_k_core, d_k_keep,
                                              alpha, beta, (long long)T, P, k, experts, lam, cap, d_s_norm, d_delta,
                                              d_score, d_flags, d_retained, d_n_retained, d_target, d_status);
  }
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

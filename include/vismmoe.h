/*
 * vismmoe.h -- C-ABI of the B200-native VisMMOE per-layer hot path.
 *
 * One shared library (paper_2605_05899_b200/libvismmoe.so, sm_100a) exports
 * every entry point below.  Conventions:
 *   - plain pointers + sizes, no torch types; device pointers are marked `d_`,
 *     host pointers `h_`;
 *   - all device entry points are asynchronous on the caller's `stream`
 *     (a cudaStream_t passed as void*); ownership of buffers stays with the
 *     caller (torch tensors passed by data_ptr);
 *   - every function returns an int status (0 = OK); on failure the message is
 *     available from vmm_last_error() (thread-local).  Codes map 1:1 onto the
 *     reference's exception classes (pkg/src/moesim/errors.py:4-29):
 *       1 ValidationError  2 ContractError  3 SimulationError  4 TraceError
 *       5 PlanningError    6 device/CUDA error
 *   - handles (engine, stack) are single-owner and not reentrant, matching the
 *     reference's single-owner cache (pkg/src/moesim/cache.py:79).
 *
 * Reference interface each group replaces is cited per function.
 */
#ifndef VISMMOE_H
#define VISMMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VMM_OK 0
#define VMM_EVALIDATION 1
#define VMM_ECONTRACT 2
#define VMM_ESIMULATION 3
#define VMM_ETRACE 4
#define VMM_EPLANNING 5
#define VMM_ECUDA 6

#define VMM_MAX_EXPERTS 256 /* expert ids are bit-packed in 4 x u64 words */

const char *vmm_last_error(void);
int vmm_abi_version(void);
/* number of kernels this library has launched in the process (all entry points) */
long long vmm_launch_count(void);
/* 0 if device `dev` is sm_100 and the kernels of this library can run there */
int vmm_device_check(int dev);

/* ------------------------------------------------------------------------
 * Token compression (prune), batched over R requests, one CTA per request.
 * Replaces compress() pkg/src/moesim/compress.py:142-185 (normalize_saliency
 * :104-114, salient core :156-157, active_experts :125-132,
 * marginal_expansion :135-139, extras order :174) and
 * CompressionPlan.retained_ids :63-65.  Selections are threshold searches over
 * order-preserving fp64 keys + an id-ordered tie scan (no sort, no size cap).
 *   d_saliency [T] f64, d_modality [T] u8 (0 visual, 1 text, 2 decode),
 *   d_routes [P][T][k] i32: routes of the prefix layers for all T tokens,
 *   d_req_off [R+1] i32 token offsets.  Budgets: d_k_core/d_k_keep [R] i32, or
 *   both NULL -> floor(alpha*n_visual), floor(beta*n_visual) of each request on
 *   the device, exactly as :151-152 (one correctly rounded product each).
 * Outputs (token-indexed, per request segment): s_norm/delta/score f64 (NaN
 * where undefined), flags u8 (bit0 core, bit1 keep, bit2 retained),
 * d_retained i32 (request-local ids, ascending, packed at d_req_off[r]),
 * d_n_retained [R] i32, d_target [R][4] u64 expert bitmask, d_status [R] i32
 * (0 ok, 1 invalid saliency [ValidationError], 3 beta budget smaller than the
 * alpha budget [ValidationError], 4 expert id outside [0, experts) [TraceError]).
 * ------------------------------------------------------------------------ */
int vmm_prune(const double *d_saliency, const uint8_t *d_modality, const int32_t *d_routes,
              const int32_t *d_req_off, const int32_t *d_k_core, const int32_t *d_k_keep,
              double alpha, double beta, int R, int T, int P, int k, int experts, double lam,
              double *d_s_norm, double *d_delta, double *d_score, uint8_t *d_flags,
              int32_t *d_retained, int32_t *d_n_retained, uint64_t *d_target, int32_t *d_status,
              void *stream);

/* Pack the per-request retained lists of vmm_prune into one ascending list of
 * global row ids (request r's ids + req_off[r]) and the offsets of each
 * request's rows in it: d_out [sum n_retained], d_out_off [R+1]. */
int vmm_retained_pack(const int32_t *d_req_off, const int32_t *d_retained, const int32_t *d_n_retained, int R,
                      int32_t *d_out, int32_t *d_out_off, void *stream);

/* Row gather (stream compaction of hidden states): dst[i] = src[idx[i]], bf16 rows of H. */
int vmm_gather_rows(const void *d_src, const int32_t *d_idx, int n, int H, void *d_dst, void *stream);

/* ------------------------------------------------------------------------
 * Router: logits = X[N,H] . W_g[E,H]^T (bf16 in, fp32 accumulate), per-token
 * top-k by (logit desc, id asc) and softmax over the k selected logits, so
 * gates are > 0 and sum to 1 (the RoutingTrace contract, trace.py:80-81,
 * :375-382).  Optional per-expert pick counts (u32 [E], accumulated) give the
 * layer's demand set (trace.active_union, trace.py:102-107).
 * No reference implementation exists (router absent in the reference).
 * ------------------------------------------------------------------------ */
int vmm_route_topk(const void *d_x, const void *d_wg, int N, int H, int E, int k,
                   int32_t *d_ids, float *d_gates, float *d_logits /* nullable [N,E] */,
                   uint32_t *d_counts /* nullable [E] */, void *stream);

/* Fused router + gate-reuse lookahead for layer `layer` of a stacked router
 * [L][E][H]: one tcgen05 GEMM against the adjacent gates of layers l and l+1;
 * writes layer l's ids/gates/counts and the pick counts of layer l+1's gate on
 * the same rows (the lookahead predictor's input).  E in {16,32,64,128}. */
int vmm_route_lookahead(const void *d_x, const void *d_router, int layer, int L, int N, int H, int E, int k,
                        int32_t *d_ids, float *d_gates, uint32_t *d_counts, uint32_t *d_la_counts, void *stream);

/* Batch-invariant forms: the N rows are a chunk of a logical batch of batch_rows
 * (>= N) rows.  The kernel choice and the K-split count (so the fp32 summation
 * order of every logit) follow batch_rows, not N, so routing a batch in chunks
 * gives bit-for-bit the ids and gates of one launch over the whole batch.  The
 * plain entry points are the _ex forms with batch_rows = N. */
int vmm_route_topk_ex(const void *d_x, const void *d_wg, int N, int H, int E, int k,
                      int32_t *d_ids, float *d_gates, float *d_logits, uint32_t *d_counts, int batch_rows,
                      void *stream);
int vmm_route_lookahead_ex(const void *d_x, const void *d_router, int layer, int L, int N, int H, int E, int k,
                           int32_t *d_ids, float *d_gates, uint32_t *d_counts, uint32_t *d_la_counts,
                           int batch_rows, void *stream);

/* ------------------------------------------------------------------------
 * Demand / predictor kernels (pkg/src/moesim/predictor.py)
 * ------------------------------------------------------------------------ */
/* counts[l][e] = #picks of expert e at layer `layers[l]` over token ids (trace.active_union,
 * predictor.demand_set :115-117).  d_routes is the full [L][T][k] table. */
int vmm_demand_counts(const int32_t *d_routes, int L, int T, int k, int E,
                      const int32_t *d_layers, int n_layers, const int32_t *d_ids, int n_ids,
                      uint32_t *d_counts, void *stream);
/* Oracle targets y[c][e] = max_{d<=W, ctx+d<=L-1} decay[d-1]*[count[ctx+d][e]>0]
 * (build_targets :120-148).  d_counts is [L][E] over all layers. */
int vmm_oracle_targets(const uint32_t *d_counts, int L, int E, const int32_t *d_ctx, int n_ctx,
                       int window, const double *d_decay, double *d_y, void *stream);
/* History histogram (routing_histogram :63-75), bit-exact: per expert, the
 * weight pow[ctx-past] is added count times in ascending past order, then the
 * vector is divided by numpy's pairwise sum.  d_counts [L][E]. */
int vmm_history(const uint32_t *d_counts, int L, int E, const int32_t *d_ctx, int n_ctx,
                const double *d_pow, double *d_y, void *stream);
/* MLP predictor (build_features :86-112 + MLPModel.forward :196-202 + sigmoid :547):
 * x = [hist(ctx) ; mean_i(emb[ids_i] + drift[ctx]) ; h_v]; y = sigmoid(Wo relu(W2 relu(W1 x+b1)+b2)+bo).
 * fp64 throughout; weights row-major as the reference stores them. */
int vmm_mlp_predict(const double *d_hist /* [n_ctx][E] */, const double *d_emb, int D,
                    const double *d_drift /* [L][D] */, const int32_t *d_ids, int n_ids,
                    const double *d_hv /* [D] */, const int32_t *d_ctx, int n_ctx, int E,
                    const double *d_w1, const double *d_b1, int d_hidden,
                    const double *d_w2, const double *d_b2, int d_bottleneck,
                    const double *d_wo, const double *d_bo,
                    double *d_feat /* nullable [n_ctx][E+2D] */, double *d_y, void *stream);
/* Column means of emb[ids[i]] (rows with d_mod[row] != 0 skipped when d_mod is
 * given) in numpy's axis-0 order, zeros when none: the MLP's static visual
 * summary over the kept visual tokens (visual_summary, predictor.py:78-83). */
int vmm_row_mean(const double *d_emb, int D, const int32_t *d_ids, int n, const uint8_t *d_mod, double *d_out,
                 void *stream);
/* Gate-reuse lookahead: counts of experts in the top-k of W_next applied to
 * layer-l hidden states, normalised by N*k -> y f64 [E]. */
int vmm_normalize_counts(const uint32_t *d_counts, int E, double denom, double *d_y, void *stream);
int vmm_gate_lookahead(const void *d_x, const void *d_wnext, int N, int H, int E, int k,
                       uint32_t *d_scratch_counts /* [E] */, double *d_y, void *stream);

/* ------------------------------------------------------------------------
 * Attention-derived saliency (Alg. 1: s = Mean_h(A^h); the input the
 * reference reads precomputed from the trace, trace.py:49 / compress.py:145-148)
 * d_q bf16 [R][Hh][Q][D] (query rows: CLS or text tokens), d_k bf16 [R][Hh][N][D]
 * (the request's N tokens), scale = 1/sqrt(D) usually.  A = softmax(q k^T *
 * scale) per (request, head, query) in fp32 into d_probs f32 [R*Hh*Q][N];
 * d_s f64 [R*N] = mean over heads and queries, summed in ascending (h, q)
 * order.  vmm_attn_map_saliency does the mean for given maps [R*HQ][N].
 * ------------------------------------------------------------------------ */
int vmm_attn_saliency(const void *d_q, const void *d_k, int R, int Hh, int Q, int N, int D, float scale,
                      float *d_probs, double *d_s, void *stream);
int vmm_attn_map_saliency(const float *d_maps, int R, int HQ, int N, double *d_s, void *stream);

/* GPU routing diagnostics (metrics.py:25-67), bit-identical to the reference:
 * from per-layer expert histograms d_counts u32 [L][E] of a token subset of
 * size n_subset (vmm_demand_counts), write d_out f64 [L][4] = {working set,
 * top-`top` coverage, cosine(l, l+1), jaccard(l, l+1)} (last layer: NaN). */
int vmm_routing_diagnostics(const uint32_t *d_counts, int L, int E, int n_subset, int k, int top, double *d_out,
                            void *stream);

/* ------------------------------------------------------------------------
 * Expert permutation and combine (no reference numerics; pipeline.py:573 order)
 * plan: stable counting sort of the N*k (token, slot) picks by expert.
 *   d_offsets [E+1] i32, d_src_row [N*k] i32 (token of each permuted row),
 *   d_pos [N*k] i32 (permuted row of pick (t, j)).
 * ------------------------------------------------------------------------ */
int vmm_permute_plan(const int32_t *d_ids, int N, int k, int E, int32_t *d_offsets,
                     int32_t *d_src_row, int32_t *d_pos, void *stream);
/* plan + row copy in one pass over the picks (token order: each X row is read
 * once and stored to its k permuted positions): same outputs as
 * vmm_permute_plan followed by vmm_permute_rows(d_x, d_src_row, N*k, H, d_xp) */
int vmm_permute(const int32_t *d_ids, int N, int k, int E, const void *d_x, int H, int32_t *d_offsets,
                int32_t *d_src_row, int32_t *d_pos, void *d_xp, void *stream);
/* Xp[p] = X[src_row[p]] for the n_rows permuted rows (bf16 rows of H) */
int vmm_permute_rows(const void *d_x, const int32_t *d_src_row, int n_rows, int H, void *d_xp, void *stream);
/* combine plus S always-resident shared experts (unit weight; rows s*N + t of d_ys) */
int vmm_combine_shared(const void *d_y, const int32_t *d_pos, const float *d_gates, const void *d_resid,
                       int N, int k, int H, const void *d_ys, int S, void *d_out, void *stream);
/* fused combine (+ shared experts, S may be 0) and the next layer's RMSNorm:
 * bit-identical to vmm_combine_shared followed by vmm_rmsnorm(w = NULL) */
int vmm_combine_norm(const void *d_y, const int32_t *d_pos, const float *d_gates, const void *d_resid,
                     int N, int k, int H, const void *d_ys, int S, float eps, void *d_out, void *d_xn,
                     void *stream);
/* shared-expert plan: src[s*N + t] = t, offsets[s] = s*N (every token to each shared expert) */
int vmm_shared_plan(int N, int S, int32_t *d_src, int32_t *d_offsets, void *stream);
/* Pre-MoE RMSNorm of the token rows (the layer's router and experts see the
 * normalised rows, the residual is the raw row): y = x * rsqrt(mean(x^2)+eps) * w
 * (w nullable = ones). */
int vmm_rmsnorm(const void *d_x, const void *d_w, int n, int H, float eps, void *d_y, void *stream);

/* Decode-token glue in one launch (n <= 4 rows, n*k <= 32 picks, trace routing):
 * out = resid + sum_j gates_prev[t,j] * y[pos_prev[t,j]] (skipped when d_y is NULL:
 * the layer input is d_resid), xn = RMSNorm(out) (eps 1e-6, no weight), ids/gates of
 * this layer from the trace rows (d_tr_l/d_tg_l = layer l's [tokens][k] slices),
 * the stable plan by expert (offsets[E+1], src_row, pos) and xp[p] = xn[src_row[p]].
 * Bit-identical to vmm_combine + vmm_rmsnorm + vmm_gather_i32/f32 + vmm_permute. */
int vmm_decode_glue(const void *d_y, const int32_t *d_pos_prev, const float *d_gates_prev, const void *d_resid,
                    int n, int k, int H, void *d_out, void *d_xn, const int32_t *d_tr_l, const float *d_tg_l,
                    const int32_t *d_rows, int E, int32_t *d_ids, float *d_gates, int32_t *d_offsets,
                    int32_t *d_src_row, int32_t *d_pos, void *d_xp, void *stream);
/* out[t] = resid[t] + sum_j gates[t,j] * Y[pos[t,j]]  (bf16 rows, fp32 accumulate, j ascending) */
int vmm_combine(const void *d_y, const int32_t *d_pos, const float *d_gates, const void *d_resid,
                int N, int k, int H, void *d_out, void *stream);

/* ------------------------------------------------------------------------
 * Grouped bf16 SwiGLU expert FFN on tcgen05/TMEM with TMA operands.
 * Expert weights live in slots of one HBM arena, `slot_stride` bf16 elements
 * apart (normally 3*I*H: one contiguous 9.44 MB block per Qwen3-VL expert, so
 * a cache fill is ONE host->device copy):
 *   W13 at d_w13_arena + s*stride : [2I][H] bf16, rows interleaved per 64-row
 *            block (64 gate rows, then the 64 matching up rows), K-major;
 *   W2  at d_w2_arena  + s*stride : [H][I]  bf16, K-major.
 * d_slot_of_expert [E] i32 maps expert -> arena slot for this layer.
 * Xp: permuted token rows [M_total][H]; d_offsets [E+1] from vmm_permute_plan.
 * H1 scratch [M_total][I] bf16; Y out [M_total][H] bf16.
 * ------------------------------------------------------------------------ */
int vmm_grouped_swiglu(const void *d_xp, const int32_t *d_offsets, int E, int M_total,
                       int H, int I, const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                       long long n_slots, const int32_t *d_slot_of_expert, void *d_h1, void *d_y, void *stream);
/* Same contraction as ONE persistent launch (GEMM1 and GEMM2 tiles interleaved,
 * H1 dependencies resolved per 128-row block through d_done, a u32 scratch of
 * ceil(M_total/128)+E words, zeroed by the call).  Bit-identical to
 * vmm_grouped_swiglu.  Copy overlap: when d_need != NULL the GEMM tiles of
 * expert e first wait until d_ready[slot_of[e] - ready_base] >= d_need[e]
 * (u32 fill sequence numbers written by the copy stream after each fill, see
 * vmm_xfer_ready), so the layer computes on landed experts while the misses
 * still stream in.  need[e] == 0: no wait.  Row gather: when d_src_row
 * != NULL (the plan's [M_total] source rows) GEMM1 reads its A rows straight
 * from d_x_rows [n_x_rows][H] with TMA tile::gather4 and d_xp is unused, so no
 * permuted copy of the tokens is materialised.  M_total <= 16 (decode): one
 * persistent weight-streaming CUDA-core launch (both projections, grid-wide
 * barrier between them), which honours d_need/d_ready as well.  d_done ==
 * NULL with M_total > 16 falls through to vmm_grouped_swiglu (d_need and
 * d_src_row must then be NULL). */
int vmm_grouped_swiglu_fused(const void *d_xp, const int32_t *d_offsets, int E, int M_total,
                             int H, int I, const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                             long long n_slots, const int32_t *d_slot_of_expert, const uint32_t *d_need,
                             const uint32_t *d_ready, int ready_base, uint32_t *d_done,
                             const void *d_x_rows, const int32_t *d_src_row, int n_x_rows, void *d_h1, void *d_y,
                             void *stream);
/* Same, walking the experts in d_order (nullable, a device permutation of
 * [0, E)) instead of id order on the CTA-pair path: the executor puts a layer's
 * resident experts first and its misses in copy-issue order, largest first, so
 * the kernel's tail after the last copy lands is the smallest expert's tiles.
 * Bit-identical to any other order (each output row depends on its own expert). */
int vmm_grouped_swiglu_fused_ex(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                                const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                                long long n_slots, const int32_t *d_slot_of_expert, const uint32_t *d_need,
                                const uint32_t *d_ready, int ready_base, uint32_t *d_done, const void *d_x_rows,
                                const int32_t *d_src_row, int n_x_rows, void *d_h1, void *d_y,
                                const int32_t *d_order, void *stream);
/* Decode-sized layer (M_total <= 16 rows): the skinny weight-streaming FFN with the slot
 * table and the fill sequences given as HOST rows [E] -- they travel in the kernel's
 * parameter block, so a decode layer needs no per-layer upload in the compute stream. */
int vmm_grouped_swiglu_decode(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                              const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                              const int32_t *h_slot_of_expert, const uint32_t *h_need, const uint32_t *d_ready,
                              int ready_base, void *d_h1, void *d_y, void *stream);
/* H1 is scratch.  On the CTA-pair path (tensor-bound batches) the last GEMM2 tile
 * that consumes an H1 block drops it from L2 without a write-back
 * (discard.global.L2), so d_h1's contents after the call are undefined; keep != 0
 * (process-wide) keeps them, e.g. to compare H1 bit for bit. */
int vmm_ffn_keep_h1(int keep);
/* Reference (CUDA-core, fp32) version of the same contraction for cross-checks. */
int vmm_grouped_swiglu_simt(const void *d_xp, const int32_t *d_offsets, int E, int M_total,
                            int H, int I, const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                            const int32_t *d_slot_of_expert, void *d_h1, void *d_y, void *stream);

/* ------------------------------------------------------------------------
 * Cache policy + logical-clock engine (C++ mirror of ExpertCache,
 * pkg/src/moesim/cache.py:78-278, and _Engine, pipeline.py:382-760).
 * ------------------------------------------------------------------------ */
typedef struct vmm_engine vmm_engine;

typedef struct {
  int layers, experts, num_slabs;
  int victim_fifo;         /* victim_policy == "fifo" */
  int speculative_grace;
  int budget, window;      /* predictor.budget / window */
  int l_pinned, shared;
  int prefetching;         /* predictor attached and budget > 0 */
  int reactive;            /* simulate_reactive */
  int event_log;
  double transfer_ms, gpu_ms;
  double boot_ms;          /* compress latency (if compressed) + bootstrap (if prefetching) */
  const double *decay;     /* [window] gamma**(d-1), host-computed */
} vmm_engine_config;

/* one transfer / eviction decision, in decision order */
typedef struct {
  double t;        /* logical time */
  int32_t kind;    /* 0 issue, 1 complete, 2 evict */
  int32_t layer, expert, slab;
} vmm_engine_event;

typedef struct {
  double makespan, total_compute, total_transfer, exposed_transfer, prefill_ms;
  long long hits, misses, stalls, rejected_loads, on_demand_transfers, inflight_waits, evictions;
  int decode_steps;
} vmm_engine_report;

int vmm_engine_create(const vmm_engine_config *cfg, vmm_engine **out);
void vmm_engine_destroy(vmm_engine *e);
/* boot interval + first emission (pipeline.py:697-707); y may be NULL if !prefetching */
int vmm_engine_begin(vmm_engine *e, const double *h_y_boot);
/* run one layer (pipeline.py:709-721 / 723-740).  demand: expert ids ascending.
 * phase 0 prefill / 1 decode; step = decode step or -1.  If the engine is
 * prefetching and the layer is emitting, h_y is the predictor output for
 * context `layer` (else NULL). */
int vmm_engine_layer(vmm_engine *e, int layer, const int32_t *h_demand, int n_demand,
                     int phase, int step, const double *h_y);
/* With h_y == NULL an emitting layer defers its emission: the caller launches
 * the layer's compute first, then calls vmm_engine_emit (so copies decided by
 * the emission can wait for that compute). */
int vmm_engine_emit(vmm_engine *e, int layer, const double *h_y);
/* slabs holding (layer, demand[i]) after the layer ran (all must be resident) */
int vmm_engine_slots(const vmm_engine *e, int layer, const int32_t *h_demand, int n, int32_t *h_slabs);
/* close a decode step (records decode_ms_per_step) */
int vmm_engine_end_step(vmm_engine *e);
int vmm_engine_finish(vmm_engine *e, vmm_engine_report *rep);
/* which layers emit after running (prefill: layer >= l_pinned && layer < L-1;
 * decode: additionally layer == l_pinned-1) -> 1/0 */
int vmm_engine_emits(const vmm_engine *e, int layer, int phase);
/* drain the parity event log (issue/complete/evict exactly as the reference's
 * event_log, pipeline.py:446-478, 617-618) since the last call; returns count */
int vmm_engine_events(vmm_engine *e, vmm_engine_event *h_out, int cap);
int vmm_engine_pending_events(const vmm_engine *e);
/* drain transfer commands (layer, expert, slab) triples in issue order; these
 * drive the copy stream (also emitted in reactive mode) */
int vmm_engine_copies(vmm_engine *e, int32_t *h_out, int cap);
/* decode_ms_per_step values; returns the count */
int vmm_engine_decode_ms(const vmm_engine *e, double *h_out, int cap);
/* per-layer stats rows: (phase, step, layer, start, end, stall, transfers, hits) */
int vmm_engine_layer_stats(vmm_engine *e, double *h_out /* [n][8] */, int cap);
/* slab currently holding (layer, expert) or -1 */
int vmm_engine_slab_of(const vmm_engine *e, int layer, int expert);
/* snapshot of one slab: key (-1 if free), state 0 free/1 loading/2 resident,
 * class 0 expired/1 speculative/2 required, priority, ready_time (NaN if none) */
int vmm_engine_slab(const vmm_engine *e, int slab, int *layer, int *expert, int *state, int *cls,
                    double *priority, double *ready);

/* Standalone cache (ExpertCache drop-in; same transitions as the engine's) */
typedef struct vmm_cache vmm_cache;
int vmm_cache_create(int num_slabs, int victim_fifo, vmm_cache **out);
void vmm_cache_destroy(vmm_cache *c);
/* returns 0 miss / 1 hit / 2 in-flight; ready NaN if none */
int vmm_cache_lookup(const vmm_cache *c, int layer, int expert, double *ready);
/* status out: 0 already resident / 1 enqueued / 2 rejected; slab -1 if none;
 * evicted (-1,-1) if none.  cls 1 speculative, 2 required */
int vmm_cache_request(vmm_cache *c, int layer, int expert, double priority, int cls, int *status,
                      int *slab, int *ev_layer, int *ev_expert);
int vmm_cache_set_ready(vmm_cache *c, int layer, int expert, double t);
int vmm_cache_complete(vmm_cache *c, int layer, int expert, double t);
int vmm_cache_cancel(vmm_cache *c, int layer, int expert);
int vmm_cache_executed(vmm_cache *c, int layer, int expert);
/* window: n keys (layer,expert) pairs; prio: n_p (layer, expert, value) triples as doubles */
int vmm_cache_reclassify(vmm_cache *c, const int32_t *h_window, int n, int grace,
                         const int32_t *h_prio_keys, const double *h_prio_vals, int n_p);
int vmm_cache_select_victim(vmm_cache *c);
int vmm_cache_info(const vmm_cache *c, long long *evictions, int *occupancy, int *step);
int vmm_cache_slab(const vmm_cache *c, int slab, int *layer, int *expert, int *state, int *cls,
                   double *priority, double *ready, int *last_window_step, int *executed, int *seq);
/* every slab in one call: ints [n][7] = layer, expert, state, cls, last_window_step,
 * executed, seq; doubles [n][2] = priority, ready (NaN if none).  Returns n (>= 0)
 * or -status.  Backs the `slabs` attribute the reference engine iterates
 * (pkg/src/moesim/pipeline.py:520-524, cache.py:91). */
int vmm_cache_slabs(const vmm_cache *c, int32_t *h_ints, double *h_dbls, int cap);
/* slab holding (layer, expert), or -1 (ExpertCache.entry, cache.py:112-114) */
int vmm_cache_find(const vmm_cache *c, int layer, int expert);

/* ------------------------------------------------------------------------
 * Expert transfer runtime: pinned host pool -> HBM slab arena on a dedicated
 * copy stream with one event per slab fill; slab reuse waits on the compute
 * event of the layer that last read the slab (pipeline.py:440-494 made real).
 * ------------------------------------------------------------------------ */
typedef struct vmm_xfer vmm_xfer;
int vmm_xfer_create(int num_slabs, size_t slab_bytes, int max_layers, vmm_xfer **out);
void vmm_xfer_destroy(vmm_xfer *x);
/* enqueue host->slab copy of `bytes` from h_src (pinned) into d_dst on the copy
 * stream; it first waits for the compute event of the last layer that was
 * fenced on this slab (so a slab is never overwritten while being read).
 * `reserved` must be 0. */
int vmm_xfer_copy(vmm_xfer *x, int slab, const void *h_src, void *d_dst, size_t bytes, int reserved);
/* make `compute_stream` wait for the newest fill among the given slabs and the
 * newest fill of every other copy stream (each stream is FIFO => covers all
 * older fills) and register them as read by the next layer */
int vmm_xfer_fence(vmm_xfer *x, const int32_t *h_slabs, int n, void *compute_stream);
/* device u32 [num_slabs] fill flags: after each fill of slab s the copy stream
 * writes that fill's sequence number to ready[s] (stream memory op, ordered
 * after the copy).  NULL when the device lacks stream memory ops. */
const uint32_t *vmm_xfer_ready(vmm_xfer *x);
/* flag-based alternative to vmm_xfer_fence (no stream wait): register the
 * slabs as read by the next layer and write, per slab, the fill sequence number
 * a reader must see in ready[] (0 = nothing pending) into h_need */
int vmm_xfer_need(vmm_xfer *x, const int32_t *h_slabs, int n, uint32_t *h_need);
/* record the compute event closing the reads registered since the last call */
int vmm_xfer_layer_done(vmm_xfer *x, int layer, void *compute_stream);
int vmm_xfer_reset_stats(vmm_xfer *x);
/* per-(layer, expert) source pointers [L*E] (sharded mode: local or IPC-mapped
 * peer HBM home copies).  vmm_xfer_issue_engine with h_pool == NULL uses them. */
int vmm_xfer_set_sources(vmm_xfer *x, const void *const *h_table, long long n);
/* data-parallel host pool (SURVEY 8(e) mode DP): the ranks of a node map ONE
 * shared-memory expert pool and each page-locks it for its own context
 * (cudaHostRegisterPortable), so every rank's copy engine DMAs from the same
 * host pages -- one copy of the experts per node instead of one per GPU. */
int vmm_host_register(void *h_ptr, size_t bytes);
int vmm_host_unregister(void *h_ptr);
/* sharded expert cache plumbing: export / map a device allocation across
 * processes (64-byte handle) and enable peer access over NVLink */
int vmm_ipc_get(const void *d_ptr, void *h_handle64);
int vmm_ipc_open(const void *h_handle64, void **d_ptr);
/* byte offset of d_ptr inside its allocation (the opener of a handle gets the base) */
int vmm_ipc_offset(const void *d_ptr, long long *off);
int vmm_ipc_close(void *d_ptr);
int vmm_peer_enable(int peer);
/* one copy-engine copy (any direction, incl. an IPC-mapped peer pointer) on `stream`;
 * used to measure the link peaks the logical clock is calibrated with */
int vmm_copy_async(void *d_dst, const void *src, size_t bytes, void *stream);
/* stream-ordered memset / strided 2-D copy (copy engine, no kernel): the host glue
 * zeroes counters and lands per-chunk prefix routes in the [L][T][k] table with them */
int vmm_memset_async(void *d_ptr, int byte_value, size_t bytes, void *stream);
int vmm_copy2d_async(void *d_dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                     void *stream);
/* drain the engine's transfer commands and enqueue each as one copy of
 * slot_bytes from the pinned host pool slot ((layer % host_layers)*experts +
 * expert) into arena slot (slab_offset + slab) */
int vmm_xfer_issue_engine(vmm_xfer *x, vmm_engine *e, const void *h_pool, int host_layers, int experts,
                          void *d_arena, long long slab_offset, size_t slot_bytes, int *n_issued);
/* Same, with the physical issue order of layer `layer_now`'s copies set by
 * h_rank[expert] (lowest first; the other layers' copies follow in decided
 * order; the decided order is kept whenever two copies target one slab).  The
 * decisions, slabs and logical clock are the engine's -- only the order in
 * which the copy engine moves them changes.  h_issued_experts (nullable, [E])
 * receives layer_now's experts in issue order. */
int vmm_xfer_issue_engine_ordered(vmm_xfer *x, vmm_engine *e, const void *h_pool, int host_layers, int experts,
                                  void *d_arena, long long slab_offset, size_t slot_bytes, int layer_now,
                                  const int32_t *h_rank, int32_t *h_issued_experts, int *n_issued);
int vmm_xfer_sync(vmm_xfer *x);
/* make compute_stream wait for every copy issued so far */
int vmm_xfer_join(vmm_xfer *x, void *compute_stream);
/* copy-stream accounting: bytes issued and wall ms between first and last copy (events) */
int vmm_xfer_stats(vmm_xfer *x, double *bytes, double *busy_ms, long long *copies);
void *vmm_xfer_stream(vmm_xfer *x);

/* ------------------------------------------------------------------------
 * Expert-parallel token exchange over peer memory: the
 * alternative to weight pulls -- experts stay on their owner rank (e % G) and
 * token rows move.  Tables are device arrays of G peer pointers (IPC-mapped
 * allocations; the own rank's entry is local).  The host exchanges the
 * per-layer (source rank, expert) counts and orders the phases (stream sync +
 * process barrier between dispatch, expert compute and return).
 *   vmm_ep_dispatch: pick i (expert e = d_ids[i], owner e % G) -> its row of
 *                    d_xn [N][H] into the owner's rows buffer at
 *                    d_base[e] + (d_pos[i] - d_my_off[e]) (d_pos / d_my_off:
 *                    this rank's vmm_permute_plan by expert), meta (int2) =
 *                    {source rank, i}: the owner's buffer is already grouped
 *                    by expert for vmm_grouped_swiglu_fused
 *   vmm_ep_return:   received row r's output -> source meta[r].x's return
 *                    buffer at pick index meta[r].y (pick order)
 * ------------------------------------------------------------------------ */
int vmm_ep_dispatch(const void *d_xn, int H, const int32_t *d_ids, int k, const int32_t *d_pos,
                    const int32_t *d_my_off, const int32_t *d_base, const void *d_rows_tab, const void *d_meta_tab,
                    int G, int rank, int M, void *stream);
int vmm_ep_return(const void *d_y_local, int H, const void *d_meta, const void *d_back_tab, int n_recv,
                  void *stream);

/* ------------------------------------------------------------------------
 * Native layer-loop executor (the per-layer body of pipeline.py:709-740 on
 * the device): rmsnorm -> route (+ fused gate lookahead) -> scores -> ONE
 * sync -> engine decisions -> copies -> slot table + fence -> permute ->
 * grouped SwiGLU -> combine -> reader event -> deferred emission.  All
 * buffers are caller-owned; the executor holds pointers only.
 * ------------------------------------------------------------------------ */
int vmm_gather_i32(const int32_t *d_src, const int32_t *d_rows, int n, int width, int32_t *d_dst, void *stream);
int vmm_gather_f32(const float *d_src, const int32_t *d_rows, int n, int width, float *d_dst, void *stream);

typedef struct {
  int layers, experts, k, hidden, inter, l_pinned;
  long long n_pinned_slots, n_slots;
  size_t slot_bytes;
  int host_layers;
  int cap_rows;              /* capacity of the row scratch buffers */
  int routing;               /* 0 live, 1 trace */
  int predictor;             /* 0 none, 1 history, 2 gate lookahead, 3 oracle table */
  int counts_preset;         /* trace routing: counts rows already filled by the caller */
  void *arena;               /* d bf16 [n_slots][3*I*H] */
  const void *pool;          /* h pinned bf16 [host_layers*E][3*I*H] */
  const void *router;        /* d bf16 [L][E][H] */
  const int32_t *pinned_slot_of; /* d [l_pinned][E] */
  const int32_t *layer_ids;  /* d [L] = 0..L-1 */
  const double *pow_table;   /* d [L+1] history decay powers */
  const double *oracle_table;/* d [L][E] (predictor 3), row = context layer */
  const int32_t *trace_routes; /* d [L][trace_tokens][k] (routing 1) */
  const float *trace_gates;    /* d [L][trace_tokens][k] */
  int trace_tokens;
  void *xn, *xp, *h1, *y, *out0, *out1; /* d scratch: [cap][H], [cap*k][H], [cap*k][I], [cap*k][H], [cap][H] x2 */
  int32_t *ids; float *gates;           /* d [cap][k] */
  int32_t *off, *src, *pos;             /* d [E+1], [cap*k], [cap*k] */
  uint32_t *counts;                     /* d [L][E] demand counts (history input) */
  uint32_t *la_counts;                  /* d [E] */
  double *y_dev;                        /* d [E] */
  int32_t *slot_dev;                    /* d [L][E] */
  int32_t *counts_host;                 /* h pinned [L][E] */
  double *y_host;                       /* h pinned [L][E] scores per context layer */
  int32_t *slot_host;                   /* h pinned [L][E] */
  int shared;                           /* S always-resident shared experts per layer (0: none) */
  const int32_t *shared_slot_of;        /* d [L][S] arena slots of the shared experts */
  int32_t *shared_src, *shared_off;     /* d [cap*S], [S+1] */
  void *xs, *h1s, *ys;                  /* d [cap*S][H], [cap*S][I], [cap*S][H] */
  uint32_t *need_host;                  /* nullable h pinned [L][E]: fill seq each expert's FFN waits for */
  uint32_t *need_dev;                   /* nullable d [L][E] (with need_host: flag-based copy overlap) */
  uint32_t *ffn_done;                   /* nullable d [cap*k/128 + E + 1] fused-FFN scratch (NULL: 2 launches) */
  /* predictor 4 = MLP (predictor.py:521-550): features from the stack's own routes
   * (history over counts[0..ctx]) + the request tokens' embeddings; fp64 weights row-major */
  const double *mlp_emb;                /* d [tokens][mlp_dim] token embeddings (rows indexed by mlp_ids) */
  const double *mlp_drift;              /* d [L][mlp_dim] cumulative layer drift (predictor.py:36-44) */
  const double *mlp_hv;                 /* d [mlp_dim] kept-visual embedding mean (predictor.py:78-83) */
  const int32_t *mlp_ids;               /* d [mlp_n_ids] retained token rows of mlp_emb */
  int mlp_dim, mlp_n_ids, mlp_hidden, mlp_bottleneck;
  const double *mlp_w1, *mlp_b1, *mlp_w2, *mlp_b2, *mlp_wo, *mlp_bo;
  double *mlp_hist;                     /* d [E] scratch: the history feature of the context layer */
  int route_batch_rows;                 /* rows of the logical batch these rows belong to (0: n_rows); the
                                           router's split count follows it (vmm_route_topk_ex) */
  int32_t *order_host;                  /* nullable h pinned [L][E]: per-layer expert walk / copy order */
  int32_t *order_dev;                   /* nullable d [L][E] (with order_host: largest experts first) */
} vmm_stack_desc;

typedef struct {
  const void *x_out;         /* device rows after the last layer (one of out0/out1) */
  int copies;                /* expert transfers issued */
  int32_t *routes;           /* nullable d [l1-l0][n_rows][k]: record of the routes used */
  void **ffn_start, **ffn_end; /* nullable cudaEvent_t arrays [l1-l0] around the grouped SwiGLU */
  int *n_demand;             /* nullable h [l1-l0] demanded experts per layer */
  double host_us[4];         /* host time: launches before the sync, sync wait, decisions+copies, launches after */
  void **copy_marks;         /* nullable cudaEvent_t [3*(l1-l0)] on the copy stream: before the layer's demand
                                copies, after them, after its emission copies */
} vmm_stack_out;

typedef struct vmm_stack vmm_stack;
int vmm_stack_create(const vmm_stack_desc *desc, vmm_stack **out);
void vmm_stack_destroy(vmm_stack *s);
/* run layers [l0, l1) on n_rows rows starting from d_x (phase 0 prefill / 1
 * decode, decode step `step`); d_rows = trace rows of these tokens (routing 1) */
int vmm_stack_layers(vmm_stack *s, vmm_engine *eng, vmm_xfer *xf, const void *d_x, int n_rows, int l0, int l1,
                     int phase, int step, const int32_t *d_rows, void *stream, vmm_stack_out *out);

#ifdef __cplusplus
}
#endif
#endif /* VISMMOE_H */

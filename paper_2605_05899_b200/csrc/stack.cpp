// Native layer-loop executor: the per-layer body of the reference engine
// (pkg/src/moesim/pipeline.py:709-740) driving the device kernels, the
// decision engine and the copy stream without returning to Python.
//
// Per layer l (prefill rows or one decode token):
//   rmsnorm -> route (live: tcgen05/skinny router, fused with the gate
//   lookahead when emitting; trace: gather the contract routes) -> predictor
//   scores -> D2H demand counts (+ scores) -> ONE stream sync -> engine
//   decisions -> expert copies -> slot table + fence -> permute -> grouped
//   SwiGLU (tcgen05) -> combine -> reader event -> deferred emission ->
//   prefetch copies.
// The host only waits once per layer (the decisions need the layer's demand
// set); everything else is asynchronous on the caller's compute stream and the
// xfer copy stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vismmoe.h"

namespace vmm {
int fail(int code, const std::string &msg);
}

namespace {
int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return VMM_OK;
  return vmm::fail(VMM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define VMM_TRY(x)           \
  do {                       \
    int _st = (x);           \
    if (_st) return _st;     \
  } while (0)
#define VMM_CUDA(x, what)                          \
  do {                                             \
    cudaError_t _e = (x);                          \
    if (_e != cudaSuccess) return cuda_status(_e, what); \
  } while (0)
}  // namespace

extern "C" {
int vmm_engine_slots(const vmm_engine *e, int layer, const int32_t *h_demand, int n, int32_t *h_slabs);
int vmm_engine_emit(vmm_engine *e, int layer, const double *h_y);
int vmm_xfer_issue_engine(vmm_xfer *x, vmm_engine *e, const void *h_pool, int host_layers, int experts,
                          void *d_arena, long long slab_offset, size_t slot_bytes, int *n_issued);
int vmm_xfer_issue_engine_ordered(vmm_xfer *x, vmm_engine *e, const void *h_pool, int host_layers, int experts,
                                  void *d_arena, long long slab_offset, size_t slot_bytes, int layer_now,
                                  const int32_t *h_rank, int32_t *h_issued_experts, int *n_issued);
int vmm_grouped_swiglu_decode(const void *d_xp, const int32_t *d_offsets, int E, int M_total, int H, int I,
                              const void *d_w13_arena, const void *d_w2_arena, long long slot_stride,
                              const int32_t *h_slot_of_expert, const uint32_t *h_need, const uint32_t *d_ready,
                              int ready_base, void *d_h1, void *d_y, void *stream);
int vmm_gather_i32(const int32_t *d_src, const int32_t *d_rows, int n, int width, int32_t *d_dst, void *stream);
int vmm_gather_f32(const float *d_src, const int32_t *d_rows, int n, int width, float *d_dst, void *stream);
const uint32_t *vmm_xfer_ready(vmm_xfer *x);
void *vmm_xfer_stream(vmm_xfer *x);
int vmm_xfer_mark(vmm_xfer *x, void *ev);
int vmm_xfer_need(vmm_xfer *x, const int32_t *h_slabs, int n, uint32_t *h_need);
}

struct vmm_stack {
  vmm_stack_desc d;
};

namespace {
// Low-latency host wait: the compute stream writes an epoch into a mapped
// pinned word (stream memory op, ordered after the preceding D2H copies) and
// the host spins on it -- a few microseconds less per layer than waking up from
// cudaStreamSynchronize, which matters for decode (one host decision per layer).
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct HostFlag {
  volatile uint32_t *h = nullptr;
  CUdeviceptr d = 0;
  uint32_t epoch = 0;
  WriteValue32Fn wv = nullptr;
  bool ok = false;
  HostFlag() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return;
    wv = reinterpret_cast<WriteValue32Fn>(p);
    void *hp = nullptr, *dp = nullptr;
    if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) != cudaSuccess) return;
    if (cudaHostGetDevicePointer(&dp, hp, 0) != cudaSuccess) return;
    h = reinterpret_cast<volatile uint32_t *>(hp);
    *h = 0;
    d = (CUdeviceptr)dp;
    ok = true;
  }
};
HostFlag &host_flag() {
  thread_local HostFlag f;  // one per host thread (handles are single-owner)
  return f;
}
// enqueue the marker after the work already in `st`
int host_mark(cudaStream_t st, uint32_t *epoch_out) {
  HostFlag &f = host_flag();
  if (!f.ok) return 1;
  const uint32_t e = ++f.epoch;
  if (f.wv((CUstream)st, f.d, e, 0) != CUDA_SUCCESS) return 1;
  *epoch_out = e;
  return 0;
}
// spin until the marker lands; every few thousand polls ask the stream whether it
// failed (a trapped kernel never writes the marker) -> returns the CUDA error
cudaError_t host_spin(cudaStream_t st, uint32_t epoch) {
  HostFlag &f = host_flag();
  for (uint32_t n = 1; (int32_t)(*f.h - epoch) < 0; ++n) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
    if ((n & 4095) == 0) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e != cudaSuccess && e != cudaErrorNotReady) return e;
      if (e == cudaSuccess && (int32_t)(*f.h - epoch) < 0) return cudaErrorUnknown;  // drained, no marker
    }
  }
  return cudaSuccess;
}
}  // namespace

extern "C" {

int vmm_stack_create(const vmm_stack_desc *desc, vmm_stack **out) {
  if (!desc || !out) return vmm::fail(VMM_ECONTRACT, "null argument");
  if (desc->experts < 1 || desc->experts > VMM_MAX_EXPERTS) return vmm::fail(VMM_EVALIDATION, "bad expert count");
  auto *s = new vmm_stack();
  s->d = *desc;
  *out = s;
  return VMM_OK;
}

void vmm_stack_destroy(vmm_stack *s) { delete s; }

int vmm_stack_layers(vmm_stack *s, vmm_engine *eng, vmm_xfer *xf, const void *d_x, int n_rows, int l0, int l1,
                     int phase, int step, const int32_t *d_rows, void *stream, vmm_stack_out *out) {
  const vmm_stack_desc &d = s->d;
  const int E = d.experts, k = d.k, H = d.hidden, I = d.inter, L = d.layers, lp = d.l_pinned;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows <= 0 || n_rows > d.cap_rows) return vmm::fail(VMM_ECONTRACT, "row count outside the buffers");
  // eng == NULL: pinned-prefix mode (layers < l_pinned on resident experts): no decisions,
  // no copies, no host sync -- the whole range is enqueued asynchronously
  const bool pinned_only = eng == nullptr;
  if (pinned_only && l1 > lp) return vmm::fail(VMM_ECONTRACT, "engine-less run must stay inside the pinned prefix");
  const size_t row_bytes = (size_t)H * 2;
  const void *cur = d_x;
  int ping = 0, copies = 0;
  std::vector<int32_t> demand, slabs;
  std::vector<uint32_t> need;
  // expert walk / copy order (largest first) for the CTA-pair FFN; VMM_NO_WALK_ORDER=1: id order
  static const bool no_walk = std::getenv("VMM_NO_WALK_ORDER") != nullptr;
  // decode-sized layers: slot / need rows as kernel parameters (VMM_DECODE_UPLOAD_ROWS=1: upload them;
  // the opt-in tensor-core decode FFN, VMM_DECODE_TC=1, reads device rows)
  static const bool by_value_rows =
      std::getenv("VMM_DECODE_UPLOAD_ROWS") == nullptr && std::getenv("VMM_DECODE_TC") == nullptr;
  std::vector<int32_t> by_size(E), rank_of(E), issued(E);
  std::vector<char> is_miss(E);
  const uint32_t *ready = vmm_xfer_ready(xf);
  // tensor-core FFN with per-expert ready flags: the layer's FFN starts while its misses still stream in
  // (VMM_FFN_FENCE=1: whole-layer event fence instead, e.g. under a serialising profiler)
  static const bool force_fence = std::getenv("VMM_FFN_FENCE") != nullptr;
  const bool flagged = !force_fence && ready && d.need_host && d.need_dev && d.ffn_done;
  // Trace routing with preset counts (oracle / no predictor): every layer's demand
  // set -- and the oracle's scores -- is known before the first layer runs.  Copy
  // them to the host once and take all the layers' decisions without a per-layer
  // GPU round trip; the kernels and copies are enqueued ahead of the GPU and the
  // FFNs wait on the copy stream's ready flags (decode: one sync per token instead
  // of one per layer).  VMM_NO_PRESYNC=1 restores the per-layer sync.
  static const bool no_presync = std::getenv("VMM_NO_PRESYNC") != nullptr;
  const bool presync = !pinned_only && !no_presync && d.routing == 1 && d.counts_preset &&
                       (d.predictor == 0 || d.predictor == 3);
  if (presync) {
    VMM_CUDA(cudaMemcpyAsync(d.counts_host + (size_t)l0 * E, d.counts + (size_t)l0 * E,
                             sizeof(uint32_t) * E * (l1 - l0), cudaMemcpyDeviceToHost, st),
             "preset counts D2H");
    if (d.predictor == 3)
      VMM_CUDA(cudaMemcpyAsync(d.y_host + (size_t)l0 * E, d.oracle_table + (size_t)l0 * E,
                               sizeof(double) * E * (l1 - l0), cudaMemcpyDeviceToHost, st),
               "oracle scores D2H");
    uint32_t ep = 0;
    if (host_mark(st, &ep) == 0) VMM_CUDA(host_spin(st, ep), "preset sync");
    else VMM_CUDA(cudaStreamSynchronize(st), "preset sync");
  }
  bool have_xn = false;  // the fused combine of the previous layer already produced this layer's xn
  // Early decisions (live routing, large batches): the previous layer's combine ->
  // norm -> this layer's route run on the first n_split rows first; their expert
  // set is a subset of the layer's demand set, and at prefill sizes it already
  // contains every expert -- then it IS the demand set, the host decides and the
  // copies start while the other 7/8 of the combine/norm/route work is still
  // running.  Otherwise the host waits for the full counts (same decisions
  // either way; VMM_NO_EARLY_DECIDE=1 disables the split).
  static const bool no_split = std::getenv("VMM_NO_EARLY_DECIDE") != nullptr;
  // first chunk: 1/VMM_SPLIT_DIV of the rows (default 8; 16 and 32 measured the same decision gap)
  static const int split_div = std::getenv("VMM_SPLIT_DIV") ? std::max(2, std::atoi(std::getenv("VMM_SPLIT_DIV"))) : 8;
  const int n_split = (!pinned_only && !no_split && d.routing == 0 && d.shared == 0 && n_rows >= 8192)
                          ? std::max(1024, n_rows / split_div) : 0;
  bool pending_rest = false;  // previous layer's combine covered rows [0, n_split) only
  const void *rest_resid = nullptr;
  void *rest_dst = nullptr;
  cudaEvent_t ev_part = nullptr, ev_y = nullptr;
  struct EvGuard {
    cudaEvent_t *a, *b;
    ~EvGuard() {
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } ev_guard{&ev_part, &ev_y};
  if (n_split) {
    VMM_CUDA(cudaEventCreateWithFlags(&ev_part, cudaEventDisableTiming), "event");
    VMM_CUDA(cudaEventCreateWithFlags(&ev_y, cudaEventDisableTiming), "event");
  }
  using clk = std::chrono::steady_clock;
  double t_pre = 0, t_sync = 0, t_dec = 0, t_post = 0;  // host microseconds per phase
  auto us = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count();
  };
  // Decode-sized layers with trace routing: the previous layer's combine, this
  // layer's RMSNorm, trace gathers, plan and row copy run as ONE launch
  // (vmm_decode_glue, bit-identical to the separate kernels) at the layer start.
  static const bool no_glue = std::getenv("VMM_NO_DECODE_GLUE") != nullptr;
  static const bool gather_env0 = std::getenv("VMM_FFN_GATHER") != nullptr;
  const bool glue = !no_glue && !gather_env0 && d.routing == 1 && d.shared == 0 && n_rows <= 4 && n_rows * k <= 16;
  const void *glue_resid = nullptr;  // pending combine: the previous layer's residual input
  for (int l = l0; l < l1; ++l) {
    auto c0 = clk::now();
    void *xn = d.xn;
    if (glue) {
      const int32_t *tr = d.trace_routes + (size_t)l * d.trace_tokens * k;
      const float *tg = d.trace_gates + (size_t)l * d.trace_tokens * k;
      VMM_TRY(vmm_decode_glue(glue_resid ? d.y : nullptr, d.pos, d.gates, glue_resid ? glue_resid : cur, n_rows, k, H,
                              const_cast<void *>(cur), xn, tr, tg, d_rows, E, d.ids, d.gates, d.off, d.src, d.pos,
                              d.xp, stream));
    } else if (!have_xn) {
      VMM_TRY(vmm_rmsnorm(cur, nullptr, n_rows, H, 1e-6f, xn, stream));
    }
    const int emits = pinned_only ? 0 : vmm_engine_emits(eng, l, phase);
    uint32_t *cnt = d.counts + (size_t)l * E;
    bool la_done = false;
    int32_t *ch = d.counts_host + (size_t)l * E;
    const bool split_now = pending_rest;
    bool part_flag = false;
    uint32_t part_epoch = 0;
    if (d.routing == 0) {
      VMM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * E, st), "counts memset");
      const bool fused_la = emits && d.predictor == 2 && l + 1 < L && (E % 16 == 0) && E <= 128;
      if (fused_la) VMM_CUDA(cudaMemsetAsync(d.la_counts, 0, sizeof(uint32_t) * E, st), "lookahead memset");
      // rows [r0, r1) of this layer's router (counts accumulate over the launches)
      auto route_rows = [&](int r0, int r1) -> int {
        const char *x0 = (const char *)xn + (size_t)r0 * H * 2;
        // the split router's numerics follow the whole batch, not the chunk (vmm_route_topk_ex)
        const int br = d.route_batch_rows > n_rows ? d.route_batch_rows : n_rows;
        if (fused_la)
          return vmm_route_lookahead_ex(x0, d.router, l, L, r1 - r0, H, E, k, d.ids + (size_t)r0 * k,
                                        d.gates + (size_t)r0 * k, cnt, d.la_counts, br, stream);
        return vmm_route_topk_ex(x0, (const char *)d.router + (size_t)l * E * H * 2, r1 - r0, H, E, k,
                                 d.ids + (size_t)r0 * k, d.gates + (size_t)r0 * k, nullptr, cnt, br, stream);
      };
      if (split_now) {
        VMM_TRY(route_rows(0, n_split));
        VMM_CUDA(cudaMemcpyAsync(ch, cnt, sizeof(uint32_t) * E, cudaMemcpyDeviceToHost, st), "partial counts D2H");
        VMM_CUDA(cudaEventRecord(ev_part, st), "partial event");
        part_flag = host_mark(st, &part_epoch) == 0;
        // the rest of the previous layer's combine (its gates/pos/Y rows are untouched by chunk 1)
        const int nr = n_rows - n_split;
        VMM_TRY(vmm_combine_norm(d.y, d.pos + (size_t)n_split * k, d.gates + (size_t)n_split * k,
                                 (const char *)rest_resid + (size_t)n_split * H * 2, nr, k, H, nullptr, 0, 1e-6f,
                                 (char *)rest_dst + (size_t)n_split * H * 2, (char *)xn + (size_t)n_split * H * 2,
                                 stream));
        VMM_TRY(route_rows(n_split, n_rows));
        pending_rest = false;
      } else {
        VMM_TRY(route_rows(0, n_rows));
      }
      la_done = fused_la;
    } else {
      const int32_t *tr = d.trace_routes + (size_t)l * d.trace_tokens * k;
      const float *tg = d.trace_gates + (size_t)l * d.trace_tokens * k;
      if (!glue) {
        VMM_TRY(vmm_gather_i32(tr, d_rows, n_rows, k, d.ids, stream));
        VMM_TRY(vmm_gather_f32(tg, d_rows, n_rows, k, d.gates, stream));
      }
      if (!d.counts_preset) {
        int32_t lay = l;
        (void)lay;
        VMM_TRY(vmm_demand_counts(d.trace_routes, L, d.trace_tokens, k, E, d.layer_ids + l, 1, d_rows, n_rows, cnt,
                                  stream));
      }
    }
    if (out && out->routes)
      VMM_CUDA(cudaMemcpyAsync(out->routes + (size_t)(l - l0) * n_rows * k, d.ids, sizeof(int32_t) * n_rows * k,
                               cudaMemcpyDeviceToDevice, st), "record routes");
    double *yh = d.y_host + (size_t)l * E;
    if (emits) {
      const double *ysrc = nullptr;
      if (la_done) {
        VMM_TRY(vmm_normalize_counts(d.la_counts, E, (double)n_rows * k, d.y_dev, stream));
        ysrc = d.y_dev;
      } else if (d.predictor == 1) {
        VMM_TRY(vmm_history(d.counts, L, E, d.layer_ids + l, 1, d.pow_table, d.y_dev, stream));
        ysrc = d.y_dev;
      } else if (d.predictor == 2) {
        VMM_TRY(vmm_gate_lookahead(xn, (const char *)d.router + (size_t)(l + 1) * E * H * 2, n_rows, H, E, k,
                                   d.la_counts, d.y_dev, stream));
        ysrc = d.y_dev;
      } else if (d.predictor == 3) {
        ysrc = presync ? nullptr : d.oracle_table + (size_t)l * E;  // presync: already in y_host
      } else if (d.predictor == 4) {  // MLP: history feature of context l, then the bottleneck MLP
        if (!d.mlp_w1 || !d.mlp_hist || !d.mlp_emb || !d.mlp_ids)
          return vmm::fail(VMM_ECONTRACT, "MLP predictor without weights / features");
        VMM_TRY(vmm_history(d.counts, L, E, d.layer_ids + l, 1, d.pow_table, d.mlp_hist, stream));
        VMM_TRY(vmm_mlp_predict(d.mlp_hist, d.mlp_emb, d.mlp_dim, d.mlp_drift, d.mlp_ids, d.mlp_n_ids, d.mlp_hv,
                                d.layer_ids + l, 1, E, d.mlp_w1, d.mlp_b1, d.mlp_hidden, d.mlp_w2, d.mlp_b2,
                                d.mlp_bottleneck, d.mlp_wo, d.mlp_bo, nullptr, d.y_dev, stream));
        ysrc = d.y_dev;
      } else {
        return vmm::fail(VMM_ECONTRACT, "emitting layer without a predictor");
      }
      if (ysrc) VMM_CUDA(cudaMemcpyAsync(yh, ysrc, sizeof(double) * E, cudaMemcpyDeviceToHost, st), "scores D2H");
      if (split_now) VMM_CUDA(cudaEventRecord(ev_y, st), "scores event");
    }
    auto c1 = clk::now(), c2 = c1;
    int n = 0;
    const int32_t *order_of = nullptr;  // FFN expert walk order (nullptr: id order)
    demand.clear();
    if (!pinned_only) {
      bool known = false;
      if (split_now) {  // the first chunk's experts: the whole demand set if they are all E
        c1 = clk::now();
        if (part_flag) VMM_CUDA(host_spin(st, part_epoch), "partial sync");
        else VMM_CUDA(cudaEventSynchronize(ev_part), "partial sync");
        c2 = clk::now();
        int n_act = 0;
        for (int e = 0; e < E; ++e) n_act += ch[e] != 0;
        known = n_act == E;
        if (known)
          for (int e = 0; e < E; ++e) demand.push_back(e);
      }
      if (!known && presync) {  // counts already on the host
        c1 = c2 = clk::now();
        for (int e = 0; e < E; ++e)
          if (ch[e]) demand.push_back(e);
      } else if (!known) {
        VMM_CUDA(cudaMemcpyAsync(ch, cnt, sizeof(uint32_t) * E, cudaMemcpyDeviceToHost, st), "counts D2H");
        c1 = clk::now();
        uint32_t ep = 0;
        if (host_mark(st, &ep) == 0) VMM_CUDA(host_spin(st, ep), "layer sync");  // counts (and scores) landed
        else VMM_CUDA(cudaStreamSynchronize(st), "layer sync");
        c2 = clk::now();
        for (int e = 0; e < E; ++e)
          if (ch[e]) demand.push_back(e);
      }
      VMM_TRY(vmm_engine_layer(eng, l, demand.data(), (int)demand.size(), phase, step, nullptr));
      if (out && out->copy_marks)
        VMM_TRY(vmm_xfer_mark(xf, out->copy_marks[3 * (l - l0)]));
      // the CTA-pair FFN (every expert >= 256 rows on average) with per-expert ready flags
      const bool walk = !no_walk && flagged && d.order_host && d.order_dev && l >= lp &&
                        (long long)n_rows * k >= 256LL * E;
      if (walk) {
        // largest experts first (the counts on the host: the first chunk's at prefill sizes): the
        // layer's misses cross PCIe in that order, and the FFN walks its resident experts first,
        // then the misses in landing order -- so the work left when the last copy lands is the
        // smallest expert's.  Issue order only: decisions and slabs are the engine's.
        for (int e = 0; e < E; ++e) by_size[e] = e;
        std::stable_sort(by_size.begin(), by_size.end(), [&](int a, int b) { return ch[a] > ch[b]; });
        for (int i = 0; i < E; ++i) rank_of[by_size[i]] = i;
        std::fill(issued.begin(), issued.end(), -1);
        VMM_TRY(vmm_xfer_issue_engine_ordered(xf, eng, d.pool, d.host_layers, E, d.arena, d.n_pinned_slots,
                                              d.slot_bytes, l, rank_of.data(), issued.data(), &n));
        // issued[]: this layer's copied experts in issue order, then -1
        std::fill(is_miss.begin(), is_miss.end(), 0);
        int n_miss = 0;
        while (n_miss < E && issued[n_miss] >= 0 && issued[n_miss] < E && !is_miss[issued[n_miss]])
          is_miss[issued[n_miss++]] = 1;
        int32_t *orow = d.order_host + (size_t)l * E;
        int w = 0;
        for (int i = 0; i < E; ++i)
          if (!is_miss[by_size[i]]) orow[w++] = by_size[i];  // resident (or not demanded) experts first
        for (int i = 0; i < n_miss; ++i) orow[w++] = issued[i];
        int32_t *odev = d.order_dev + (size_t)l * E;
        VMM_CUDA(cudaMemcpyAsync(odev, orow, sizeof(int32_t) * E, cudaMemcpyHostToDevice, st), "order H2D");
        order_of = odev;
      } else {
        VMM_TRY(vmm_xfer_issue_engine(xf, eng, d.pool, d.host_layers, E, d.arena, d.n_pinned_slots, d.slot_bytes,
                                      &n));
      }
      copies += n;
      if (out && out->copy_marks)
        VMM_TRY(vmm_xfer_mark(xf, out->copy_marks[3 * (l - l0) + 1]));
    }
    const int32_t *slot_of;
    const uint32_t *need_of = nullptr;
    bool host_rows = false;  // decode-sized layer: slot / need rows passed by value (see below)
    const int32_t *h_slot_row = nullptr;
    const uint32_t *h_need_row = nullptr;
    if (l < lp) {
      slot_of = d.pinned_slot_of + (size_t)l * E;
    } else {
      slabs.resize(demand.size());
      VMM_TRY(vmm_engine_slots(eng, l, demand.data(), (int)demand.size(), slabs.data()));
      int32_t *row = d.slot_host + (size_t)l * E;
      std::memset(row, 0, sizeof(int32_t) * E);
      for (size_t i = 0; i < demand.size(); ++i) row[demand[i]] = slabs[i] + (int32_t)d.n_pinned_slots;
      int32_t *drow = d.slot_dev + (size_t)l * E;
      // decode-sized layers hand the rows to the skinny FFN as kernel parameters
      // (vmm_grouped_swiglu_decode): no per-layer uploads in the compute stream
      host_rows = by_value_rows && (long long)n_rows * k <= 16 && flagged && d.shared == 0;
      if (!host_rows)
        VMM_CUDA(cudaMemcpyAsync(drow, row, sizeof(int32_t) * E, cudaMemcpyHostToDevice, st), "slot table H2D");
      if (flagged) {
        need.resize(demand.size());
        VMM_TRY(vmm_xfer_need(xf, slabs.data(), (int)slabs.size(), need.data()));
        uint32_t *nrow = d.need_host + (size_t)l * E;
        std::memset(nrow, 0, sizeof(uint32_t) * E);
        for (size_t i = 0; i < demand.size(); ++i) nrow[demand[i]] = need[i];
        uint32_t *ndev = d.need_dev + (size_t)l * E;
        if (host_rows) {
          h_need_row = nrow;
        } else {
          VMM_CUDA(cudaMemcpyAsync(ndev, nrow, sizeof(uint32_t) * E, cudaMemcpyHostToDevice, st), "need H2D");
        }
        need_of = ndev;
      } else {
        VMM_TRY(vmm_xfer_fence(xf, slabs.data(), (int)slabs.size(), stream));
      }
      slot_of = drow;
      h_slot_row = row;
    }
    auto c3 = clk::now();
    const int M = n_rows * k;
    // VMM_FFN_GATHER=1: the tensor-core FFN gathers its rows from xn (TMA gather4) instead of a
    // permuted copy.  Measured slower on B200 (32 gather4 issues per 16 KB A stage: 20.0 vs 10.9 ms
    // at 1.25M rows), so the permuted copy is the default.
    static const bool gather_env = std::getenv("VMM_FFN_GATHER") != nullptr;
    const bool gather = gather_env && d.ffn_done && M > 16;
    if (glue) {
      // plan and row copy done by the layer's glue launch
    } else if (gather) {
      VMM_TRY(vmm_permute_plan(d.ids, n_rows, k, E, d.off, d.src, d.pos, stream));
    } else {
      VMM_TRY(vmm_permute(d.ids, n_rows, k, E, xn, H, d.off, d.src, d.pos, d.xp, stream));
    }
    if (out && out->ffn_start)
      VMM_CUDA(cudaEventRecord((cudaEvent_t)out->ffn_start[l - l0], st), "ffn start event");
    if (host_rows)
      VMM_TRY(vmm_grouped_swiglu_decode(d.xp, d.off, E, M, H, I, d.arena,
                                        (const char *)d.arena + (size_t)2 * I * H * 2, (long long)3 * I * H,
                                        h_slot_row, h_need_row, ready, (int)d.n_pinned_slots, d.h1, d.y, stream));
    else
      VMM_TRY(vmm_grouped_swiglu_fused_ex(d.xp, d.off, E, M, H, I, d.arena,
                                          (const char *)d.arena + (size_t)2 * I * H * 2, (long long)3 * I * H,
                                          d.n_slots, slot_of, need_of, ready, (int)d.n_pinned_slots, d.ffn_done,
                                          gather ? xn : nullptr, gather ? d.src : nullptr, n_rows, d.h1, d.y,
                                          order_of, stream));
    if (out && out->ffn_end) VMM_CUDA(cudaEventRecord((cudaEvent_t)out->ffn_end[l - l0], st), "ffn end event");
    void *dst = ping ? d.out1 : d.out0;
    const int S = d.shared;
    if (S > 0) {
      // always-resident shared experts: every token through each, grouped GEMM over S groups
      const int MS = n_rows * S;
      const bool gather_s = gather_env && d.ffn_done && MS > 16;
      VMM_TRY(vmm_shared_plan(n_rows, S, d.shared_src, d.shared_off, stream));
      if (!gather_s) VMM_TRY(vmm_permute_rows(xn, d.shared_src, MS, H, d.xs, stream));
      VMM_TRY(vmm_grouped_swiglu_fused(d.xs, d.shared_off, S, MS, H, I, d.arena,
                                       (const char *)d.arena + (size_t)2 * I * H * 2, (long long)3 * I * H, d.n_slots,
                                       d.shared_slot_of + (size_t)l * S, nullptr, nullptr, 0, d.ffn_done,
                                       gather_s ? xn : nullptr, gather_s ? d.shared_src : nullptr, n_rows, d.h1s,
                                       d.ys, stream));
    }
    if (out && out->n_demand) out->n_demand[l - l0] = (int)demand.size();
    // the slabs this layer read are free for refills once its FFNs are done
    if (l >= lp && !pinned_only) VMM_TRY(vmm_xfer_layer_done(xf, l, stream));
    if (l + 1 < l1 && glue) {  // the combine runs in the next layer's glue launch
      glue_resid = cur;
    } else if (l + 1 < l1) {  // combine fused with the next layer's RMSNorm (xn is free again: consumed above)
      if (n_split) {  // first chunk only; the rest runs after the next layer's first-chunk route
        VMM_TRY(vmm_combine_norm(d.y, d.pos, d.gates, cur, n_split, k, H, nullptr, 0, 1e-6f, dst, xn, stream));
        pending_rest = true;
        rest_resid = cur;
        rest_dst = dst;
      } else {
        VMM_TRY(vmm_combine_norm(d.y, d.pos, d.gates, cur, n_rows, k, H, S > 0 ? d.ys : nullptr, S, 1e-6f, dst, xn,
                                 stream));
      }
      have_xn = true;
    } else if (S > 0) {
      VMM_TRY(vmm_combine_shared(d.y, d.pos, d.gates, cur, n_rows, k, H, d.ys, S, dst, stream));
    } else {
      VMM_TRY(vmm_combine(d.y, d.pos, d.gates, cur, n_rows, k, H, dst, stream));
    }
    cur = dst;
    ping ^= 1;
    auto c4 = clk::now();
    t_pre += us(c0, c1);
    t_sync += us(c1, c2);
    t_dec += us(c2, c3);
    t_post += us(c3, c4);
    if (emits) {
      if (split_now) VMM_CUDA(cudaEventSynchronize(ev_y), "scores sync");  // yh landed (after the full route)
      VMM_TRY(vmm_engine_emit(eng, l, yh));
      VMM_TRY(vmm_xfer_issue_engine(xf, eng, d.pool, d.host_layers, E, d.arena, d.n_pinned_slots, d.slot_bytes, &n));
      copies += n;
    }
    if (out && out->copy_marks && !pinned_only)
      VMM_TRY(vmm_xfer_mark(xf, out->copy_marks[3 * (l - l0) + 2]));
  }
  if (out) {
    out->host_us[0] = t_pre;
    out->host_us[1] = t_sync;
    out->host_us[2] = t_dec;
    out->host_us[3] = t_post;
    out->x_out = cur;
    out->copies = copies;
  }
  (void)row_bytes;
  return VMM_OK;
}

}  // extern "C"

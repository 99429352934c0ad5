// Expert transfer runtime: pinned host pool -> HBM slab arena.
//
// Makes the reference's logical transfer channel (pkg/src/moesim/pipeline.py:
// 440-494: one serial channel, issue order decided by the policy) real: every
// decided issue becomes a cudaMemcpyAsync on a dedicated copy stream, followed
// by an event and a ready-flag write.  Issues go round-robin over several copy
// streams -- 2 for the pinned host pool, 4 once HBM / NVLink sources are set
// (VMM_COPY_STREAMS=N forces N): the flag write's memory barrier stalls a
// stream between copies, and the other streams keep the link busy through the
// stall (PCIe: 52.6 -> 53.6 GB/s for back-to-back 9.44 MB copies).  Per-slab
// write-after-read and write-after-write waits keep every slab's fills and
// readers ordered across the streams.
//   * compute never reads a slab before its fill lands: per-expert ready
//     flags (the FFN spins on them), or vmm_xfer_fence, which makes the
//     compute stream wait for the newest fill among the slabs a layer reads
//     plus the newest fill of every other copy stream (FIFO per stream);
//   * a slab is never overwritten while a layer may still read it: the copy
//     into slab s first waits for the compute event of the last layer fenced
//     on s (again one wait per newer reader, FIFO on the compute stream).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vismmoe.h"

namespace vmm {
int fail(int code, const std::string &msg);
}  // namespace vmm

namespace {
int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return VMM_OK;
  return vmm::fail(VMM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

namespace {
constexpr int kRing = 8192;

// cuStreamWriteValue32 through the runtime's driver entry point (no -lcuda)
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value_fn() {
  static WriteValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(p);
  });
  return fn;
}
}  // namespace

struct vmm_xfer {
  cudaStream_t stream = nullptr;       // copy stream 0 (also the timing / marks stream)
  static constexpr int kMaxCS = 4;
  cudaStream_t cs[kMaxCS] = {};        // copy streams (cs[0] == stream)
  int ncs = 1, nact = 1;               // created / in use (2 for the host pool, 4 for HBM/NVLink sources)
  long long waited[kMaxCS] = {};       // newest reader event each copy stream already waits for
  long long last_fill[kMaxCS] = {};    // fill sequence of the newest copy on each stream
  std::vector<int8_t> slab_fill_stream;  // copy stream of each slab's newest fill
  std::vector<cudaEvent_t> fill_ev, read_ev;
  std::vector<long long> slab_fill_seq, slab_read_seq;
  long long fill_seq = 0, read_seq = 0;
  std::vector<int> pending_readers;
  double bytes = 0.0;
  long long copies = 0;
  cudaEvent_t t_first = nullptr, t_last = nullptr;
  bool timing_started = false;
  std::vector<const void *> sources;  // optional per-(layer, expert) source pointers (sharded mode)
  uint32_t *ready = nullptr;          // d [num_slabs] fill sequence flags (stream memory op after each fill)
};

extern "C" {

int vmm_xfer_create(int num_slabs, size_t slab_bytes, int max_layers, vmm_xfer **out) {
  (void)slab_bytes;
  (void)max_layers;
  auto *x = new vmm_xfer();
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  cudaError_t e = cudaStreamCreateWithPriority(&x->stream, cudaStreamNonBlocking, prio_hi);
  if (e != cudaSuccess) { delete x; return cuda_status(e, "copy stream"); }
  x->cs[0] = x->stream;
  const char *ns = std::getenv("VMM_COPY_STREAMS");
  const int want = ns ? std::atoi(ns) : 0;  // 0: automatic (2, or 4 once peer/HBM sources are set)
  x->ncs = want >= 1 ? (want > vmm_xfer::kMaxCS ? vmm_xfer::kMaxCS : want) : vmm_xfer::kMaxCS;
  x->nact = want >= 1 ? x->ncs : 2;
  for (int i = 1; i < x->ncs; ++i) {
    e = cudaStreamCreateWithPriority(&x->cs[i], cudaStreamNonBlocking, prio_hi);
    if (e != cudaSuccess) { vmm_xfer_destroy(x); return cuda_status(e, "copy stream"); }
  }
  x->fill_ev.resize(kRing);
  x->read_ev.resize(kRing);
  for (int i = 0; i < kRing; ++i) {
    if ((e = cudaEventCreateWithFlags(&x->fill_ev[i], cudaEventDisableTiming)) != cudaSuccess) break;
    if ((e = cudaEventCreateWithFlags(&x->read_ev[i], cudaEventDisableTiming)) != cudaSuccess) break;
  }
  if (e == cudaSuccess) e = cudaEventCreate(&x->t_first);
  if (e == cudaSuccess) e = cudaEventCreate(&x->t_last);
  if (e != cudaSuccess) { vmm_xfer_destroy(x); return cuda_status(e, "copy events"); }
  x->slab_fill_seq.assign(num_slabs, 0);
  x->slab_fill_stream.assign(num_slabs, 0);
  x->slab_read_seq.assign(num_slabs, 0);
  if (write_value_fn() && num_slabs > 0) {
    if ((e = cudaMalloc(&x->ready, sizeof(uint32_t) * num_slabs)) != cudaSuccess ||
        (e = cudaMemset(x->ready, 0, sizeof(uint32_t) * num_slabs)) != cudaSuccess) {
      vmm_xfer_destroy(x);
      return cuda_status(e, "ready flags");
    }
  }
  *out = x;
  return VMM_OK;
}

void vmm_xfer_destroy(vmm_xfer *x) {
  if (!x) return;
  for (int i = 0; i < vmm_xfer::kMaxCS; ++i)
    if (x->cs[i]) cudaStreamSynchronize(x->cs[i]);
  for (auto ev : x->fill_ev) if (ev) cudaEventDestroy(ev);
  for (auto ev : x->read_ev) if (ev) cudaEventDestroy(ev);
  if (x->t_first) cudaEventDestroy(x->t_first);
  if (x->t_last) cudaEventDestroy(x->t_last);
  for (int i = 0; i < vmm_xfer::kMaxCS; ++i)
    if (x->cs[i]) cudaStreamDestroy(x->cs[i]);
  if (x->ready) cudaFree(x->ready);
  delete x;
}

int vmm_xfer_copy(vmm_xfer *x, int slab, const void *h_src, void *d_dst, size_t bytes, int wait_layer) {
  (void)wait_layer;
  if (slab < 0 || slab >= (int)x->slab_fill_seq.size()) return vmm::fail(VMM_ECONTRACT, "slab out of range");
  cudaError_t e;
  const int k = (int)(x->fill_seq % x->nact);  // round-robin over the copy streams
  cudaStream_t st = x->cs[k];
  long long &waited = x->waited[k];
  // write-after-write: a previous fill of this slab still in flight on the OTHER copy stream
  // (a fill can be evicted and refilled before any layer reads it) must land first
  const long long pf = x->slab_fill_seq[slab];
  if (pf > 0 && x->slab_fill_stream[slab] != k) {
    if ((e = cudaStreamWaitEvent(st, x->fill_ev[(pf - 1) % kRing], 0)) != cudaSuccess)
      return cuda_status(e, "copy wait previous fill");
  }
  long long r = x->slab_read_seq[slab];
  if (r > waited) {  // write-after-read: the last layer that read this slab has finished
    if ((e = cudaStreamWaitEvent(st, x->read_ev[(r - 1) % kRing], 0)) != cudaSuccess)
      return cuda_status(e, "copy wait reader");
    waited = r;
  }
  if (!x->timing_started) {
    cudaEventRecord(x->t_first, x->stream);
    x->timing_started = true;
  }
  // cudaMemcpyDefault: pinned host pool (PCIe), local HBM home copy (D2D) or a
  // peer GPU's HBM home copy (NVLink P2P) -- UVA resolves the direction
  if ((e = cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyDefault, st)) != cudaSuccess)
    return cuda_status(e, "expert copy");
  x->fill_seq++;
  if (x->ready) {  // ordered after the copy, with a memory barrier: readers polling ready[] see the data
    CUresult r = write_value_fn()((CUstream)st, (CUdeviceptr)(x->ready + slab), (cuuint32_t)x->fill_seq, 0);
    if (r != CUDA_SUCCESS) return vmm::fail(VMM_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
  }
  // the fill event is recorded AFTER the flag write: a refill of this slab on another copy
  // stream waits on it (write-after-write above), so the newer fill's flag can never be
  // overwritten by this older one -- ready[slab] only moves forward
  if ((e = cudaEventRecord(x->fill_ev[(x->fill_seq - 1) % kRing], st)) != cudaSuccess)
    return cuda_status(e, "fill event");
  x->last_fill[k] = x->fill_seq;
  x->slab_fill_seq[slab] = x->fill_seq;
  x->slab_fill_stream[slab] = (int8_t)k;
  x->bytes += (double)bytes;
  x->copies++;
  return VMM_OK;
}

int vmm_xfer_fence(vmm_xfer *x, const int32_t *slabs, int n, void *compute_stream) {
  long long need = 0;
  for (int i = 0; i < n; ++i) {
    int s = slabs[i];
    if (s < 0 || s >= (int)x->slab_fill_seq.size()) continue;
    if (x->slab_fill_seq[s] > need) need = x->slab_fill_seq[s];
    x->pending_readers.push_back(s);
  }
  if (need > 0) {
    cudaError_t e = cudaStreamWaitEvent((cudaStream_t)compute_stream, x->fill_ev[(need - 1) % kRing], 0);
    if (e != cudaSuccess) return cuda_status(e, "fence wait");
    // two copy streams: older fills may sit on the other stream -- also wait for its newest fill
    // (conservative: it may be younger than needed)
    for (int k = 0; k < vmm_xfer::kMaxCS; ++k) {
      const long long f = x->last_fill[k];
      if (f > 0 && f != need) {
        e = cudaStreamWaitEvent((cudaStream_t)compute_stream, x->fill_ev[(f - 1) % kRing], 0);
        if (e != cudaSuccess) return cuda_status(e, "fence wait");
      }
    }
  }
  return VMM_OK;
}

const uint32_t *vmm_xfer_ready(vmm_xfer *x) { return x->ready; }

int vmm_xfer_need(vmm_xfer *x, const int32_t *slabs, int n, uint32_t *need) {
  if (!x->ready) return vmm::fail(VMM_ECONTRACT, "no ready flags (stream memory ops unavailable)");
  for (int i = 0; i < n; ++i) {
    int s = slabs[i];
    if (s < 0 || s >= (int)x->slab_fill_seq.size()) return vmm::fail(VMM_ECONTRACT, "slab out of range");
    need[i] = (uint32_t)x->slab_fill_seq[s];
    x->pending_readers.push_back(s);
  }
  return VMM_OK;
}

int vmm_xfer_layer_done(vmm_xfer *x, int layer, void *compute_stream) {
  (void)layer;
  if (x->pending_readers.empty()) return VMM_OK;
  x->read_seq++;
  cudaError_t e = cudaEventRecord(x->read_ev[(x->read_seq - 1) % kRing], (cudaStream_t)compute_stream);
  if (e != cudaSuccess) return cuda_status(e, "reader event");
  for (int s : x->pending_readers) x->slab_read_seq[s] = x->read_seq;
  x->pending_readers.clear();
  return VMM_OK;
}

int vmm_xfer_join(vmm_xfer *x, void *compute_stream) {
  if (x->fill_seq == 0) return VMM_OK;
  for (int k = 0; k < vmm_xfer::kMaxCS; ++k) {
    const long long f = x->last_fill[k];
    if (f <= 0) continue;
    cudaError_t e = cudaStreamWaitEvent((cudaStream_t)compute_stream, x->fill_ev[(f - 1) % kRing], 0);
    if (e != cudaSuccess) return cuda_status(e, "join copy stream");
  }
  return VMM_OK;
}

int vmm_xfer_sync(vmm_xfer *x) {
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < vmm_xfer::kMaxCS && e == cudaSuccess; ++i)
    if (x->cs[i]) e = cudaStreamSynchronize(x->cs[i]);
  return cuda_status(e, "copy sync");
}

int vmm_xfer_stats(vmm_xfer *x, double *bytes, double *busy_ms, long long *copies) {
  *bytes = x->bytes;
  *copies = x->copies;
  *busy_ms = 0.0;
  if (x->timing_started) {
    for (int i = 1; i < vmm_xfer::kMaxCS; ++i)  // the window ends when every copy stream is done
      if (x->last_fill[i] > 0) cudaStreamWaitEvent(x->stream, x->fill_ev[(x->last_fill[i] - 1) % kRing], 0);
    cudaEventRecord(x->t_last, x->stream);
    cudaEventSynchronize(x->t_last);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, x->t_first, x->t_last);
    *busy_ms = ms;
  }
  return VMM_OK;
}

int vmm_xfer_reset_stats(vmm_xfer *x) {
  x->bytes = 0.0;
  x->copies = 0;
  x->timing_started = false;
  return VMM_OK;
}

void *vmm_xfer_stream(vmm_xfer *x) { return (void *)x->stream; }

// record `ev` once every copy issued so far has landed (diagnostic marks; joins stream 1 into stream 0)
int vmm_xfer_mark(vmm_xfer *x, void *ev) {
  for (int i = 1; i < vmm_xfer::kMaxCS; ++i) {
    if (x->last_fill[i] <= 0) continue;
    cudaError_t e = cudaStreamWaitEvent(x->stream, x->fill_ev[(x->last_fill[i] - 1) % kRing], 0);
    if (e != cudaSuccess) return cuda_status(e, "mark join");
  }
  return cuda_status(cudaEventRecord((cudaEvent_t)ev, x->stream), "copy mark");
}

int vmm_xfer_set_sources(vmm_xfer *x, const void *const *h_table, long long n) {
  x->sources.assign(h_table, h_table + n);
  // HBM / NVLink sources: the per-copy flag stall is a larger share of a ~10 us copy -> 4 streams
  if (!std::getenv("VMM_COPY_STREAMS")) x->nact = x->ncs;
  return VMM_OK;
}

int vmm_engine_copies(vmm_engine *e, int32_t *out, int cap);

int vmm_xfer_issue_engine_ordered(vmm_xfer *x, vmm_engine *e, const void *h_pool, int host_layers, int experts,
                                  void *d_arena, long long slab_offset, size_t slot_bytes, int layer_now,
                                  const int32_t *h_rank, int32_t *h_issued_experts, int *n_issued) {
  // every decided copy, in the engine's order
  std::vector<int32_t> all;
  int32_t buf[3 * 256];
  for (;;) {
    int n = vmm_engine_copies(e, buf, 256);
    if (n <= 0) break;
    all.insert(all.end(), buf, buf + 3 * n);
  }
  const int n = (int)all.size() / 3;
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  if (h_rank && n > 1) {
    // Physical issue order only (the decisions, slabs and logical clock are the engine's): this
    // layer's copies by h_rank (lowest first), then the rest in decided order.  Kept as decided
    // when two copies target one slab, so a slab's fills land in decided order.
    const int nslabs = (int)x->slab_fill_seq.size();
    std::vector<char> seen((size_t)nslabs, 0);
    bool distinct = true;
    for (int i = 0; i < n && distinct; ++i) {
      const int slab = all[3 * i + 2];
      if (slab < 0 || slab >= nslabs || seen[slab]) distinct = false;
      else seen[slab] = 1;
    }
    if (distinct)
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
        const bool ca = all[3 * a] == layer_now, cb = all[3 * b] == layer_now;
        if (ca != cb) return ca;
        if (!ca) return false;
        return h_rank[all[3 * a + 1]] < h_rank[all[3 * b + 1]];
      });
  }
  int n_now = 0;
  for (int j = 0; j < n; ++j) {
    const int i = idx[j];
    int layer = all[3 * i], expert = all[3 * i + 1], slab = all[3 * i + 2];
    const char *src = h_pool ? (const char *)h_pool + ((size_t)(layer % host_layers) * experts + expert) * slot_bytes
                             : (const char *)x->sources.at((size_t)layer * experts + expert);
    char *dst = (char *)d_arena + (size_t)(slab_offset + slab) * slot_bytes;
    int st = vmm_xfer_copy(x, slab, src, dst, slot_bytes, 0);
    if (st) return st;
    if (h_issued_experts && layer == layer_now && n_now < experts) h_issued_experts[n_now++] = expert;
  }
  if (n_issued) *n_issued = n;
  return VMM_OK;
}

int vmm_xfer_issue_engine(vmm_xfer *x, vmm_engine *e, const void *h_pool, int host_layers, int experts,
                          void *d_arena, long long slab_offset, size_t slot_bytes, int *n_issued) {
  return vmm_xfer_issue_engine_ordered(x, e, h_pool, host_layers, experts, d_arena, slab_offset, slot_bytes, -1,
                                       nullptr, nullptr, n_issued);
}

}  // extern "C"

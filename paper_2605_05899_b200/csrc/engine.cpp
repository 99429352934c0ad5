// Expert-cache policy and logical-clock engine (host C++, single owner).
//
// Mirrors the reference decision path so that hit/miss/eviction/issue
// sequences are bit-identical:
//   Cache  : pkg/src/moesim/cache.py:78-278 (slab table, residency classes,
//            monotone upgrade, Expired-only eviction by (priority, layer,
//            expert) or FIFO insertion order, free list yielding slab 0 first,
//            lazily validated victim heap :124-153, grace window :246-278)
//   Engine : pkg/src/moesim/pipeline.py:382-760 (serial channel :440-494,
//            demand-first issue, prefetch claims its slab at issue time
//            :435-438, sorted-demand lookups :559-651, reactive :653-691,
//            window emission :498-542, exposed time :351-374)
// The policy is inherently sequential and latency-bound (one decision per
// expert), so it runs on the host next to the copy engine; the device side
// of the cache is the slab arena + per-layer slot table it produces.
// Compiled with -ffp-contract=off: every double op rounds like CPython's.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/vismmoe.h"

namespace vmm {
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
}  // namespace vmm

namespace {

enum { FREE = 0, LOADING = 1, RESIDENT = 2 };
enum { EXPIRED = 0, SPECULATIVE = 1, REQUIRED = 2 };
const double kNaN = std::numeric_limits<double>::quiet_NaN();
const double kInf = std::numeric_limits<double>::infinity();

struct Slab {
  int key = -1;  // layer * E + expert
  int state = FREE;
  int cls = EXPIRED;
  double pri = 0.0;
  double ready = kNaN;  // NaN == None
  bool has_ready = false;
  long long last_step = -1;
  bool executed = false;
  long long seq = -1;
};

struct HeapItem {
  double pri;
  int layer, expert;
  long long seq;
  int slab, key;
};

struct Cache {
  int n, E, n_keys;
  bool fifo;
  std::vector<Slab> slabs;
  std::unordered_map<int, int> where;
  long long step = 0, evictions = 0, counter = 0;
  std::vector<int> free_list;
  struct Cmp {
    bool fifo;
    // std::priority_queue is a max-heap: return true if a should come AFTER b
    bool operator()(const HeapItem &a, const HeapItem &b) const {
      if (fifo) {
        if (a.seq != b.seq) return a.seq > b.seq;
      } else {
        if (a.pri != b.pri) return a.pri > b.pri;
        if (a.layer != b.layer) return a.layer > b.layer;
        if (a.expert != b.expert) return a.expert > b.expert;
      }
      if (a.slab != b.slab) return a.slab > b.slab;
      return a.key > b.key;
    }
  };
  std::priority_queue<HeapItem, std::vector<HeapItem>, Cmp> heap;

  Cache(int n_, int E_, bool fifo_) : n(n_), E(E_), fifo(fifo_), slabs(n_), heap(Cmp{fifo_}) {
    for (int i = n - 1; i >= 0; --i) free_list.push_back(i);
  }
  int layer_of(int key) const { return key / E; }
  int expert_of(int key) const { return key % E; }

  void push(int i) {
    const Slab &s = slabs[i];
    heap.push(HeapItem{s.pri, layer_of(s.key), expert_of(s.key), s.seq, i, s.key});
  }
  bool valid(const HeapItem &h) const {
    const Slab &s = slabs[h.slab];
    if (!(s.state == RESIDENT && s.cls == EXPIRED && s.key == h.key)) return false;
    if (fifo) return s.seq == h.seq;
    return s.pri == h.pri && layer_of(s.key) == h.layer && expert_of(s.key) == h.expert;
  }
  int victim() {
    while (!heap.empty()) {
      if (valid(heap.top())) return heap.top().slab;
      heap.pop();
    }
    return -1;
  }
  int find(int key) const {
    auto it = where.find(key);
    return it == where.end() ? -1 : it->second;
  }
  // 0 miss / 1 hit / 2 in-flight
  int lookup(int key, double *ready) const {
    int i = find(key);
    if (i < 0) { *ready = kNaN; return 0; }
    *ready = slabs[i].has_ready ? slabs[i].ready : kNaN;
    return slabs[i].state == RESIDENT ? 1 : 2;
  }
  // status 0 already resident / 1 enqueued / 2 rejected
  int request(int key, double pri, int cls, int *slab_out, int *evicted) {
    *evicted = -1;
    int i = find(key);
    if (i >= 0) {
      Slab &s = slabs[i];
      if (cls > s.cls) s.cls = cls;
      s.pri = pri;
      s.last_step = step;
      s.executed = false;
      *slab_out = i;
      return 0;
    }
    if (!free_list.empty()) {
      i = free_list.back();
      free_list.pop_back();
    } else {
      i = victim();
      if (i < 0) { *slab_out = -1; return 2; }
      Slab &v = slabs[i];
      *evicted = v.key;
      evictions++;
      where.erase(v.key);
      v.key = -1; v.state = FREE; v.has_ready = false; v.ready = kNaN; v.executed = false;
    }
    Slab &s = slabs[i];
    s.key = key; s.state = LOADING; s.cls = cls; s.pri = pri;
    s.has_ready = false; s.ready = kNaN; s.last_step = step; s.executed = false;
    s.seq = counter++;
    where[key] = i;
    *slab_out = i;
    return 1;
  }
  int set_ready(int key, double t) {
    int i = find(key);
    if (i < 0 || slabs[i].state != LOADING) return vmm::fail(VMM_ECONTRACT, "set_ready requires a loading entry");
    slabs[i].ready = t; slabs[i].has_ready = true;
    return VMM_OK;
  }
  int complete(int key, double t) {
    int i = find(key);
    if (i < 0 || slabs[i].state != LOADING) return vmm::fail(VMM_ECONTRACT, "complete_load requires a loading entry");
    slabs[i].state = RESIDENT; slabs[i].ready = t; slabs[i].has_ready = true;
    return VMM_OK;
  }
  int cancel(int key) {
    int i = find(key);
    if (i < 0 || slabs[i].state != LOADING) return vmm::fail(VMM_ECONTRACT, "cancel_load requires a loading entry");
    where.erase(key);
    Slab &s = slabs[i];
    s.key = -1; s.state = FREE; s.has_ready = false; s.ready = kNaN;
    free_list.push_back(i);
    return VMM_OK;
  }
  int executed(int key) {
    int i = find(key);
    if (i < 0 || slabs[i].state != RESIDENT) return vmm::fail(VMM_ECONTRACT, "mark_executed requires a resident key");
    slabs[i].cls = EXPIRED; slabs[i].executed = true;
    push(i);
    return VMM_OK;
  }
  // window: membership test; fresh: optional priority per key (nullptr = none)
  template <class InWindow, class Fresh>
  void reclassify(InWindow in_window, long long grace, Fresh fresh) {
    step++;
    for (int i = 0; i < n; ++i) {
      Slab &s = slabs[i];
      if (s.state != RESIDENT) continue;
      double p;
      if (fresh(s.key, &p)) s.pri = p;
      if (in_window(s.key)) {
        s.cls = REQUIRED; s.last_step = step; s.executed = false;
      } else if (!s.executed && s.last_step >= 0 && step - s.last_step <= grace) {
        s.cls = SPECULATIVE;
      } else {
        s.cls = EXPIRED;
        push(i);
      }
    }
  }
};

}  // namespace

// ===========================================================================
// Engine
// ===========================================================================
struct vmm_engine {
  vmm_engine_config c;
  std::vector<double> decay;
  Cache cache;
  int busy = -1;
  double busy_until = 0.0;
  std::deque<int> demand_q;
  struct Pend { double pri; long long seq; };
  std::unordered_map<int, Pend> pending;
  long long pseq = 0;
  std::vector<std::pair<double, double>> xfer, comp;
  double t_comp = 0.0, t_xfer = 0.0;
  long long hits = 0, misses = 0, stalls = 0, rejected = 0, on_demand = 0, inflight_waits = 0;
  std::vector<std::array<double, 8>> layer_rows;
  std::vector<vmm_engine_event> events;  // parity log (reference event_log)
  size_t events_drained = 0;
  std::vector<std::array<int32_t, 3>> copies;  // (layer, expert, slab) in issue order
  size_t copies_drained = 0;
  size_t rows_drained = 0;
  double cursor = 0.0;
  double step_start = 0.0;
  double prefill_ms = kNaN;
  std::vector<double> decode_ms;
  bool begun = false;

  explicit vmm_engine(const vmm_engine_config &cfg)
      : c(cfg), decay(cfg.decay, cfg.decay + (cfg.window > 0 ? cfg.window : 0)),
        cache(cfg.num_slabs, cfg.experts, cfg.victim_fifo != 0) {}

  int key(int l, int e) const { return l * c.experts + e; }

  void log(double t, int kind, int k, int slab) {
    events.push_back(vmm_engine_event{t, kind, k / c.experts, k % c.experts, slab});
  }

  void start(int k, double t) {
    busy = k;
    busy_until = t + c.transfer_ms;
    cache.set_ready(k, busy_until);
    xfer.emplace_back(t, busy_until);
    t_xfer += c.transfer_ms;
    int slab = cache.find(k);
    log(t, 0, k, slab);
    copies.push_back({k / c.experts, k % c.experts, slab});
  }

  void issue(double t) {
    while (busy < 0) {
      if (!demand_q.empty()) {
        int k = demand_q.front();
        demand_q.pop_front();
        start(k, t);
        return;
      }
      if (pending.empty()) return;
      int best = -1;
      Pend bp{0, 0};
      for (auto &kv : pending) {
        int k = kv.first;
        const Pend &p = kv.second;
        if (best < 0) { best = k; bp = p; continue; }
        // key = (-pri, layer, expert, seq)
        double a = -p.pri, b = -bp.pri;
        bool less;
        if (a != b) less = a < b;
        else if (k / c.experts != best / c.experts) less = (k / c.experts) < (best / c.experts);
        else if (k % c.experts != best % c.experts) less = (k % c.experts) < (best % c.experts);
        else less = p.seq < bp.seq;
        if (less) { best = k; bp = p; }
      }
      pending.erase(best);
      double r;
      if (cache.lookup(best, &r) != 0) continue;
      int slab, ev;
      int st = cache.request(best, bp.pri, REQUIRED, &slab, &ev);
      if (st == 2) { rejected++; continue; }
      if (ev >= 0) log(t, 2, ev, slab);
      start(best, t);
    }
  }

  void run_until(double t) {
    while (busy >= 0 && busy_until <= t) {
      int k = busy;
      double r = busy_until;
      busy = -1;
      cache.complete(k, r);
      log(r, 1, k, cache.find(k));
      issue(r);
    }
  }

  int wait_resident(int k, double t, double *ready) {
    run_until(t);
    for (;;) {
      int i = cache.find(k);
      if (i >= 0 && cache.slabs[i].state == RESIDENT) {
        *ready = cache.slabs[i].has_ready ? cache.slabs[i].ready : 0.0;
        return VMM_OK;
      }
      if (busy < 0)
        return vmm::fail(VMM_ESIMULATION, "deadlock waiting for expert ExpertRef(layer=" + std::to_string(k / c.experts) +
                                              ", expert=" + std::to_string(k % c.experts) + ")");
      run_until(busy_until);
    }
  }

  // predictor emission (pipeline.py:498-542)
  void emit(int ctx, double t, const double *y) {
    run_until(t);
    const int E = c.experts;
    int budget = c.budget < E ? c.budget : E;
    std::vector<int> order(E);
    for (int e = 0; e < E; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      double ya = -y[a], yb = -y[b];
      if (ya != yb) return ya < yb;
      return a < b;
    });
    std::vector<int> cands;
    for (int i = 0; i < budget; ++i)
      if (y[order[i]] > 0.0) cands.push_back(order[i]);
    std::vector<std::pair<int, double>> win;  // (key, pri)
    std::unordered_map<int, double> pri;
    for (int d = 1; d <= c.window; ++d) {
      int l2 = ctx + d;
      if (l2 > c.layers - 1) break;
      if (l2 < c.l_pinned) continue;
      double w = decay[d - 1];
      for (int e : cands) {
        int k = key(l2, e);
        double p = y[e] * w;
        if (pri.find(k) == pri.end()) win.emplace_back(k, p);
        pri[k] = p;
      }
    }
    cache.reclassify([&](int k) { return pri.find(k) != pri.end(); }, c.speculative_grace,
                     [&](int k, double *p) { *p = y[k % E]; return true; });
    std::sort(win.begin(), win.end(), [&](const std::pair<int, double> &a, const std::pair<int, double> &b) {
      double pa = -a.second, pb = -b.second;
      if (pa != pb) return pa < pb;
      if (a.first / E != b.first / E) return a.first / E < b.first / E;
      return a.first % E < b.first % E;
    });
    for (auto &kp : win) {
      double r;
      if (cache.lookup(kp.first, &r) != 0) {
        int slab, ev;
        cache.request(kp.first, kp.second, REQUIRED, &slab, &ev);
        continue;
      }
      auto it = pending.find(kp.first);
      if (it == pending.end()) pending[kp.first] = Pend{kp.second, pseq++};
      else it->second.pri = kp.second;
    }
    for (auto it = pending.begin(); it != pending.end();) {
      if (pri.find(it->first) == pri.end()) it = pending.erase(it);
      else ++it;
    }
    if (busy < 0) issue(t);
  }

  double compute(double start, long long n) {
    double dur = (double)n * c.gpu_ms;
    if (dur > 0) comp.emplace_back(start, start + dur);
    t_comp += dur;
    return start + dur;
  }

  void row(int phase, int step, int layer, double s, double e, double stall, int xf, int h) {
    layer_rows.push_back({(double)phase, (double)step, (double)layer, s, e, stall, (double)xf, (double)h});
  }

  int pinned_layer(int layer, int n_demand, int phase, int step) {
    double end = compute(cursor, (long long)n_demand + c.shared);
    row(phase, step, layer, cursor, end, 0.0, 0, 0);
    cursor = end;
    return VMM_OK;
  }

  int cached_layer(int layer, const int32_t *dem, int n, int phase, int step) {
    const double t0 = cursor;
    run_until(t0);
    int lh = 0, lx = 0;
    double stall = 0.0;
    std::vector<int> run;
    double horizon = busy >= 0 ? busy_until : t0;
    double q = 0.0;
    for (size_t i = 0; i < demand_q.size(); ++i) q += c.transfer_ms;
    horizon += q;
    for (int i = 0; i < n; ++i) {
      int k = key(layer, dem[i]);
      double ready;
      int st = cache.lookup(k, &ready);
      int slab, ev;
      if (st == 1) {
        hits++; lh++;
        cache.request(k, kInf, REQUIRED, &slab, &ev);
        run.push_back(k);
        continue;
      }
      misses++; lx++;
      if (st == 2 && !std::isnan(ready)) {
        inflight_waits++;
        cache.request(k, kInf, REQUIRED, &slab, &ev);
        run.push_back(k);
        continue;
      }
      pending.erase(k);
      int rs = cache.request(k, kInf, REQUIRED, &slab, &ev);
      if (rs == 2) {
        rejected++;
        return vmm::fail(VMM_ESIMULATION, "cache too small for layer " + std::to_string(layer) +
                                              " demand (no evictable slab)");
      }
      if (ev >= 0) log(t0, 2, ev, slab);
      on_demand++;
      demand_q.push_back(k);
      if (busy < 0) issue(t0);
      horizon = (horizon > t0 ? horizon : t0) + c.transfer_ms;
      run.push_back(k);
    }
    double cur = cursor;
    for (int k : run) {
      double r;
      int st = wait_resident(k, cur, &r);
      if (st) return st;
      double start = cur > r ? cur : r;
      if (start > cur) { stall += start - cur; stalls++; }
      cur = compute(start, 1);
    }
    if (c.shared) cur = compute(cur, c.shared);
    for (int k : run) cache.executed(k);
    row(phase, step, layer, t0, cur, stall, lx, lh);
    cursor = cur;
    return VMM_OK;
  }

  int reactive_layer(int layer, const int32_t *dem, int n, int phase, int step) {
    const double t0 = cursor;
    double cur = cursor;
    int lh = 0, lx = 0;
    double stall = 0.0;
    std::vector<int> run;
    for (int i = 0; i < n; ++i) {
      int k = key(layer, dem[i]);
      double ready;
      int slab, ev;
      if (cache.lookup(k, &ready) == 1) {
        hits++; lh++;
        cache.request(k, kInf, REQUIRED, &slab, &ev);
      } else {
        misses++; on_demand++; lx++;
        int rs = cache.request(k, kInf, REQUIRED, &slab, &ev);
        if (rs == 2)
          return vmm::fail(VMM_ESIMULATION, "cache too small for layer " + std::to_string(layer) +
                                                " demand (no evictable slab)");
        xfer.emplace_back(cur, cur + c.transfer_ms);
        t_xfer += c.transfer_ms;
        cache.set_ready(k, cur + c.transfer_ms);
        copies.push_back({layer, dem[i], slab});
        cache.complete(k, cur + c.transfer_ms);
        stall += c.transfer_ms;
        stalls++;
        cur += c.transfer_ms;
      }
      cur = compute(cur, 1);
      run.push_back(k);
    }
    if (c.shared) cur = compute(cur, c.shared);
    for (int k : run) cache.executed(k);
    row(phase, step, layer, t0, cur, stall, lx, lh);
    cursor = cur;
    return VMM_OK;
  }
};

namespace {

double exposed_time(const std::vector<std::pair<double, double>> &tr, const std::vector<std::pair<double, double>> &cp) {
  double out = 0.0;
  size_t ci = 0;
  for (auto &x : tr) {
    double ts = x.first, te = x.second;
    if (te <= ts) continue;
    while (ci < cp.size() && cp[ci].second <= ts) ci++;
    double t = ts;
    size_t j = ci;
    while (j < cp.size() && cp[j].first < te && t < te) {
      double cs = cp[j].first, ce = cp[j].second;
      if (cs > t) out += (cs < te ? cs : te) - t;
      double m = ce < te ? ce : te;
      t = t > m ? t : m;
      j++;
    }
    if (t < te) out += te - t;
  }
  return out;
}

}  // namespace

extern "C" {

int vmm_engine_create(const vmm_engine_config *cfg, vmm_engine **out) {
  if (!cfg || !out) return vmm::fail(VMM_ECONTRACT, "null argument");
  if (cfg->num_slabs < 1) return vmm::fail(VMM_ECONTRACT, "num_slabs must be >= 1");
  if (cfg->experts < 1 || cfg->layers < 1) return vmm::fail(VMM_EVALIDATION, "layers and experts must be >= 1");
  if (cfg->prefetching && cfg->window > 0 && !cfg->decay) return vmm::fail(VMM_ECONTRACT, "decay table required");
  try {
    *out = new vmm_engine(*cfg);
  } catch (...) {
    return vmm::fail(VMM_ECONTRACT, "engine allocation failed");
  }
  return VMM_OK;
}

void vmm_engine_destroy(vmm_engine *e) { delete e; }

int vmm_engine_begin(vmm_engine *e, const double *y) {
  if (e->begun) return vmm::fail(VMM_ECONTRACT, "engine already begun");
  e->begun = true;
  double boot = e->c.boot_ms;
  if (boot > 0) e->comp.emplace_back(0.0, boot);
  e->cursor = boot;
  if (e->c.prefetching && e->c.l_pinned > 0) {
    if (!y) return vmm::fail(VMM_ECONTRACT, "boot emission needs predictor scores");
    e->emit(e->c.l_pinned - 1, boot, y);
  }
  return VMM_OK;
}

int vmm_engine_emits(const vmm_engine *e, int layer, int phase) {
  if (!e->c.prefetching) return 0;
  if (layer < e->c.l_pinned) return (phase == 1 && layer == e->c.l_pinned - 1) ? 1 : 0;
  return layer < e->c.layers - 1 ? 1 : 0;
}

int vmm_engine_layer(vmm_engine *e, int layer, const int32_t *dem, int n, int phase, int step, const double *y) {
  if (!e->begun) return vmm::fail(VMM_ECONTRACT, "engine not begun");
  if (layer < 0 || layer >= e->c.layers) return vmm::fail(VMM_ETRACE, "trace has no layer " + std::to_string(layer));
  if (phase == 1 && layer == 0) {
    if (std::isnan(e->prefill_ms)) e->prefill_ms = e->cursor;
    e->step_start = e->cursor;
  }
  int st;
  if (layer < e->c.l_pinned) st = e->pinned_layer(layer, n, phase, step);
  else if (e->c.reactive) st = e->reactive_layer(layer, dem, n, phase, step);
  else st = e->cached_layer(layer, dem, n, phase, step);
  if (st) return st;
  // with y == NULL an emitting layer defers its emission to vmm_engine_emit
  if (y && vmm_engine_emits(e, layer, phase)) e->emit(layer, e->cursor, y);
  return VMM_OK;
}

int vmm_engine_emit(vmm_engine *e, int layer, const double *y) {
  if (!y) return vmm::fail(VMM_ECONTRACT, "emission needs predictor scores");
  e->emit(layer, e->cursor, y);
  return VMM_OK;
}

int vmm_engine_slots(const vmm_engine *e, int layer, const int32_t *demand, int n, int32_t *out) {
  for (int i = 0; i < n; ++i) {
    int s = e->cache.find(e->key(layer, demand[i]));
    if (s < 0 || e->cache.slabs[s].state != RESIDENT)
      return vmm::fail(VMM_ECONTRACT, "expert (" + std::to_string(layer) + ", " + std::to_string(demand[i]) +
                                          ") is not resident after its layer ran");
    out[i] = s;
  }
  return VMM_OK;
}

int vmm_engine_end_step(vmm_engine *e) {
  e->decode_ms.push_back(e->cursor - e->step_start);
  return VMM_OK;
}

int vmm_engine_finish(vmm_engine *e, vmm_engine_report *r) {
  std::memset(r, 0, sizeof(*r));
  r->makespan = e->cursor;
  r->total_compute = e->t_comp;
  r->total_transfer = e->t_xfer;
  r->exposed_transfer = exposed_time(e->xfer, e->comp);
  r->prefill_ms = std::isnan(e->prefill_ms) ? e->cursor : e->prefill_ms;
  r->hits = e->hits; r->misses = e->misses; r->stalls = e->stalls; r->rejected_loads = e->rejected;
  r->on_demand_transfers = e->on_demand; r->inflight_waits = e->inflight_waits;
  r->evictions = e->cache.evictions;
  r->decode_steps = (int)e->decode_ms.size();
  return VMM_OK;
}

int vmm_engine_decode_ms(const vmm_engine *e, double *out, int cap) {
  int n = (int)e->decode_ms.size();
  for (int i = 0; i < n && i < cap; ++i) out[i] = e->decode_ms[i];
  return n;
}

int vmm_engine_events(vmm_engine *e, vmm_engine_event *out, int cap) {
  int n = 0;
  while (e->events_drained < e->events.size() && n < cap) out[n++] = e->events[e->events_drained++];
  return n;
}

int vmm_engine_pending_events(const vmm_engine *e) { return (int)(e->events.size() - e->events_drained); }

int vmm_engine_copies(vmm_engine *e, int32_t *out, int cap) {
  int n = 0;
  while (e->copies_drained < e->copies.size() && n < cap) {
    const auto &c = e->copies[e->copies_drained++];
    out[3 * n] = c[0]; out[3 * n + 1] = c[1]; out[3 * n + 2] = c[2];
    n++;
  }
  return n;
}

int vmm_engine_layer_stats(vmm_engine *e, double *out, int cap) {
  int n = 0;
  while (e->rows_drained < e->layer_rows.size() && n < cap) {
    std::memcpy(out + 8 * n, e->layer_rows[e->rows_drained].data(), 8 * sizeof(double));
    e->rows_drained++;
    n++;
  }
  return n;
}

int vmm_engine_slab_of(const vmm_engine *e, int layer, int expert) {
  return e->cache.find(e->key(layer, expert));
}

int vmm_engine_slab(const vmm_engine *e, int slab, int *layer, int *expert, int *state, int *cls, double *priority,
                    double *ready) {
  if (slab < 0 || slab >= e->cache.n) return vmm::fail(VMM_ECONTRACT, "slab out of range");
  const Slab &s = e->cache.slabs[slab];
  *layer = s.key < 0 ? -1 : s.key / e->c.experts;
  *expert = s.key < 0 ? -1 : s.key % e->c.experts;
  *state = s.state; *cls = s.cls; *priority = s.pri;
  *ready = s.has_ready ? s.ready : kNaN;
  return VMM_OK;
}

// ---------------------------------------------------------------------------
// standalone cache (ExpertCache drop-in)
// ---------------------------------------------------------------------------
struct vmm_cache {
  Cache c;
  vmm_cache(int n, bool fifo) : c(n, 1 << 20, fifo) {}
};

static inline int ckey(int layer, int expert) { return layer * (1 << 20) + expert; }

int vmm_cache_create(int num_slabs, int fifo, vmm_cache **out) {
  if (num_slabs < 1) return vmm::fail(VMM_ECONTRACT, "num_slabs must be >= 1");
  *out = new vmm_cache(num_slabs, fifo != 0);
  return VMM_OK;
}
void vmm_cache_destroy(vmm_cache *c) { delete c; }
int vmm_cache_lookup(const vmm_cache *c, int layer, int expert, double *ready) {
  return c->c.lookup(ckey(layer, expert), ready);
}
int vmm_cache_request(vmm_cache *c, int layer, int expert, double pri, int cls, int *status, int *slab,
                      int *ev_layer, int *ev_expert) {
  if (cls != SPECULATIVE && cls != REQUIRED) return vmm::fail(VMM_ECONTRACT, "cannot request a load with class Expired");
  int ev;
  *status = c->c.request(ckey(layer, expert), pri, cls, slab, &ev);
  *ev_layer = ev < 0 ? -1 : ev / (1 << 20);
  *ev_expert = ev < 0 ? -1 : ev % (1 << 20);
  return VMM_OK;
}
int vmm_cache_set_ready(vmm_cache *c, int layer, int expert, double t) { return c->c.set_ready(ckey(layer, expert), t); }
int vmm_cache_complete(vmm_cache *c, int layer, int expert, double t) { return c->c.complete(ckey(layer, expert), t); }
int vmm_cache_cancel(vmm_cache *c, int layer, int expert) { return c->c.cancel(ckey(layer, expert)); }
int vmm_cache_executed(vmm_cache *c, int layer, int expert) { return c->c.executed(ckey(layer, expert)); }
int vmm_cache_reclassify(vmm_cache *c, const int32_t *win, int n, int grace, const int32_t *pk, const double *pv,
                         int np) {
  std::unordered_map<int, char> w;
  for (int i = 0; i < n; ++i) w[ckey(win[2 * i], win[2 * i + 1])] = 1;
  std::unordered_map<int, double> p;
  for (int i = 0; i < np; ++i) p[ckey(pk[2 * i], pk[2 * i + 1])] = pv[i];
  c->c.reclassify([&](int k) { return w.find(k) != w.end(); }, grace,
                  [&](int k, double *v) {
                    auto it = p.find(k);
                    if (it == p.end()) return false;
                    *v = it->second;
                    return true;
                  });
  return VMM_OK;
}
int vmm_cache_select_victim(vmm_cache *c) { return c->c.victim(); }
int vmm_cache_info(const vmm_cache *c, long long *evictions, int *occupancy, int *step) {
  *evictions = c->c.evictions;
  *occupancy = (int)c->c.where.size();
  *step = (int)c->c.step;
  return VMM_OK;
}
int vmm_cache_slab(const vmm_cache *c, int slab, int *layer, int *expert, int *state, int *cls, double *priority,
                   double *ready, int *last_window_step, int *executed, int *seq) {
  if (slab < 0 || slab >= c->c.n) return vmm::fail(VMM_ECONTRACT, "slab out of range");
  const Slab &s = c->c.slabs[slab];
  *layer = s.key < 0 ? -1 : s.key / (1 << 20);
  *expert = s.key < 0 ? -1 : s.key % (1 << 20);
  *state = s.state; *cls = s.cls; *priority = s.pri;
  *ready = s.has_ready ? s.ready : kNaN;
  *last_window_step = (int)s.last_step; *executed = s.executed; *seq = (int)s.seq;
  return VMM_OK;
}

/* slab holding (layer, expert), or -1 (ExpertCache.entry, cache.py:112-114) */
int vmm_cache_find(const vmm_cache *c, int layer, int expert) {
  return c->c.find(ckey(layer, expert));
}

/* all slabs at once (one call per `slabs` snapshot): ints [n][7] = layer,
 * expert, state, cls, last_window_step, executed, seq; doubles [n][2] =
 * priority, ready (NaN if none).  Returns n. */
int vmm_cache_slabs(const vmm_cache *c, int32_t *h_ints, double *h_dbls, int cap) {
  if (cap < c->c.n) return -vmm::fail(VMM_ECONTRACT, "slab snapshot buffer too small");
  for (int i = 0; i < c->c.n; ++i) {
    const Slab &s = c->c.slabs[i];
    int32_t *o = h_ints + 7 * (size_t)i;
    o[0] = s.key < 0 ? -1 : (int32_t)(s.key / (1 << 20));
    o[1] = s.key < 0 ? -1 : (int32_t)(s.key % (1 << 20));
    o[2] = s.state; o[3] = s.cls; o[4] = (int32_t)s.last_step; o[5] = s.executed ? 1 : 0; o[6] = (int32_t)s.seq;
    h_dbls[2 * (size_t)i] = s.pri;
    h_dbls[2 * (size_t)i + 1] = s.has_ready ? s.ready : kNaN;
  }
  return c->c.n;
}

}  // extern "C"

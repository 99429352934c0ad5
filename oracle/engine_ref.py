"""Oracle: slab cache policy + two-stream logical-clock engine.

Independent Python restatement of the reference's decision path:

* slab cache   `pkg/src/moesim/cache.py:78-278`  (classes Required/Speculative/
  Expired, monotone upgrade, Expired-only eviction by (priority, layer, expert)
  or FIFO insertion order, free list yielding slab 0 first, grace window)
* engine       `pkg/src/moesim/pipeline.py:382-760` (serial transfer channel,
  demand-first issue, prefetch claims a slab only at issue time, per-layer
  sorted-demand lookups, stall accounting, window emission, decode loop)
* exposed time `pkg/src/moesim/pipeline.py:351-374`

Hybrid CPU dispatch (pipeline.py:587-628) is out of scope for the device path
(no CPU fallback) and is not restated.  Predictor scores come from a callback
`scores(context_layer, token_ids) -> float64[E]` so any predictor (oracle,
history, MLP, recorded device output) can drive the replay.
"""
from __future__ import annotations

import heapq
import math

REQ, SPEC, EXP = 2, 1, 0  # residency class ranks
FREE, LOADING, RESIDENT = 0, 1, 2


class OracleSimError(RuntimeError):
    pass


class Slab:
    __slots__ = ("idx", "key", "state", "rank", "pri", "ready", "last_step", "done", "seq")

    def __init__(self, idx):
        self.idx = idx
        self.key = None
        self.state = FREE
        self.rank = EXP
        self.pri = 0.0
        self.ready = None
        self.last_step = -1
        self.done = False
        self.seq = -1


class SlabCache:
    def __init__(self, n, fifo=False):
        if n < 1:
            raise OracleSimError("num_slabs must be >= 1")
        self.n = n
        self.fifo = fifo
        self.slabs = [Slab(i) for i in range(n)]
        self.where = {}
        self.step = 0
        self.evictions = 0
        self.counter = 0
        self.free = list(range(n - 1, -1, -1))
        self.heap = []

    def _okey(self, s):
        return (s.seq,) if self.fifo else (s.pri, s.key[0], s.key[1])

    def _push(self, s):
        heapq.heappush(self.heap, (self._okey(s), s.idx, s.key))

    def victim(self):
        h = self.heap
        while h:
            okey, idx, key = h[0]
            s = self.slabs[idx]
            if s.state == RESIDENT and s.rank == EXP and s.key == key and self._okey(s) == okey:
                return idx
            heapq.heappop(h)
        return None

    def status(self, key):
        """('miss'|'hit'|'inflight', ready_time)."""
        i = self.where.get(key)
        if i is None:
            return "miss", None
        s = self.slabs[i]
        return ("hit" if s.state == RESIDENT else "inflight"), s.ready

    def request(self, key, pri, rank):
        """-> ('resident'|'enqueued'|'rejected', slab, evicted_key)."""
        i = self.where.get(key)
        if i is not None:
            s = self.slabs[i]
            if rank > s.rank:
                s.rank = rank
            s.pri = pri
            s.last_step = self.step
            s.done = False
            return "resident", i, None
        evicted = None
        if self.free:
            i = self.free.pop()
        else:
            i = self.victim()
            if i is None:
                return "rejected", None, None
            v = self.slabs[i]
            evicted = v.key
            self.evictions += 1
            del self.where[v.key]
            v.key, v.state, v.ready, v.done = None, FREE, None, False
        s = self.slabs[i]
        s.key, s.state, s.rank, s.pri = key, LOADING, rank, pri
        s.ready, s.last_step, s.done = None, self.step, False
        s.seq = self.counter
        self.counter += 1
        self.where[key] = i
        return "enqueued", i, evicted

    def landed(self, key, t):
        s = self.slabs[self.where[key]]
        s.state = RESIDENT
        s.ready = t

    def executed(self, key):
        s = self.slabs[self.where[key]]
        if s.state != RESIDENT:
            raise OracleSimError("mark_executed requires a resident key")
        s.rank = EXP
        s.done = True
        self._push(s)

    def reclassify(self, window, grace, fresh):
        self.step += 1
        for s in self.slabs:
            if s.state != RESIDENT:
                continue
            if s.key in fresh:
                s.pri = fresh[s.key]
            if s.key in window:
                s.rank = REQ
                s.last_step = self.step
                s.done = False
            elif not s.done and s.last_step >= 0 and self.step - s.last_step <= grace:
                s.rank = SPEC
            else:
                s.rank = EXP
                self._push(s)


def exposed(transfers, computes):
    """Transfer time not covered by compute-busy intervals (pipeline.py:351-374)."""
    out = 0.0
    ci = 0
    nc = len(computes)
    for ts, te in transfers:
        if te <= ts:
            continue
        while ci < nc and computes[ci][1] <= ts:
            ci += 1
        t = ts
        j = ci
        while j < nc and computes[j][0] < te and t < te:
            cs, ce = computes[j]
            if cs > t:
                out += min(cs, te) - t
            t = max(t, min(ce, te))
            j += 1
        if t < te:
            out += te - t
    return out


class Replay:
    """One request through the layer stack on the logical clock.

    cfg keys: transfer_ms, gpu_ms, num_slabs, fifo, grace, budget, window,
    decay_table (gamma**(d-1), d=1..W), l_pinned, shared, prefetching,
    reactive, compress_ms (0 if no compression), bootstrap_ms (0 unless
    prefetching), decode_steps, event_log.
    """

    def __init__(self, L, E, cfg, scores):
        self.L, self.E, self.c, self.scores = L, E, cfg, scores
        self.cache = SlabCache(cfg["num_slabs"], cfg["fifo"])
        self.busy_key = None
        self.busy_until = 0.0
        self.demand_fifo = []
        self.pending = {}  # key -> (pri, seq)
        self.pseq = 0
        self.xfer = []
        self.comp = []
        self.t_comp = 0.0
        self.t_xfer = 0.0
        self.n = dict(hits=0, misses=0, stalls=0, rejected=0, on_demand=0, inflight_waits=0)
        self.layers = []
        self.events = []

    # -- channel -------------------------------------------------------------
    def _log(self, *ev):
        if self.c["event_log"]:
            self.events.append(ev)

    def _start(self, key, t):
        tm = self.c["transfer_ms"]
        self.busy_key = key
        self.busy_until = t + tm
        i = self.cache.where[key]
        self.cache.slabs[i].ready = self.busy_until
        self.xfer.append((t, self.busy_until))
        self.t_xfer += tm
        self._log(t, "issue", key[0], key[1])

    def _issue(self, t):
        while self.busy_key is None:
            if self.demand_fifo:
                self._start(self.demand_fifo.pop(0), t)
                return
            if not self.pending:
                return
            key = min(self.pending, key=lambda q: (-self.pending[q][0], q[0], q[1], self.pending[q][1]))
            pri, _ = self.pending.pop(key)
            if self.cache.status(key)[0] != "miss":
                continue
            st, _, ev = self.cache.request(key, pri, REQ)
            if st == "rejected":
                self.n["rejected"] += 1
                continue
            if ev is not None:
                self._log(t, "evict", ev[0], ev[1])
            self._start(key, t)

    def _run_until(self, t):
        while self.busy_key is not None and self.busy_until <= t:
            key, r = self.busy_key, self.busy_until
            self.busy_key = None
            self.cache.landed(key, r)
            self._log(r, "complete", key[0], key[1])
            self._issue(r)

    def _wait(self, key, t):
        self._run_until(t)
        while True:
            i = self.cache.where.get(key)
            if i is not None and self.cache.slabs[i].state == RESIDENT:
                r = self.cache.slabs[i].ready
                return r if r is not None else 0.0
            if self.busy_key is None:
                raise OracleSimError(f"deadlock waiting for expert {key}")
            self._run_until(self.busy_until)

    # -- emission --------------------------------------------------------------
    def _emit(self, ctx, t, ids):
        c = self.c
        self._run_until(t)
        y = self.scores(ctx, ids)
        order = sorted(range(self.E), key=lambda e: (-float(y[e]), e))[: min(c["budget"], self.E)]
        cands = [e for e in order if float(y[e]) > 0.0]
        pri = {}
        for d in range(1, c["window"] + 1):
            l2 = ctx + d
            if l2 > self.L - 1:
                break
            if l2 < c["l_pinned"]:
                continue
            w = c["decay_table"][d - 1]
            for e in cands:
                pri[(l2, e)] = float(y[e]) * w
        fresh = {s.key: float(y[s.key[1]]) for s in self.cache.slabs if s.state == RESIDENT}
        self.cache.reclassify(pri, c["grace"], fresh)
        for key in sorted(pri, key=lambda q: (-pri[q], q[0], q[1])):
            if self.cache.status(key)[0] != "miss":
                self.cache.request(key, pri[key], REQ)
                continue
            prev = self.pending.get(key)
            if prev is None:
                self.pending[key] = (pri[key], self.pseq)
                self.pseq += 1
            else:
                self.pending[key] = (pri[key], prev[1])
        for key in [q for q in self.pending if q not in pri]:
            del self.pending[key]
        if self.busy_key is None:
            self._issue(t)

    # -- layers ----------------------------------------------------------------
    def _compute(self, start, n):
        dur = n * self.c["gpu_ms"]
        if dur > 0:
            self.comp.append((start, start + dur))
        self.t_comp += dur
        return start + dur

    def _pinned(self, layer, demand, cur, phase, step):
        end = self._compute(cur, len(demand) + self.c["shared"])
        self.layers.append((phase, step, layer, cur, end, 0.0, 0, 0))
        return end

    def _cached(self, layer, demand, cur, phase, step):
        c = self.c
        t0 = cur
        self._run_until(t0)
        hits = xfers = 0
        stall = 0.0
        run = []
        tm = c["transfer_ms"]
        horizon = self.busy_until if self.busy_key is not None else t0
        q = 0.0
        for _ in self.demand_fifo:
            q += tm
        horizon += q
        for e in sorted(demand):
            key = (layer, e)
            st, ready = self.cache.status(key)
            if st == "hit":
                self.n["hits"] += 1
                hits += 1
                self.cache.request(key, math.inf, REQ)
                run.append(key)
                continue
            self.n["misses"] += 1
            xfers += 1
            if st == "inflight" and ready is not None:
                self.n["inflight_waits"] += 1
                self.cache.request(key, math.inf, REQ)
                run.append(key)
                continue
            self.pending.pop(key, None)
            res, _, ev = self.cache.request(key, math.inf, REQ)
            if res == "rejected":
                self.n["rejected"] += 1
                raise OracleSimError(f"cache too small for layer {layer} demand (no evictable slab)")
            if ev is not None:
                self._log(t0, "evict", ev[0], ev[1])
            self.n["on_demand"] += 1
            self.demand_fifo.append(key)
            if self.busy_key is None:
                self._issue(t0)
            horizon = max(horizon, t0) + tm
            run.append(key)
        for key in run:
            r = self._wait(key, cur)
            start = max(cur, r)
            if start > cur:
                stall += start - cur
                self.n["stalls"] += 1
            cur = self._compute(start, 1)
        if c["shared"]:
            cur = self._compute(cur, c["shared"])
        for key in run:
            self.cache.executed(key)
        self.layers.append((phase, step, layer, t0, cur, stall, xfers, hits))
        return cur

    def _reactive(self, layer, demand, cur, phase, step):
        tm = self.c["transfer_ms"]
        t0 = cur
        hits = xfers = 0
        stall = 0.0
        run = []
        for e in sorted(demand):
            key = (layer, e)
            if self.cache.status(key)[0] == "hit":
                self.n["hits"] += 1
                hits += 1
                self.cache.request(key, math.inf, REQ)
            else:
                self.n["misses"] += 1
                self.n["on_demand"] += 1
                xfers += 1
                res, _, _ = self.cache.request(key, math.inf, REQ)
                if res == "rejected":
                    raise OracleSimError(f"cache too small for layer {layer} demand (no evictable slab)")
                self.xfer.append((cur, cur + tm))
                self.t_xfer += tm
                self.cache.slabs[self.cache.where[key]].ready = cur + tm
                self.cache.landed(key, cur + tm)
                stall += tm
                self.n["stalls"] += 1
                cur += tm
            cur = self._compute(cur, 1)
            run.append(key)
        if self.c["shared"]:
            cur = self._compute(cur, self.c["shared"])
        for key in run:
            self.cache.executed(key)
        self.layers.append((phase, step, layer, t0, cur, stall, xfers, hits))
        return cur

    def _layer(self, layer, demand, cur, phase, step):
        if self.c["reactive"]:
            return self._reactive(layer, demand, cur, phase, step)
        return self._cached(layer, demand, cur, phase, step)

    # -- run -------------------------------------------------------------------
    def run(self, prefill_demand, pinned_demand, retained, decode_tokens, decode_demand):
        """prefill_demand[l] / pinned_demand[l]: expert sets; decode_demand[s][l]."""
        c = self.c
        pf = c["prefetching"]
        boot = c["compress_ms"] + (c["bootstrap_ms"] if pf else 0.0)
        if boot > 0:
            self.comp.append((0.0, boot))
        cur = boot
        lp = c["l_pinned"]
        if pf and lp > 0:
            self._emit(lp - 1, boot, retained)
        for layer in range(self.L):
            if layer < lp:
                cur = self._pinned(layer, pinned_demand[layer], cur, "prefill", -1)
            else:
                cur = self._layer(layer, prefill_demand[layer], cur, "prefill", -1)
                if pf and layer < self.L - 1:
                    self._emit(layer, cur, retained)
        prefill = cur
        dec = []
        for s, tok in enumerate(decode_tokens):
            s0 = cur
            for layer in range(self.L):
                dem = decode_demand[s][layer]
                if layer < lp:
                    cur = self._pinned(layer, dem, cur, "decode", s)
                    if pf and layer == lp - 1:
                        self._emit(layer, cur, [tok])
                else:
                    cur = self._layer(layer, dem, cur, "decode", s)
                    if pf and layer < self.L - 1:
                        self._emit(layer, cur, [tok])
            dec.append(cur - s0)
        n = self.n
        return dict(
            makespan=cur,
            total_compute=self.t_comp,
            total_transfer=self.t_xfer,
            exposed_transfer=exposed(self.xfer, self.comp),
            hits=n["hits"],
            misses=n["misses"],
            stalls=n["stalls"],
            rejected_loads=n["rejected"],
            cpu_dispatches=0,
            on_demand_transfers=n["on_demand"],
            inflight_waits=n["inflight_waits"],
            evictions=self.cache.evictions,
            prefill_ms=prefill,
            decode_ms_per_step=dec,
            per_layer=[list(x) for x in self.layers],
            events=[list(e) for e in self.events],
        )

"""Expert slab cache: the reference `ExpertCache` interface over the native
policy (drop-in for pkg/src/moesim/cache.py:78-278).

The policy state machine lives in C++ (csrc/engine.cpp) and is shared with
the layer-stack engine; this class exposes the same methods, NamedTuple
results and `slabs` entries (`SlabEntry` snapshots with .key/.state/.cls/
.priority/.ready_time) that the reference engine reads.  The device side of
the cache -- the HBM slab arena and the per-layer slot table -- lives in
moe.py (`ExpertStore`).

Drop-in inside the reference engine.  `moesim.pipeline._Engine` compares the
cache's results with `is` against the enum classes IT imported
(pkg/src/moesim/pipeline.py:23-29, 462-465, 488-494, 520-524, 576-607), so a
cache constructed there must hand back those very members.  `ExpertCache`
therefore binds its four enum classes per instance: explicitly
(`ExpertCache(n, policy, enums=moesim.cache)`), or -- by default -- from the
module that constructs it, when that module's globals hold value-compatible
`ResidencyClass` / `SlabState` / `LookupStatus` / `RequestStatus` classes
(that is what `moesim.pipeline.ExpertCache = ExpertCache` needs).  Inputs are
mapped by `.value`, so either family is accepted everywhere.
"""
from __future__ import annotations

import ctypes as C
import math
import sys
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

import numpy as np

from . import _lib
from ._lib import check
from .errors import ContractError
from .trace import ExpertRef


class ResidencyClass(Enum):
    REQUIRED = "required"
    SPECULATIVE = "speculative"
    EXPIRED = "expired"


_CLS_CODE = {ResidencyClass.EXPIRED: 0, ResidencyClass.SPECULATIVE: 1, ResidencyClass.REQUIRED: 2}
_CODE_CLS = {v: k for k, v in _CLS_CODE.items()}


class SlabState(Enum):
    FREE = "free"
    LOADING = "loading"
    RESIDENT = "resident"


_STATE = {0: SlabState.FREE, 1: SlabState.LOADING, 2: SlabState.RESIDENT}


class LookupStatus(Enum):
    HIT = "hit"
    IN_FLIGHT = "in_flight"
    MISS = "miss"


class LookupResult(NamedTuple):
    status: LookupStatus
    ready_time: float | None


class RequestStatus(Enum):
    ALREADY_RESIDENT = "already_resident"
    ENQUEUED = "enqueued"
    REJECTED = "rejected"


class RequestResult(NamedTuple):
    status: RequestStatus
    slab: int | None
    evicted: ExpertRef | None


@dataclass
class SlabEntry:
    slab: int
    key: ExpertRef | None = None
    state: SlabState = SlabState.FREE
    cls: ResidencyClass = ResidencyClass.EXPIRED
    priority: float = 0.0
    ready_time: float | None = None
    last_window_step: int = -1
    executed: bool = False
    seq: int = -1


def _opt(x: float):
    return None if math.isnan(x) else x


_OWN_ENUMS = {"ResidencyClass": ResidencyClass, "SlabState": SlabState, "LookupStatus": LookupStatus,
              "RequestStatus": RequestStatus}
_CLS_BY_VALUE = {"expired": 0, "speculative": 1, "required": 2}


def _bind_enums(source) -> dict:
    """Enum classes to return: value-compatible classes found in `source`
    (a module or a globals mapping), else this package's own."""
    ns = vars(source) if hasattr(source, "__dict__") and not isinstance(source, dict) else (source or {})
    out = {}
    for name, own in _OWN_ENUMS.items():
        cand = ns.get(name)
        ok = (isinstance(cand, type) and issubclass(cand, Enum)
              and sorted(m.value for m in cand) == sorted(m.value for m in own))
        out[name] = cand if ok else own
    return out


def _constructor_globals() -> dict:
    f = sys._getframe(2)  # caller of ExpertCache.__init__
    while f is not None and f.f_globals.get("__name__") == __name__:
        f = f.f_back
    return f.f_globals if f is not None else {}


class ExpertCache:
    """Single-owner slab cache; same transitions and tie-breaks as the reference."""

    def __init__(self, num_slabs: int, victim_policy: str = "priority", enums=None):
        if num_slabs < 1:
            raise ContractError("num_slabs must be >= 1")
        if victim_policy not in ("priority", "fifo"):
            raise ContractError("victim_policy must be 'priority' or 'fifo'")
        self.num_slabs = num_slabs
        self.victim_policy = victim_policy
        self._L = _lib.load()
        h = C.c_void_p()
        check(self._L.vmm_cache_create(num_slabs, int(victim_policy == "fifo"), C.byref(h)))
        self._h = h
        ns = _bind_enums(enums if enums is not None else _constructor_globals())
        self._Res, self._State = ns["ResidencyClass"], ns["SlabState"]
        self._Lookup, self._Request = ns["LookupStatus"], ns["RequestStatus"]
        self._code_cls = {_CLS_BY_VALUE[m.value]: m for m in self._Res}
        self._state_of = {0: self._State("free"), 1: self._State("loading"), 2: self._State("resident")}
        self._ints = np.zeros((num_slabs, 7), dtype=np.int32)
        self._dbls = np.zeros((num_slabs, 2), dtype=np.float64)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.vmm_cache_destroy(h)
            self._h = None

    # -- queries --------------------------------------------------------------
    def lookup(self, key) -> LookupResult:
        r = C.c_double()
        st = self._L.vmm_cache_lookup(self._h, int(key[0]), int(key[1]), C.byref(r))
        if st == 0:
            return LookupResult(self._Lookup("miss"), None)
        return LookupResult(self._Lookup("hit" if st == 1 else "in_flight"), _opt(r.value))

    def _slab(self, i: int) -> SlabEntry:
        l, e, s, c, lw, ex, sq = (C.c_int() for _ in range(7))
        p, r = C.c_double(), C.c_double()
        check(self._L.vmm_cache_slab(self._h, i, C.byref(l), C.byref(e), C.byref(s), C.byref(c), C.byref(p),
                                     C.byref(r), C.byref(lw), C.byref(ex), C.byref(sq)))
        key = ExpertRef(l.value, e.value) if l.value >= 0 else None
        return SlabEntry(i, key, self._state_of[s.value], self._code_cls[c.value], p.value, _opt(r.value),
                         lw.value, bool(ex.value), sq.value)

    @property
    def slabs(self) -> list[SlabEntry]:
        """Snapshot of every slab (one native call; the reference engine iterates
        this on every emission, pipeline.py:520-524)."""
        n = self._L.vmm_cache_slabs(self._h, self._ints.ctypes.data, self._dbls.ctypes.data, self.num_slabs)
        check(0 if n >= 0 else -n)
        out = []
        for i, (row, (p, r)) in enumerate(zip(self._ints.tolist(), self._dbls.tolist())):
            key = ExpertRef(row[0], row[1]) if row[0] >= 0 else None
            out.append(SlabEntry(i, key, self._state_of[row[2]], self._code_cls[row[3]], p,
                                 None if r != r else r, row[4], bool(row[5]), row[6]))
        return out

    def entry(self, key) -> SlabEntry | None:
        i = self._L.vmm_cache_find(self._h, int(key[0]), int(key[1]))
        return None if i < 0 else self._slab(i)

    @property
    def evictions(self) -> int:
        ev, occ, step = C.c_longlong(), C.c_int(), C.c_int()
        self._L.vmm_cache_info(self._h, C.byref(ev), C.byref(occ), C.byref(step))
        return ev.value

    @property
    def step(self) -> int:
        ev, occ, step = C.c_longlong(), C.c_int(), C.c_int()
        self._L.vmm_cache_info(self._h, C.byref(ev), C.byref(occ), C.byref(step))
        return step.value

    def occupancy(self) -> int:
        ev, occ, step = C.c_longlong(), C.c_int(), C.c_int()
        self._L.vmm_cache_info(self._h, C.byref(ev), C.byref(occ), C.byref(step))
        return occ.value

    def resident_keys(self) -> list[ExpertRef]:
        resident = self._State("resident")
        return sorted(s.key for s in self.slabs if s.state is resident)

    def select_victim(self) -> int | None:
        v = self._L.vmm_cache_select_victim(self._h)
        return None if v < 0 else v

    # -- mutation -------------------------------------------------------------
    def request_load(self, key, priority: float, cls: ResidencyClass) -> RequestResult:
        code = _CLS_BY_VALUE[cls.value]  # either enum family (mapped by value)
        if code == 0:
            raise ContractError("cannot request a load with class Expired")
        st, slab, el, ee = (C.c_int() for _ in range(4))
        check(self._L.vmm_cache_request(self._h, int(key[0]), int(key[1]), float(priority), code,
                                        C.byref(st), C.byref(slab), C.byref(el), C.byref(ee)))
        status = self._Request(("already_resident", "enqueued", "rejected")[st.value])
        ev = ExpertRef(el.value, ee.value) if el.value >= 0 else None
        return RequestResult(status, slab.value if slab.value >= 0 else None, ev)

    def set_ready(self, key, ready_time: float) -> None:
        check(self._L.vmm_cache_set_ready(self._h, int(key[0]), int(key[1]), float(ready_time)))

    def complete_load(self, key, time: float) -> None:
        check(self._L.vmm_cache_complete(self._h, int(key[0]), int(key[1]), float(time)))

    def cancel_load(self, key) -> None:
        check(self._L.vmm_cache_cancel(self._h, int(key[0]), int(key[1])))

    def mark_executed(self, key) -> None:
        check(self._L.vmm_cache_executed(self._h, int(key[0]), int(key[1])))

    def reclassify(self, window_keys, speculative_grace: int, priorities=None) -> None:
        win = np.asarray([[int(k[0]), int(k[1])] for k in window_keys], dtype=np.int32).reshape(-1, 2)
        if priorities:
            pk = np.asarray([[int(k[0]), int(k[1])] for k in priorities], dtype=np.int32).reshape(-1, 2)
            pv = np.asarray([float(v) for v in priorities.values()], dtype=np.float64)
        else:
            pk = np.zeros((0, 2), dtype=np.int32)
            pv = np.zeros(0, dtype=np.float64)
        check(self._L.vmm_cache_reclassify(self._h, win.ctypes.data, len(win), int(speculative_grace),
                                           pk.ctypes.data, pv.ctypes.data, len(pv)))

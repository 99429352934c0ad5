"""Expert slab cache: the reference `ExpertCache` interface over the native
policy (drop-in for pkg/src/moesim/cache.py:78-278).

The policy state machine lives in C++ (csrc/engine.cpp) and is shared with
the layer-stack engine; this class exposes the same methods, NamedTuple
results and `slabs` entries (`SlabEntry` snapshots with .key/.state/.cls/
.priority/.ready_time) that the reference engine reads.  The device side of
the cache -- the HBM slab arena and the per-layer slot table -- lives in
moe.py (`ExpertStore`).
"""
from __future__ import annotations

import ctypes as C
import math
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


class ExpertCache:
    """Single-owner slab cache; same transitions and tie-breaks as the reference."""

    def __init__(self, num_slabs: int, victim_policy: str = "priority"):
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
            return LookupResult(LookupStatus.MISS, None)
        return LookupResult(LookupStatus.HIT if st == 1 else LookupStatus.IN_FLIGHT, _opt(r.value))

    def _slab(self, i: int) -> SlabEntry:
        l, e, s, c, lw, ex, sq = (C.c_int() for _ in range(7))
        p, r = C.c_double(), C.c_double()
        check(self._L.vmm_cache_slab(self._h, i, C.byref(l), C.byref(e), C.byref(s), C.byref(c), C.byref(p),
                                     C.byref(r), C.byref(lw), C.byref(ex), C.byref(sq)))
        key = ExpertRef(l.value, e.value) if l.value >= 0 else None
        return SlabEntry(i, key, _STATE[s.value], _CODE_CLS[c.value], p.value, _opt(r.value), lw.value,
                         bool(ex.value), sq.value)

    @property
    def slabs(self) -> list[SlabEntry]:
        return [self._slab(i) for i in range(self.num_slabs)]

    def entry(self, key) -> SlabEntry | None:
        for s in self.slabs:
            if s.key == tuple(key):
                return s
        return None

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
        return sorted(s.key for s in self.slabs if s.state is SlabState.RESIDENT)

    def select_victim(self) -> int | None:
        v = self._L.vmm_cache_select_victim(self._h)
        return None if v < 0 else v

    # -- mutation -------------------------------------------------------------
    def request_load(self, key, priority: float, cls: ResidencyClass) -> RequestResult:
        if cls is ResidencyClass.EXPIRED:
            raise ContractError("cannot request a load with class Expired")
        st, slab, el, ee = (C.c_int() for _ in range(4))
        check(self._L.vmm_cache_request(self._h, int(key[0]), int(key[1]), float(priority), _CLS_CODE[cls],
                                        C.byref(st), C.byref(slab), C.byref(el), C.byref(ee)))
        status = (RequestStatus.ALREADY_RESIDENT, RequestStatus.ENQUEUED, RequestStatus.REJECTED)[st.value]
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

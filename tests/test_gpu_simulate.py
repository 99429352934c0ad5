"""simulate()/simulate_reactive() through device demand/predictor kernels and the
native engine reproduce the reference's reports and event logs exactly."""
import math

import pytest

from conftest import load_golden
from paper_2605_05899_b200 import (
    CompressionConfig, PredictorSpec, SimConfig, SimulationError, build_plan, simulate, simulate_reactive,
)
from paper_2605_05899_b200.trace import TraceGenConfig, generate_trace, trace_digest

pytestmark = pytest.mark.gpu

_F = ("makespan", "total_compute", "total_transfer", "exposed_transfer", "hits", "misses", "stalls", "rejected_loads",
      "on_demand_transfers", "inflight_waits", "evictions", "prefill_ms", "decode_ms_per_step")


def sim_cfg(d):
    d = dict(d)
    p = PredictorSpec(**d.pop("predictor"))
    for k, v in list(d.items()):
        if v == "inf":
            d[k] = math.inf
    d.pop("memory", None)
    return SimConfig(predictor=p, **d)


def regen(d, digest):
    d = dict(d)
    d["saliency_shape"] = tuple(d["saliency_shape"])
    tr = generate_trace(TraceGenConfig(**d))
    assert trace_digest(tr) == digest
    return tr


@pytest.mark.parametrize("part", [0, 1])
def test_engine_cases_match_reference(part):
    for i, c in enumerate(load_golden("engine.json")):
        if i % 2 != part:
            continue
        tr = regen(c["gen"], c["digest"])
        cfg = sim_cfg(c["sim"])
        cc = c["compression"]
        ccfg = None if cc is None else CompressionConfig(cc["alpha"], cc["beta"], cc["lam"], tuple(cc["prefix"]))
        plan = build_plan(tr, cfg, ccfg)
        run = simulate_reactive if c["reactive"] else simulate
        if c["error"] is not None:
            with pytest.raises(SimulationError):
                run(tr, plan, cfg)
            continue
        r = run(tr, plan, cfg)
        rep = r.to_dict()
        exp = c["report"]
        for k in _F:
            assert rep[k] == exp[k], (i, c.get("name"), k)
        assert rep["per_layer"] == exp["per_layer"], (i, c.get("name"))
        got_ev = [list(e) for e in r.events]
        assert got_ev == exp["events"], (i, c.get("name"))

"""Native cache policy (ExpertCache drop-in) vs golden ops recorded from the reference."""
import math

import pytest

from conftest import load_golden
from paper_2605_05899_b200.cache import ExpertCache, ResidencyClass
from paper_2605_05899_b200.errors import ContractError
from paper_2605_05899_b200.trace import ExpertRef


def test_golden_op_sequences_exact():
    cls = {"required": ResidencyClass.REQUIRED, "speculative": ResidencyClass.SPECULATIVE}
    for case in load_golden("cache_ops.json"):
        c = ExpertCache(case["num_slabs"], case["policy"])
        for op in case["ops"]:
            kind = op[0]
            if kind == "request":
                pri = math.inf if op[2] == "inf" else op[2]
                r = c.request_load(ExpertRef(*op[1]), pri, cls[op[3]])
                assert (r.status.value, r.slab) == (op[4], op[5])
                assert (list(r.evicted) if r.evicted else None) == op[6]
            elif kind == "complete":
                c.complete_load(ExpertRef(*op[1]), 1.0)
            elif kind == "executed":
                c.mark_executed(ExpertRef(*op[1]))
            elif kind == "cancel":
                c.cancel_load(ExpertRef(*op[1]))
            elif kind == "reclassify":
                c.reclassify([ExpertRef(*k) for k in op[1]], op[2], {ExpertRef(*k): v for k, v in op[3]})
            snap = op[-1]
            mine = sorted([[s.slab, list(s.key), s.state.value, s.cls.value,
                            "inf" if s.priority == math.inf else s.priority] for s in c.slabs if s.key])
            assert mine == snap
        assert c.evictions == case["evictions"]
        assert c.select_victim() == case["victim"]


def test_tie_breaks_and_contracts():
    c = ExpertCache(2)
    for key in (ExpertRef(1, 3), ExpertRef(0, 5)):
        c.request_load(key, 0.5, ResidencyClass.REQUIRED)
        c.complete_load(key, 0.0)
        c.mark_executed(key)
    # equal priority: lower layer is the victim
    assert c.slabs[c.select_victim()].key == ExpertRef(0, 5)
    r = c.request_load(ExpertRef(2, 0), 1.0, ResidencyClass.REQUIRED)
    assert r.evicted == ExpertRef(0, 5)
    with pytest.raises(ContractError):
        c.request_load(ExpertRef(3, 0), 1.0, ResidencyClass.EXPIRED)
    with pytest.raises(ContractError):
        c.mark_executed(ExpertRef(9, 9))
    with pytest.raises(ContractError):
        ExpertCache(0)

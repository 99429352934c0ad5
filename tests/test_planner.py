"""Reference acceptance A10 (pkg/tests/test_acceptance.py:358-376): the prefix
planner's Eq. 9 arithmetic (host Python, no GPU)."""
import pytest

from paper_2605_05899_b200.errors import PlanningError
from paper_2605_05899_b200.pipeline import plan_prefix


def test_a10_prefix_planner_arithmetic():
    s_layer = 128 * 17.3
    assert s_layer == 2214.4
    for l_semantic in range(0, 10):
        plan = plan_prefix(35_900.0, s_layer, 14_300.0, l_semantic)
        assert plan.hi == 9 and plan.chosen == l_semantic and plan.lo <= plan.chosen <= 9
    assert plan_prefix(35_900.0, s_layer, 14_300.0, 8, override=9).chosen == 9
    with pytest.raises(PlanningError):
        plan_prefix(35_900.0, s_layer, 14_300.0, 10)
    with pytest.raises(PlanningError):
        plan_prefix(10_000.0, s_layer, 14_300.0, 0)


def test_a5_random_baseline_calibration():
    """Reference acceptance A5 (pkg/tests/test_acceptance.py:181-206): the random predictor's
    mean next-layer hot recall over 1200 trials sits within 3 sigma of B/E (E=128)."""
    import math

    import numpy as np

    from paper_2605_05899_b200.predictor import RandomPredictor
    from paper_2605_05899_b200.trace import TraceGenConfig, generate_trace

    tr = generate_trace(TraceGenConfig(n_visual=24, n_text=8, layers=6, experts=128, k=4, clusters=4,
                                       cluster_support=10, rho=0.8, visual_noise=0.2, seed=0))
    ids = tr.prefill_ids()
    layer = 2
    act = tr.active_union(layer + 1, ids)
    actual = len(act)
    trials = 1200
    for budget in (10, 20, 30):
        rand = RandomPredictor(tr.experts, seed=1000 + budget)
        recalls = [len(act & set(rand.predict(layer, budget))) / actual for _ in range(trials)]
        mean = float(np.mean(recalls))
        expect = budget / tr.experts
        var_one = (budget * (actual / 128) * (1 - actual / 128) * (128 - budget) / 127) / actual ** 2
        assert abs(mean - expect) <= 3 * math.sqrt(var_one / trials), (budget, mean, expect)

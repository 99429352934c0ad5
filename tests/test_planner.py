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

"""Workload accounting used by bench.py (SURVEY 8(d) algorithmic units) and the
K1 host plan sizes, against the counts measured with the reference in the survey."""

import pytest

import bench
from paper_1907_01005_b200 import problem as P
from paper_1907_01005_b200.comm import serial_context
from paper_1907_01005_b200.matfree import _CellPlan


@pytest.mark.parametrize("name,pairs,nnzx,nnzhx", [
    ("smoke", 992, 5_320, 10_584),
    ("q2", 165_752, 996_992, 1_495_808),
    ("q4", 165_752, 7_428_672, 11_275_200),
])
def test_algorithmic_counts_match_survey(name, pairs, nnzx, nnzhx):
    prob = P.build_problem(name)
    st = P.make_rank_setup(serial_context("cpu"), prob, device="cpu")
    cnt = bench.workload_counts(st)
    assert (cnt["pairs"], cnt["nnzX"], cnt["nnzHX"]) == (pairs, nnzx, nnzhx)
    n = prob.cfg.degree + 1
    assert cnt["flops_hx_reference_formulation"] == pairs * (36 * n**4 + 8 * n**3)
    plan = _CellPlan(st.op, st.x, st.hx, upload=False)
    assert plan.n_pairs == pairs
    if name != "smoke":
        assert plan.n_visits == 70_882  # reference OpCounters.col_blocks_visited

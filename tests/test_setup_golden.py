"""Index maps and sparsity patterns: bit-exact against the reference.

Golden arrays (tests/golden/*.npz) and sha256 digests of the full-size
BASELINE configs (tests/golden/digests.json) were produced by the
reference package itself (tests/golden/make_golden.py).
"""

import hashlib
import os
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1907_01005_b200.energy import projected_pattern
from paper_1907_01005_b200.localization import (
    build_support_sparsity,
    column_supports,
    grow_sparsity_for_operator,
    order_and_block_columns,
)
from paper_1907_01005_b200.mesh import build_mesh, enumerate_dofs, partition_and_order_cells
from paper_1907_01005_b200.problem import baseline_config, build_problem

GOLD = Path(__file__).resolve().parent / "golden"


def structure(part, num, lay, sup, pat, gro, proj=None):
    d = {
        "ordered_cells": part.ordered_cells,
        "rank_group_start": part.rank_group_start,
        "new_index_of_node": num.new_index_of_node,
        "row_block_sizes": num.row_blocks.sizes,
        "owned_ranges": np.asarray(num.owned_ranges, dtype=np.int64),
        "rank_block_start": num.rank_block_start,
        "old_col_of_new": lay.old_col_of_new,
        "col_block_sizes": lay.column_blocks.sizes,
        "col_rank_block_start": lay.rank_block_start,
        "support_ptr": np.concatenate([[0], np.cumsum([s.size for s in sup])]),
        "support_rows": np.concatenate(sup),
        "pattern_row_start": pat.row_start,
        "pattern_col_index": pat.col_index,
        "grown_row_start": gro.row_start,
        "grown_col_index": gro.col_index,
    }
    if proj is not None:
        d["proj_row_start"] = proj.row_start
        d["proj_col_index"] = proj.col_index
    return d


def build(ext, sp, level, degree, centers, radius, vpc, bs, n_ranks):
    mesh = build_mesh(ext, sp, level)
    part = partition_and_order_cells(mesh, n_ranks)
    num = enumerate_dofs(mesh, part, degree)
    lay = order_and_block_columns(mesh, part, centers, radius, vpc, bs)
    sup = column_supports(mesh, num, lay)
    pat = build_support_sparsity(mesh, part, num, lay, sup)
    gro = grow_sparsity_for_operator(pat, mesh, num)
    return mesh, part, num, lay, sup, pat, gro


def test_smoke_structure_bit_exact(golden_smoke):
    g = golden_smoke
    prob = build_problem("smoke")
    got = structure(prob.partition, prob.numbering, prob.loc_layout, prob.supports, prob.pattern,
                    prob.grown, prob.proj_pattern)
    for k, v in got.items():
        assert np.array_equal(v, g[k]), k


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
@pytest.mark.parametrize("n_ranks", [1, 2, 4])
def test_random_structures_bit_exact(golden_random, degree, n_ranks):
    g = golden_random
    ext = tuple(int(v) for v in g[f"p{degree}_extents"])
    _, part, num, lay, sup, pat, gro = build(ext, (1.0, 1.0, 1.0), 1, degree,
                                             g[f"p{degree}_centers"],
                                             float(g[f"p{degree}_radius"]), 2, 3, n_ranks)
    got = structure(part, num, lay, sup, pat, gro)
    for k, v in got.items():
        assert np.array_equal(v, g[f"p{degree}_r{n_ranks}_{k}"]), k


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def _low_memory() -> bool:
    try:
        import psutil

        return psutil.virtual_memory().available < 32 * 2**30
    except Exception:
        return False


_WEAK8 = pytest.param("weak8", marks=pytest.mark.skipif(
    os.environ.get("BMV_SKIP_WEAK8") == "1" or _low_memory(),
    reason="135 M DoFs: needs ~20 GB of host memory (about a minute)"))


@pytest.mark.parametrize("name", ["q2", "q4", "proj", "weak1", "weak2", "weak4", _WEAK8])
def test_full_size_index_maps_match_reference_digests(name):
    want = json.loads((GOLD / "digests.json").read_text())[name]
    n_ranks = int(name[4:]) if name.startswith("weak") else 1
    prob = build_problem(baseline_config(name, n_ranks), n_ranks)
    proj = prob.proj_pattern if "proj_row_start" in want else None
    got = structure(prob.partition, prob.numbering, prob.loc_layout, prob.supports, prob.pattern,
                    prob.grown, proj)
    assert want["_sizes"]["n_dofs"] == prob.numbering.n_dofs
    for k, v in got.items():
        assert _digest(v) == want[k], k

"""The input generator reproduces the reference's problems (golden fixtures)."""

import numpy as np
import pytest

from conftest import SMALL_CASES, load_golden
from harness import inputs


@pytest.mark.parametrize("case", SMALL_CASES)
def test_problem_matches_reference(case):
    g = load_golden(case)
    prob = inputs.Problem(str(g["physics"]), int(g["dim"]), int(g["cells"]), int(g["subs"]))
    assert prob.n_sub == int(g["n_sub"])
    assert prob.n_multipliers == int(g["n_multipliers"])
    np.testing.assert_array_equal(prob.c, g["c"])
    for s in range(prob.n_sub):
        np.testing.assert_array_equal(prob.gids[s], g[f"s{s}_gids"])
        np.testing.assert_array_equal(prob.bcol[s], g[f"s{s}_bcol"])
        np.testing.assert_array_equal(prob.bval[s], g[f"s{s}_bval"])
        k, load, q = prob.subdomain_system(s)
        np.testing.assert_array_equal(k.indptr, g[f"s{s}_k_indptr"])
        np.testing.assert_array_equal(k.indices, g[f"s{s}_k_indices"])
        np.testing.assert_allclose(k.data, g[f"s{s}_k_data"], rtol=1e-13, atol=1e-13 * np.abs(k.data).max())
        np.testing.assert_allclose(load, g[f"s{s}_force"], rtol=1e-14, atol=0)
        np.testing.assert_allclose(q, g[f"s{s}_kernel"], rtol=0, atol=1e-13)


def test_cluster_layout_contiguous():
    prob = inputs.Problem("heat", 2, 3, 2, n_clusters=2)
    lay = prob.layout
    assert lay.n_clusters == 2
    assert list(lay.clusters[0].subdomain_ids) == [0, 1]
    for cl in lay.clusters:
        for s, sc in zip(cl.subdomain_ids, cl.scatter):
            np.testing.assert_array_equal(cl.dual_ids[sc], prob.gids[s])
    with pytest.raises(ValueError):
        prob.build_clusters(3)


@pytest.mark.parametrize("cfg,n,mult", [("c1", 289, 467), ("c2", 729, 103807), ("c3", 9261, 68319),
                                        ("c4", 10125, 103221)])
def test_config_sizes(cfg, n, mult):
    # DOFs per subdomain and global multiplier counts
    prob = inputs.Problem(*inputs.CONFIGS[cfg])
    assert prob.n_dofs == n
    assert prob.n_multipliers == mult


def test_c3_interior_subdomain_matches_reference():
    g = load_golden("c3_sub21")
    prob = inputs.Problem(*inputs.CONFIGS["c3"])
    s = int(g["sub_index"])
    assert prob.n_multipliers == int(g["n_multipliers"])
    np.testing.assert_array_equal(prob.gids[s], g["gids"])
    np.testing.assert_array_equal(prob.bcol[s], g["bcol"])
    np.testing.assert_array_equal(prob.bval[s], g["bval"])
    k, _, _ = prob.subdomain_system(s)
    np.testing.assert_array_equal(k.indptr, g["k_indptr"])
    np.testing.assert_array_equal(k.indices, g["k_indices"])
    np.testing.assert_allclose(k.data, g["k_data"], rtol=1e-13, atol=1e-13 * np.abs(k.data).max())

"""Multi-rank composition of the apply (CPU, gloo, world_size 2).

Cluster r of the reference's contiguous layout (decomposition.py:227-243)
lives on rank r; every rank applies its own subdomains into a full-length
dual vector and the contributions are summed by an all-reduce.  On the GPU
box the all-reduce is NCCL over NVLink; here gloo exercises the same code
(paper_2502_08382_b200.distributed) with the oracle as the local apply.
"""

import os
import socket

import numpy as np
import pytest

from oracle import feti_oracle as ora
from paper_2502_08382_b200 import distributed as fd
from harness import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_parts(prob):
    facs, cons = [], []
    for s in range(prob.n_sub):
        k, _, q = prob.subdomain_system(s)
        kr = inputs.regularized_csr(k, q)
        sym = ora.symbolic_factorize(kr.shape[0], kr.indptr, kr.indices)
        vals = ora.numeric_factorize(sym, kr.data)
        facs.append(dict(up=sym.up, ui=sym.ui, values=vals, perm=sym.perm, iperm=sym.iperm, n=sym.n))
        cons.append((prob.gids[s], prob.bcol[s], prob.bval[s]))
    op = ora.OracleOperator(facs, cons)
    op.preprocess()
    return op


def _worker(rank, world, port, outdir, assign="contiguous"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = inputs.Problem("heat", 2, 3, 2, n_clusters=world)
        op = _oracle_parts(prob)
        if assign == "lpt":
            owned = fd.lpt_subdomains(fd.apply_weights(prob.constraints()), world, rank)
        else:
            owned = fd.owned_subdomains(prob.layout, rank)
        p = np.random.default_rng(0).normal(size=prob.n_multipliers)

        def local_apply(vec):
            out = np.zeros_like(vec)
            for s in owned:
                g = prob.gids[s]
                q = np.empty(g.shape[0])
                ora.lib().ora_symv_upper(g.shape[0], op.fmats[s].ctypes.data,
                                         np.ascontiguousarray(vec[g]).ctypes.data, q.ctypes.data)
                out[g] += q
            return out

        q = fd.contributions_sum(local_apply, p)
        np.save(os.path.join(outdir, f"q{rank}.npy"), q)
        np.save(os.path.join(outdir, f"owned{rank}.npy"), np.array(owned))
    finally:
        dist.destroy_process_group()


def test_two_rank_apply_equals_single_operator(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    prob = inputs.Problem("heat", 2, 3, 2, n_clusters=2)
    op = _oracle_parts(prob)
    p = np.random.default_rng(0).normal(size=prob.n_multipliers)
    ref = op.apply(p)
    q0, q1 = np.load(tmp_path / "q0.npy"), np.load(tmp_path / "q1.npy")
    assert np.array_equal(q0, q1)                       # every rank holds the sum
    assert np.linalg.norm(q0 - ref) <= 1e-14 * np.linalg.norm(ref)
    owned = [list(np.load(tmp_path / f"owned{r}.npy")) for r in range(2)]
    assert owned == [[0, 1], [2, 3]]                    # contiguous clusters
    del torch


def test_owned_subdomains_layout():
    prob = inputs.Problem("heat", 3, 2, 2, n_clusters=4)
    got = [fd.owned_subdomains(prob.layout, r) for r in range(4)]
    assert got == [[0, 1], [2, 3], [4, 5], [6, 7]]
    with pytest.raises(ValueError):
        fd.owned_subdomains(prob.layout, 4)


def test_two_rank_lpt_apply_equals_single_operator(tmp_path):
    """The LPT assignment (mixed subdomain sets per rank) composes to the same q."""
    pytest.importorskip("torch")
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), "lpt"), nprocs=2, join=True)
    prob = inputs.Problem("heat", 2, 3, 2, n_clusters=2)
    op = _oracle_parts(prob)
    p = np.random.default_rng(0).normal(size=prob.n_multipliers)
    ref = op.apply(p)
    q0, q1 = np.load(tmp_path / "q0.npy"), np.load(tmp_path / "q1.npy")
    assert np.array_equal(q0, q1)
    assert np.linalg.norm(q0 - ref) <= 1e-14 * np.linalg.norm(ref)
    owned = [set(np.load(tmp_path / f"owned{r}.npy").tolist()) for r in range(2)]
    assert owned[0] | owned[1] == set(range(prob.n_sub)) and not owned[0] & owned[1]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_lpt_balances_config3_apply_work(world):
    """Config 3: contiguous clusters leave max/mean 1.20 of packed
    F~ bytes at 4 and 8 ranks; LPT is within one subdomain's share of the mean,
    deterministic, and a partition."""
    prob = inputs.Problem(*inputs.CONFIGS["c3"], n_clusters=world)
    w = fd.apply_weights(prob.constraints())
    parts = [fd.lpt_subdomains(w, world, r) for r in range(world)]
    assert sorted(s for p in parts for s in p) == list(range(prob.n_sub))
    assert parts == [fd.lpt_subdomains(w, world, r) for r in range(world)]
    loads = [sum(w[s] for s in p) for p in parts]
    mean = sum(w) / world
    assert max(loads) - mean <= max(w)
    contiguous = [sum(w[s] for s in fd.owned_subdomains(prob.layout, r)) for r in range(world)]
    assert max(loads) <= 1.001 * max(contiguous)
    assert max(loads) / mean < 1.05

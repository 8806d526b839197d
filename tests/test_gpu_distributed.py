"""N > 1 on the device path: two ranks (gloo, sharing cuda:0) each own one
cluster, apply their subdomains and all-reduce -- must equal one rank owning
everything.  On a multi-GPU box the same code runs over NCCL (bench.py)."""

import os
import socket

import numpy as np
import pytest

from paper_2502_08382_b200 import distributed as fd
from paper_2502_08382_b200 import dualop
from harness import inputs

pytestmark = pytest.mark.gpu
CFG = dualop.DualOpConfig(strategy="explicit", path="syrk")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = inputs.Problem("heat", 3, 4, 2, n_clusters=world)
        mats, cons, lay = inputs.reference_inputs(prob)
        owned = fd.owned_subdomains(lay, rank)
        with dualop.prepare(mats, cons, lay, CFG, device=0, subdomains=owned) as op:
            op.preprocess()
            dco = fd.ClusterDualOperator(op, prob.n_multipliers, torch.device("cuda", 0))
            p = np.random.default_rng(5).normal(size=prob.n_multipliers)
            q = dco.apply(p if rank == 0 else None)
            np.save(os.path.join(outdir, f"q{rank}.npy"), q)
    finally:
        dist.destroy_process_group()


def test_two_ranks_match_single_rank(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    mp.spawn(_rank, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    prob = inputs.Problem("heat", 3, 4, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    p = np.random.default_rng(5).normal(size=prob.n_multipliers)
    with dualop.prepare(mats, cons, lay, CFG, device=0) as op:
        op.preprocess()
        ref = op.apply(p)
    q0, q1 = np.load(tmp_path / "q0.npy"), np.load(tmp_path / "q1.npy")
    assert np.array_equal(q0, q1)
    assert np.linalg.norm(q0 - ref) <= 1e-13 * np.linalg.norm(ref)
    del torch

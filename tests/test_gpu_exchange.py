"""Fused cross-rank exchange of the apply (csrc/feti_exchange.cu) with two
processes: each owns one cluster (decomposition.py:227-243) and exchanges its
contributions through CUDA IPC peer memory.  On the one-GPU test box both
ranks share the device (IPC across processes on one device); on a node each
rank has its own GPU and the stores cross NVLink.  q must equal the
single-operator apply of the whole problem to rounding, be identical on both
ranks, and repeat bit for bit."""

import os
import socket

import numpy as np
import pytest

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


def _worker(rank, world, port, outdir, assign="contiguous"):
    import torch
    import torch.distributed as dist

    from paper_2502_08382_b200 import distributed as fd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ndev = torch.cuda.device_count()
        dev = torch.device("cuda", rank % ndev)
        torch.cuda.set_device(dev)
        prob = inputs.Problem("heat", 3, 4, 2, n_clusters=world)
        mats, cons, lay = inputs.reference_inputs(prob)
        owned = (fd.lpt_subdomains(fd.apply_weights(cons), world, rank) if assign == "lpt"
                 else fd.owned_subdomains(lay, rank))
        with dualop.prepare(mats, cons, lay, CFG, device=dev.index, subdomains=owned) as op:
            op.preprocess()
            dco = fd.ClusterDualOperator(op, prob.n_multipliers, dev)
            assert dco.p2p
            p = torch.from_numpy(np.random.default_rng(0).normal(size=prob.n_multipliers)).to(dev)
            qs = []
            for _ in range(5):
                q = torch.empty_like(p)
                dco.apply_device(p, q)
                torch.cuda.synchronize(dev)
                qs.append(q.cpu().numpy())
            op.exchange_status()
            np.save(os.path.join(outdir, f"q{rank}.npy"), np.stack(qs))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,assign", [(2, "contiguous"), (4, "contiguous"), (8, "contiguous"), (4, "lpt")])
def test_fused_exchange_multi_rank(tmp_path, world, assign):
    """2, 4 and 8 ranks (one subdomain per rank at 8) time-sharing the box's
    GPU through CUDA IPC, contiguous clusters or the LPT assignment: q equals
    the single-operator apply, is identical on every rank and repeats bit for
    bit over successive epochs (slab parity reuse)."""
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _port(), str(tmp_path), assign), nprocs=world, join=True)
    prob = inputs.Problem("heat", 3, 4, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    with dualop.prepare(mats, cons, lay, CFG, device=0) as op:
        op.preprocess()
        ref = op.apply(np.random.default_rng(0).normal(size=prob.n_multipliers))
    qs = [np.load(tmp_path / f"q{r}.npy") for r in range(world)]
    for q in qs[1:]:
        assert np.array_equal(q, qs[0])
    for k in range(1, qs[0].shape[0]):
        assert np.array_equal(qs[0][k], qs[0][0])
    assert np.linalg.norm(qs[0][0] - ref) <= 1e-12 * np.linalg.norm(ref)

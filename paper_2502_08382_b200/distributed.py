"""Subdomains across GPUs: one process per GPU, one cluster per rank.

The reference lays subdomains out in contiguous clusters
(``build_clusters``, decomposition.py:227-243) and the paper maps one cluster
to one GPU, synchronising cluster dual vectors between
processes.  Here:

* assembly is embarrassingly parallel: rank r assembles the F~_i of cluster r
  on its own GPU, no communication;
* apply has one exchange step.  Default (``exchange="p2p"``): the
  exchange is fused into the apply's reduction (csrc/feti_exchange.cu): each
  rank's reduction kernel stores its per-multiplier sums straight into every
  rank's receive slab over NVLink (CUDA IPC peer memory), publishes an epoch
  flag, and a second kernel sums the slabs in rank order once every flag
  arrived -- no collective library call, deterministic, identical on every
  rank.  ``exchange="nccl"``: the rank's contribution over all multipliers
  is summed with an NCCL all-reduce (the baseline).  The p vector is
  broadcast from rank 0 when it starts on the host.

Within a rank the summation order is the reference's fixed gather order
(dualop.py:375-379); across ranks it is rank order (p2p) or NCCL's, so
results agree with the reference to rounding (<=1e-10 relative).
"""

from __future__ import annotations

import numpy as np


def owned_subdomains(layout, rank: int):
    """Subdomain ids of cluster ``rank`` (the contiguous layout of the reference)."""
    if rank >= len(layout.clusters):
        raise ValueError(f"layout has {len(layout.clusters)} clusters, no cluster for rank {rank}")
    return [int(s) for s in layout.clusters[rank].subdomain_ids]


def lpt_subdomains(weights, world: int, rank: int):
    """Longest-processing-time-first assignment of subdomains to ranks: by
    decreasing weight (ties by index), each subdomain goes to the currently
    least-loaded rank (ties by rank).  Deterministic on every rank.  Weights:
    ``apply_weights`` (packed F~ bytes, the per-iteration HBM stream) or any
    per-subdomain work estimate.  The reference's contiguous layout
    (decomposition.py:227-243) leaves max/mean 1.20 at 4 and 8 GPUs on configs
    3-4; LPT gets within one subdomain of the mean.  Returns the
    rank's subdomain ids in ascending order (the operator applies them in the
    reference's gather order, dualop.py:375-379)."""
    w = [float(x) for x in weights]
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    loads = [0.0] * world
    owner = [0] * len(w)
    for s in sorted(range(len(w)), key=lambda i: (-w[i], i)):
        r = min(range(world), key=lambda k: (loads[k], k))
        owner[s] = r
        loads[r] += w[s]
    return [s for s in range(len(w)) if owner[s] == rank]


def apply_weights(constraints):
    """Per-subdomain apply work: packed F~ bytes 8 m (m + 1) / 2."""
    return [4.0 * m * (m + 1) for m in (len(sc.multiplier_ids) for sc in constraints.per_subdomain)]


def allreduce_sum_(q, group=None):
    """In-place sum of per-rank dual-vector contributions."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(q, op=dist.ReduceOp.SUM, group=group)
    return q


class ClusterDualOperator:
    """The rank-local explicit dual operator plus the cross-rank exchange.

    ``local`` is any object with ``apply_device(p, q, stream)`` writing this
    rank's contribution over all multipliers (the B200 ``DualOperator`` built
    with ``subdomains=owned_subdomains(layout, rank)``).
    """

    def __init__(self, local, n_multipliers: int, device, group=None, exchange: str = "p2p"):
        import torch
        import torch.distributed as dist

        if exchange not in ("p2p", "nccl"):
            raise ValueError("exchange must be 'p2p' or 'nccl'")
        self.local = local
        self.n = int(n_multipliers)
        self.device = device
        self.group = group
        self.p_dev = torch.empty(self.n, dtype=torch.float64, device=device)
        self.q_dev = torch.empty(self.n, dtype=torch.float64, device=device)
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        self.p2p = exchange == "p2p" and multi and hasattr(local, "exchange_setup")
        if self.p2p:
            rank, world = dist.get_rank(group), dist.get_world_size(group)
            handle = local.exchange_setup(rank, world)
            handles = [None] * world
            dist.all_gather_object(handles, handle, group=group)
            local.exchange_connect(handles)
            dist.barrier(group=group)

    def apply_device(self, p_dev, q_dev):
        import torch

        stream = torch.cuda.current_stream(self.device).cuda_stream
        if self.p2p:
            self.local.apply_exchange_device(p_dev, q_dev, stream)
            return q_dev
        self.local.apply_device(p_dev, q_dev, stream)
        allreduce_sum_(q_dev, self.group)
        return q_dev

    def check(self):
        """Raise if the fused exchange ever timed out waiting for a peer (the
        kernels then wrote NaN into q); a no-op for the NCCL exchange."""
        if self.p2p:
            self.local.exchange_status()

    def apply(self, p=None, out=None, src: int = 0):
        """Host-facing apply: p on rank ``src``'s host, q returned on every rank."""
        import torch
        import torch.distributed as dist

        if p is not None:
            self.p_dev.copy_(torch.from_numpy(np.ascontiguousarray(p, dtype=np.float64)), non_blocking=False)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.broadcast(self.p_dev, src=src, group=self.group)
        self.apply_device(self.p_dev, self.q_dev)
        host = self.q_dev.cpu().numpy()
        self.check()
        if out is None:
            return host
        out[:] = host
        return out


def contributions_sum(local_apply, p, group=None):
    """Reference semantics of the exchange for any local apply callable (CPU
    tests with gloo): q = sum over ranks of local_apply(p)."""
    import torch

    q = torch.from_numpy(np.asarray(local_apply(p), dtype=np.float64).copy())
    allreduce_sum_(q, group)
    return q.numpy()

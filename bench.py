#!/usr/bin/env python
"""Benchmark of the explicit FETI dual operator on B200 (driver contract).

Metric (BASELINE.json): F assembly seconds + apply ms/iteration on 3D heat
with ~10k-DOF subdomains (config 3: 64 subdomains of 20^3 cells, 9261 DOFs,
68,319 multipliers) at 1-8 B200, and the amortization iteration count.

One "step" = the whole preprocess of every F~_i of the job through the
drop-in's default route for configs 3-5, the sparse-factor route
(DualOperator(factorization="sparse")): device factorization of K_s = K +
rho E E^T into block-sparse FP64 tiles, pruned forward solve + SYRK on the
interface block, and the exact rank-2r correction to the reference's F~.
``value`` = device time per step with the sparse K and kernel basis already
resident in HBM (CUDA events on the launching stream, max over ranks);
``e2e`` = the same step through the public API from host arrays (K values
and Q host->device inside the timed region) followed by one apply with host
vectors (H2D p, D2H q).  The step therefore includes the factorization,
which the CPU baseline (the reference's CPU explicit assembly) does not.

``reference_factor_path`` holds the same measurements for the reference's
own factor (dense K_reg, RCM): assembly from that factor resident in HBM,
and e2e from pinned HOST factor buffers (22 GB H2D at config 3).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                    [--config c1..c5] [--route dense|sparse]

Input factors for the reference-factor path: the reference's K_reg of every
subdomain (inputs.py restates the reference's mesh/assembly/regularization),
ordered by reverse Cuthill-McKee exactly as the reference's symbolic stage
(reversed natural order on the dense K_reg), factored once during setup with
torch.linalg.cholesky on the GPU (input generation only -- outside every
timed region; the drop-in's own host LAPACK factorization is timed
separately on one subdomain and reported as ``host_factorization``).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "F assembly s + apply ms/iter (3D heat, 1–8×B200); amortization iterations"
UNIT = "s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------


def rcm_perm_dense(n):
    """RCM of the complete graph = reversed natural order (factor.rcm_ordering)."""
    return np.arange(n - 1, -1, -1, dtype=np.int64)


def interface_last_perm(n, bcol):
    base = rcm_perm_dense(n)
    mark = np.zeros(n, bool)
    mark[bcol] = True
    return np.concatenate([base[~mark[base]], np.sort(np.flatnonzero(mark))]).astype(np.int64)


def device_factor(prob, s, perm, dev, mask_cache):
    """Packed col-major lower Cholesky factor of P K_reg P^T, built on the GPU
    (input generation only)."""
    import torch

    k, _load, q = prob.subdomain_system(s)
    n = k.shape[0]
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(k.indptr))
    A = torch.zeros((n, n), dtype=torch.float64, device=dev)
    A[torch.from_numpy(rows).to(dev), torch.from_numpy(k.indices).to(dev)] = torch.from_numpy(k.data).to(dev)
    qo, _ = np.linalg.qr(q)
    Q = torch.from_numpy(qo).to(dev)
    rho = torch.trace(A) / n
    S = Q @ Q.T
    A += rho * (0.5 * (S + S.T))
    dense_ok = bool(torch.count_nonzero(A).item() == n * n)
    P = torch.from_numpy(perm).to(dev)
    A = A.index_select(0, P).index_select(1, P)
    L = torch.linalg.cholesky(A)
    del A
    if n not in mask_cache:
        mask_cache.clear()
        mask_cache[n] = torch.ones((n, n), dtype=torch.bool, device=dev).triu_()
    packed = L.T.contiguous()[mask_cache[n]]     # rows of U = columns of L
    del L
    return packed, dense_ok


# ---------------------------------------------------------------------------
# CPU reference measurements (oracle port, bounded samples)
# ---------------------------------------------------------------------------


class CpuReference:
    """The reference's CPU paths for this path, timed on the box's host cores
    per multiplier-count class: CPU BLAS cost depends only on
    (n, m), so one subdomain per m-class, weighted by the class's subdomain
    count, times the whole job exactly up to noise.

    * explicit assembly, the reference's dense-storage config as is
      (assemble_explicit_local, dualop.py:427-501: densify P B~^T,
      factor_to_dense fancy scatter sparse.py:539-563, BLAS dtrsm
      sparse.py:517-536, dsyrk dualop.py:488-501, zero_lower) on the
      reference-layout factor of the dense K_reg -- the faster of
      {1 worker x all BLAS threads} and {`nconc` workers x 1 BLAS thread},
      decided on the largest class;
    * the reference's default config (sparse storage: utsolve_rows,
      _kernels.py:168-181, one thread per subdomain) on a 128-column sample
      of the largest class, scaled by sum(m) / 128 (its cost is linear in
      the number of right-hand sides), over `threads` workers;
    * explicit apply: symv_upper over every subdomain (dualop.py:348-388);
    * implicit apply: apply_implicit_local (dualop.py:504-521) per class,
      `nconc` concurrent, weighted by the class counts.
    The dense K_reg factorizations (LAPACK) are setup, outside every timing.
    """

    def __init__(self, prob, threads=None, log_fn=None):
        from oracle import feti_oracle as ora
        from paper_2502_08382_b200 import factor as fct

        self.ora = ora
        self.prob = prob
        self.threads = threads or os.cpu_count()
        n = prob.n_dofs
        ms = prob.m_per_subdomain()
        self.n = n
        self.perm = rcm_perm_dense(n)
        self.iperm = fct.inverse_permutation(self.perm)
        self.up, self.ui = ora.dense_pattern(n)
        self.classes = []      # (m, representative subdomain, count)
        for m in sorted(set(int(x) for x in ms)):
            members = np.flatnonzero(ms == m)
            self.classes.append((m, int(members[0]), int(members.size)))
        t0 = time.perf_counter()
        self.values = {}
        for m, s, _ in self.classes:
            kreg = prob.kreg_dense(s)
            self.values[s] = ora.dense_factor_values(kreg, self.perm)
            del kreg
        self.setup_s = time.perf_counter() - t0
        self.host_factorization_s = self.setup_s / len(self.classes)
        if log_fn:
            log_fn(f"[cpu] {len(self.classes)} m-classes, dense K_reg + LAPACK factor per class in {self.setup_s:.1f} s")
        self.fmats = {}
        self.variant = None

    def _assemble(self, s):
        ora, prob = self.ora, self.prob
        return ora.assemble_explicit_local(self.up, self.ui, self.values[s], self.n, self.iperm, prob.bcol[s],
                                           prob.bval[s], storage="dense")

    def choose_threading(self):
        """Faster of 1 worker x all BLAS threads / nconc workers x 1 BLAS thread,
        per subdomain-equivalent, on the largest class."""
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits

        m, s, _ = self.classes[-1]
        self._assemble(s)
        t0 = time.perf_counter()
        self._assemble(s)
        t_blas = time.perf_counter() - t0
        nconc = max(1, min(self.threads, 8, self.prob.n_sub))
        with threadpool_limits(limits=1, user_api="blas"):
            t0 = time.perf_counter()
            with ThreadPoolExecutor(nconc) as ex:
                list(ex.map(lambda _: self._assemble(s), range(nconc)))
            t_workers = (time.perf_counter() - t0) / nconc
        self.nconc = nconc
        self.variant = "blas" if t_blas <= t_workers else "workers"
        self.threading = {"1 worker x all BLAS threads (s per max-m subdomain)": t_blas,
                          f"{nconc} workers x 1 BLAS thread (s per max-m subdomain, amortized)": t_workers}
        return self.variant

    def time_assembly(self):
        """One timed pass over the classes; returns (total s, {m: s per subdomain})."""
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits

        if self.variant is None:
            self.choose_threading()
        per, total = {}, 0.0
        for m, s, cnt in self.classes:
            if self.variant == "blas":
                t0 = time.perf_counter()
                self.fmats[m] = self._assemble(s)
                t = time.perf_counter() - t0
            else:
                k = min(self.nconc, cnt)
                with threadpool_limits(limits=1, user_api="blas"):
                    t0 = time.perf_counter()
                    with ThreadPoolExecutor(k) as ex:
                        outs = list(ex.map(lambda _: self._assemble(s), range(k)))
                    t = (time.perf_counter() - t0) / k
                self.fmats[m] = outs[0]
            per[m] = t
            total += t * cnt
        return total, per

    def time_sparse_storage(self, cols=128):
        """The reference's default (sparse-storage) forward solve on `cols`
        columns of the largest class, scaled by sum(m) / cols over `threads`
        concurrent subdomains."""
        from concurrent.futures import ThreadPoolExecutor

        ora, prob = self.ora, self.prob
        m, s, _ = self.classes[-1]
        cols = min(cols, m)
        bc, bv = prob.bcol[s][:cols], prob.bval[s][:cols]
        k = max(1, min(self.threads, prob.n_sub))
        t0 = time.perf_counter()
        with ThreadPoolExecutor(k) as ex:
            list(ex.map(lambda _: ora.assemble_explicit_local(self.up, self.ui, self.values[s], self.n, self.iperm,
                                                              bc, bv, storage="sparse"), range(k)))
        t = (time.perf_counter() - t0) / k
        sum_m = float(prob.m_per_subdomain().sum())
        return t * sum_m / cols, {"sample_cols": cols, "sample_s_per_copy": t, "concurrent_copies": k}

    def time_applies(self, reps=3):
        """(explicit apply s, implicit apply s) for the whole job."""
        from concurrent.futures import ThreadPoolExecutor

        ora, prob = self.ora, self.prob
        if not self.fmats:
            self.time_assembly()
        ms = prob.m_per_subdomain()
        cons = [(prob.gids[s], prob.bcol[s], prob.bval[s]) for s in range(prob.n_sub)]
        op = ora.OracleOperator([None] * prob.n_sub, cons, workers=self.threads)
        op.fmats = [self.fmats[int(ms[s])] for s in range(prob.n_sub)]
        p = np.random.default_rng(0).normal(size=prob.n_multipliers)
        op.apply(p)
        tt = []
        for _ in range(reps):
            t0 = time.perf_counter()
            op.apply(p)
            tt.append(time.perf_counter() - t0)
        t_expl = min(tt)
        k = max(1, min(self.threads, prob.n_sub))
        t_impl = 0.0
        with ThreadPoolExecutor(k) as ex:
            for m, s, cnt in self.classes:
                pl = np.random.default_rng(1).normal(size=m)
                c = min(k, cnt)
                t0 = time.perf_counter()
                list(ex.map(lambda _: ora.apply_implicit_local(self.up, self.ui, self.values[s], self.iperm,
                                                               prob.bcol[s], prob.bval[s], pl), range(c)))
                t_impl += (time.perf_counter() - t0) * math.ceil(cnt / c)
        return t_expl, t_impl

    def describe(self, per):
        return ", ".join(f"m={m}: {per[m]:.3f} s x{cnt}" for m, _, cnt in self.classes)


def amortization_point(impl, expl):
    """bench.py:99-116 of the reference (ceil of the crossing; 0; "never")."""
    t_pre_i, t_app_i = impl
    t_pre_e, t_app_e = expl
    denom = t_app_i - t_app_e
    numer = t_pre_e - t_pre_i
    if denom <= 0:
        return "never"
    if numer <= 0:
        return 0
    return int(math.ceil(numer / denom))


def dgemm_peak(dev):
    """Measured cuBLAS DGEMM ceiling (FP64 tensor pipe), TFLOP/s, best of 5."""
    import torch

    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6549.4)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config, ordering):
    """dram bytes per launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return {}
    with open(path) as fh:
        d = json.load(fh)
    return d.get(f"{config}/{ordering}", {})


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    if rank != 0:
        return
    from harness import inputs

    prob = inputs.Problem(*inputs.CONFIGS[args.config])
    ms = prob.m_per_subdomain()
    sample = int(np.argmax(ms))
    threads = os.cpu_count()
    if args.config == "c5":
        # the reference's dense K_reg path cannot run config 5: time the
        # oracle's sparse restatement instead, one bounded sample per step
        vals = []
        for i in range(args.warmup + args.steps):
            r = cpu_sparse_reference(prob, sample, min(threads, 8))
            log(f"[reference] step {i}: assembly {r['assembly_total_s']:.1f} s (sample {r['sample_s']:.1f} s)")
            if i >= args.warmup:
                vals.append(r)
        value = statistics.median(r["assembly_total_s"] for r in vals)
        r = vals[0]
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference problem generator)",
            "config": {"workload": f"{args.config}: {prob.physics} {prob.dim}D, {prob.n_sub} subdomains x "
                                   f"{prob.n_dofs} DOFs, {prob.n_multipliers} multipliers",
                       "parallelism": f"cpu{r['threads']}"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"], "kind": "port",
                             "sample": f"oracle sparse route (SuperLU + Woodbury) on subdomain {sample}, "
                                       f"{r['threads']} concurrent copies x{r['waves']} waves"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    cpu = CpuReference(prob, threads, log_fn=log)
    cpu.choose_threading()
    totals = []
    per = None
    for i in range(args.warmup + args.steps):
        total, per = cpu.time_assembly()
        if i >= args.warmup:
            totals.append(total)
        log(f"[reference] step {i}: assembly {total:.2f} s over {len(cpu.classes)} m-classes")
    value = statistics.median(totals)
    t_sparse, sp_info = cpu.time_sparse_storage()
    app_e, app_i = cpu.time_applies()
    sample = (f"explicit SYRK assembly, the reference's dense-storage config as is (densify, factor_to_dense, "
              f"dtrsm, dsyrk, zero_lower), one subdomain per multiplier-count class weighted by the class "
              f"counts ({cpu.describe(per)}), {cpu.variant} threading on {threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference problem generator)",
        "config": {"workload": f"{args.config}: {prob.physics} {prob.dim}D, {prob.n_sub} subdomains x "
                               f"{prob.n_dofs} DOFs, {prob.n_multipliers} multipliers", "ordering": "rcm",
                   "parallelism": f"cpu{threads}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "per_class_s": {str(k): v for k, v in per.items()},
                         "threading_s": cpu.threading,
                         "default_sparse_storage_s": t_sparse, "default_sparse_storage_sample": sp_info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "apply": {"explicit_ms_per_iter": app_e * 1e3, "implicit_ms_per_iter": app_i * 1e3},
        "host_factorization": {"lapack_s_per_subdomain": cpu.host_factorization_s},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def cpu_sparse_reference(prob, sample, threads):
    """CPU counterpart of the sparse-factor route (config 5, where the
    reference's dense K_reg path is infeasible): the oracle's SuperLU +
    Woodbury restatement of F~ = B~ K_reg^-1 B~^T on one max-m subdomain,
    `threads` concurrent copies, scaled to the job."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import feti_oracle as ora

    k, _, q = prob.subdomain_system(sample)
    n = prob.n_dofs
    bcol, bval = prob.bcol[sample], prob.bval[sample]
    nconc = max(1, min(threads, prob.n_sub))

    def one(_):
        sol = ora.WoodburyKregSolver(n, k.indptr, k.indices, k.data, q)
        return ora.fmatrix_via_solver(sol, n, bcol, bval)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(nconc) as ex:
        list(ex.map(one, range(nconc)))
    t = time.perf_counter() - t0
    waves = math.ceil(prob.n_sub / nconc)
    return {"assembly_total_s": t * waves, "sample_s": t, "threads": nconc, "waves": waves,
            "sample_subdomain": int(sample), "sample_m": int(bcol.shape[0])}


def merge_reference_factor_path(line, dense):
    """Attach the reference-factor-path measurements (assembly from the
    reference's own RCM factor) to the sparse-route headline line; the CPU
    baseline and amortization points come from that run's CPU legs."""
    keys = ("value", "roofline", "phases_ms", "flops", "apply", "e2e", "device_bytes", "solve",
            "device_factorization", "ordering_interface_last", "clocks", "gpu_launches")
    line["reference_factor_path"] = {k: dense[k] for k in keys if k in dense}
    line["reference_factor_path"]["what"] = (
        "F~ assembled from the reference's own factor (dense K_reg = K + rho Q Q^T, RCM = reversed natural order), "
        "factor resident in HBM (value) or uploaded from pinned host memory (e2e); host factorization excluded")
    for k in ("cpu_baseline", "host_factorization"):
        if k in dense:
            line[k] = dense[k]
    if "cpu_baseline" in dense:
        cpu = dense["cpu_baseline"]
        t_app = line["apply"]["e2e_ms_per_iter"] / 1e3
        line["amortization"] = {
            "vs_cpu_implicit": amortization_point((0.0, cpu["implicit_apply_ms"] / 1e3), (line["e2e"]["value"], t_app)),
            "vs_cpu_explicit": amortization_point((cpu["value"], cpu["explicit_apply_ms"] / 1e3),
                                                  (line["e2e"]["value"], t_app)),
            "with_factorization_vs_cpu_implicit": amortization_point(
                (dense.get("amortization", {}).get("host_factorization_total_s_estimate", 0.0),
                 cpu["implicit_apply_ms"] / 1e3), (line["e2e"]["value"], t_app)),
            "basis": "T_pre = sparse-route preprocess through the drop-in (K upload + device factorization + "
                     "assembly + correction, e2e); t_app = host-vector apply; the CPU implicit side pays its host "
                     "factorization in the last entry"}


def run_sparse(args, rank, world, local_rank):
    """Config 5 (2D elasticity, 256 x 33,282 DOFs) through the sparse-factor
    route: one step = device factorization of every K_s (block-sparse tiles,
    DMMA) + explicit assembly + rank-2r correction of every F~_i."""
    import torch
    import torch.distributed as dist

    from paper_2502_08382_b200 import _lib
    from paper_2502_08382_b200 import distributed as fd
    from harness import inputs
    from paper_2502_08382_b200 import dualop

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    multi = world > 1

    def barrier():
        if multi:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if not multi:
            return float(x)
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    prob = inputs.Problem(*inputs.CONFIGS[args.config], n_clusters=world)
    cons = prob.constraints()
    if args.assign == "lpt":
        owned = fd.lpt_subdomains(fd.apply_weights(cons), world, rank)
    else:
        owned = fd.owned_subdomains(prob.layout, rank)
    n = prob.n_dofs
    cfg = dualop.DualOpConfig(strategy="explicit", path="syrk")
    t0 = time.time()
    ks, qs, fs = {}, {}, {}
    pinned = []      # the step's inputs live in page-locked host memory (e2e contract)
    for s in owned:
        k, f, q = prob.subdomain_system(s)
        pk = _lib.PinnedArray(k.data.shape[0])
        pk.array[:] = k.data
        pq = _lib.PinnedArray(q.size)
        pq.array[:] = q.ravel()
        pinned += [pk, pq]
        ks[s] = inputs.Csr(k.shape, k.indptr, k.indices, pk.array)
        qs[s], fs[s] = pq.array.reshape(q.shape), f
    stiff = [ks.get(s) for s in range(prob.n_sub)]
    kern = [qs.get(s) for s in range(prob.n_sub)]
    mats = [inputs.ShapeOnly((n, n)) for _ in range(prob.n_sub)]
    log(f"[rank {rank}] {args.config}: inputs for {len(owned)} subdomains in {time.time() - t0:.1f}s")
    t0 = time.time()
    op = dualop.DualOperator(mats, cons, prob.layout, cfg, device=local_rank, subdomains=owned,
                             factorization="sparse", stiffness=stiff, kernels=kern)
    op.prepare()
    t_prepare = time.time() - t0
    log(f"[rank {rank}] prepare (ordering, fixing DOFs, block symbolic, allocation) {t_prepare:.1f}s")
    walls, fac_ms, asm_ms, pre_ms, host_up = [], [], [], [], []
    sampler = None
    # e2e: the public preprocess() from host arrays (K values + kernel basis
    # H2D inside the step)
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        op.preprocess()
        barrier()
        if i >= args.warmup:
            walls.append(time.perf_counter() - t0)
            host_up.append(op.timings.get("stiffness_upload_s", 0.0))
    # value: the device step with K resident in HBM (CUDA events on the
    # library's streams: factorization start -> last group's correction)
    for i in range(args.warmup + args.steps):
        if i == args.warmup and rank == 0:
            sampler = ClockSampler(local_rank).start()
        barrier()
        op.preprocess_resident()
        barrier()
        if i >= args.warmup:
            st = op.stats()
            fac_ms.append(st["ms_factorize"])
            asm_ms.append(st["ms_assemble"])
            pre_ms.append(st["ms_preprocess"])
    clocks = sampler.stop() if sampler else None
    st = op.stats()
    step_ms = max_over_ranks(statistics.mean(pre_ms))
    pre_wall = max_over_ranks(statistics.mean(walls))
    dco = fd.ClusterDualOperator(op, prob.n_multipliers, dev)
    p_dev = torch.from_numpy(np.random.default_rng(0).normal(size=prob.n_multipliers)).to(dev)
    q_dev = torch.empty_like(p_dev)
    for _ in range(10):
        dco.apply_device(p_dev, q_dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream(dev).cuda_stream
    # the whole apply at N GPUs: local SYMV + the fused cross-rank exchange
    # (max over ranks); at N = 1 the exchange is absent
    e0.record()
    for _ in range(args.applies):
        dco.apply_device(p_dev, q_dev)
    e1.record()
    e1.synchronize()
    dco.check()
    apply_ms = max_over_ranks(e0.elapsed_time(e1) / args.applies)
    e0.record()
    for _ in range(args.applies):
        op.apply_device(p_dev, q_dev, stream)
    e1.record()
    e1.synchronize()
    apply_kernel_ms = max_over_ranks(e0.elapsed_time(e1) / args.applies)
    p_host = np.random.default_rng(1).normal(size=prob.n_multipliers)
    q_host = np.zeros(prob.n_multipliers)
    ta = []
    for _ in range(20):
        barrier()
        t0 = time.perf_counter()
        if multi:
            dco.apply(p_host if rank == 0 else None, out=q_host)
        else:
            op.apply(p_host, out=q_host)
        ta.append(time.perf_counter() - t0)
    apply_e2e_ms = max_over_ranks(statistics.median(ta) * 1e3)
    h2d = int(sum(ks[s].indptr[-1] * 8 + qs[s].size * 8 for s in owned)) + 8 * prob.n_multipliers
    recipe = op.sparse_recipe
    op.close()
    del op, dco, p_dev, q_dev
    torch.cuda.empty_cache()
    implicit = None
    if world == 1:
        # the reference's default strategy on the same route: no F~, each apply
        # = two block sweeps over K_s's trailing tiles + the rank-2r correction;
        # the amortization point vs the explicit strategy (the paper's metric)
        iop = dualop.DualOperator(mats, cons, prob.layout, dualop.DualOpConfig(strategy="implicit"),
                                  device=local_rank, subdomains=owned, factorization="sparse", stiffness=stiff,
                                  kernels=kern)
        iop.prepare()
        iop.preprocess()
        ipre = []
        for i in range(args.warmup + args.steps):
            barrier()
            iop.preprocess_resident()
            barrier()
            if i >= args.warmup:
                ipre.append(iop.stats()["ms_preprocess"])
        p_dev = torch.from_numpy(np.random.default_rng(0).normal(size=prob.n_multipliers)).to(dev)
        q_dev = torch.empty_like(p_dev)
        for _ in range(5):
            iop.apply_implicit_device(p_dev, q_dev, stream)
        n_impl = max(10, args.applies // 10)
        e0.record()
        for _ in range(n_impl):
            iop.apply_implicit_device(p_dev, q_dev, stream)
        e1.record()
        e1.synchronize()
        imp_ms = e0.elapsed_time(e1) / n_impl
        ipre_ms = statistics.mean(ipre)
        implicit = {"preprocess_ms": ipre_ms, "apply_ms_per_iter": imp_ms,
                    "amortization_explicit_vs_implicit": amortization_point(
                        (ipre_ms / 1e3, imp_ms / 1e3), (step_ms / 1e3, apply_kernel_ms / 1e3)),
                    "what": "strategy='implicit' on the sparse route (device, K resident): preprocess = K_s "
                            "factorization + diagonal inverses + block scaling + U2 backward sweep; apply = "
                            "forward/backward block sweeps (2-CTA cluster per subdomain) + correction + reduction"}
        log(f"[rank {rank}] implicit strategy: preprocess {ipre_ms:.1f} ms, apply {imp_ms:.3f} ms")
        iop.close()
        del iop, p_dev, q_dev
        torch.cuda.empty_cache()
    solve = None
    if world == 1 and args.solve:
        # the device-native PCPG on this route: the loads
        # are factored along (d = B~ K^+ f from the device), G / G^T G / e on
        # the host (mesh-only, sparse), the whole iteration on the device
        from paper_2502_08382_b200.pcpg import DevicePCPG

        forces = [fs.get(s) for s in range(prob.n_sub)]
        t0 = time.perf_counter()
        sop = dualop.DualOperator(mats, cons, prob.layout, cfg, device=local_rank, subdomains=owned,
                                  factorization="sparse", stiffness=stiff, kernels=kern, forces=forces)
        sop.prepare()
        sop.preprocess()
        t_pre = time.perf_counter() - t0
        t0 = time.perf_counter()
        solver = DevicePCPG(sop, kern, forces, prob.c)
        t_setup = time.perf_counter() - t0
        solver.solve(tol=1e-9)                                 # warm-up (graph capture)
        lam, iters, t_wall = solver.solve(tol=1e-9)
        dev_ms = solver.last_device_ms
        solve = {"pcpg_iterations": iters, "tol": 1e-9, "device_loop_ms": dev_ms,
                 "ms_per_iteration": dev_ms / max(iters, 1), "solve_call_s": t_wall,
                 "dual_system_setup_s": t_setup, "lambda_norm": float(np.linalg.norm(lam)),
                 "relative_residual": solver.relative_residual,
                 "what": "feti_pcpg_solve: apply + projections + inner products + stopping test on the device "
                         "(graph of 8 iterations, one status read per graph); dual_system_setup_s = G, G^T G "
                         "and e on the host + d = B~ K^+ f read back from the factorization (the loads factored "
                         "along), after a preprocess of " f"{t_pre:.1f} s (prepare included)"}
        log(f"[rank {rank}] device PCPG {iters} iterations, {dev_ms:.1f} ms loop, setup {t_setup:.3f} s")
        sop.close()
        del sop, solver
        torch.cuda.empty_cache()
    if rank != 0:
        return None
    peak_f64 = dgemm_peak(dev)
    hbm_peak, hbm_src = load_peaks()
    fac_s = statistics.mean(fac_ms) / 1e3
    app_bytes = st["apply_bytes_alg"]
    line = {
        "metric": METRIC, "value": step_ms / 1e3, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's problem regenerated (inputs.py); sparse K + kernel basis per subdomain",
        "config": {"workload": f"{args.config}: {prob.physics} {prob.dim}D, {prob.n_sub} subdomains x {n} DOFs, "
                               f"{prob.n_multipliers} multipliers", "route": "sparse-factor (K_s + rank-2r correction)",
                   "ordering": f"constrained DOFs last; interior recipe {recipe!r} (tile-flop estimator, sparse_route.choose_ordering)",
                   "parallelism": f"cluster-per-gpu x{world} ({args.assign})",
                   "l2": f"inputs larger than L2 (block-sparse factor tiles {st['bytes_temporary'] / 1e9:.0f} GB, "
                         f"packed F~ {8 * sum(m * (m + 1) / 2 for m in prob.m_per_subdomain()) / 1e9:.2f} GB "
                         f"per apply)"},
        # the step is one captured CUDA graph per subdomain group: the group's factorization
        # (sp_gemm8 tile tasks + sp_potrf) with its interface assembly (TRSM
        # chain, U2, SYRK + correction) behind it on the group's stream
        "roofline": (lambda alg, ex: {
            "bound": "tensor",
            "kernel": "the step's CUDA graphs (one per subdomain group): sp_gemm8_kernel + sp_potrf_kernel (factorization) and trsm_chain / "
                      "sp_u2 / syrk (interface assembly), FP64 DMMA tile work",
            "achieved": alg / (step_ms / 1e3) / 1e12, "peak": peak_f64, "unit": "TFLOP/s",
            "frac": alg / (step_ms / 1e3) / 1e12 / peak_f64,
            "peak_source": "measured in-run: cuBLAS DGEMM 8192^3 f64 (torch.matmul), best of 5",
            "traffic": load_traffic(args.config, "sparse").get("step (fused graph, per step)"),
            "traffic_note": "DRAM read+write of every launch of one step (ncu dram__bytes_*.sum summed over the "
                            "launch list, profiles/ncu_traffic.json); tiles are re-read per tile product, but at "
                            "~1 TB/s the step is not HBM-bound",
            "algorithmic": "scalar Cholesky flops of K_s in the chosen ordering, sum_j c_j (c_j + 3) from the exact "
                           "column counts (+ the y = L^-1 P Q solve), plus the pruned interface TRSM "
                           "sum_j (n_I - r_j)^2 and SYRK sum_(a<=b) 2 (n_I - max(r_a, r_b)) flops, per step",
            "algorithmic_flops": alg, "executed_tile_flops": ex,
            "achieved_executed": ex / (step_ms / 1e3) / 1e12,
            "frac_executed": ex / (step_ms / 1e3) / 1e12 / peak_f64,
            "note": f"128-row tiles execute executed/algorithmic = {ex / max(alg, 1.0):.2f}x; frac_executed is "
                    "the DMMA pipe's utilisation over the step"})(
            st["flops_factor_alg"] + st["flops_trsm_alg"] + st["flops_syrk_alg"],
            st["flops_factor_exec"] + st["flops_trsm_exec"] + st["flops_syrk_exec"] + st["flops_scale_exec"]),
        "roofline_factorization": {
            "bound": "tensor", "kernel": "sp_gemm8_kernel + sp_potrf_kernel", "unit": "TFLOP/s", "peak": peak_f64,
            "algorithmic_flops": st["flops_factor_alg"], "executed_tile_flops": st["flops_factor_exec"],
            "achieved": st["flops_factor_alg"] / fac_s / 1e12, "frac": st["flops_factor_alg"] / fac_s / 1e12 / peak_f64,
            "frac_executed": st["flops_factor_exec"] / fac_s / 1e12 / peak_f64,
            "what": "supplementary: factorization flops over ms_factorize (the last group's factorization end; "
                    "in the fused graph that span also carries the earlier groups' interface assembly)"},
        "assembly_flops": {k: st[k] for k in ("flops_trsm_alg", "flops_trsm_exec", "flops_syrk_alg",
                                              "flops_syrk_exec", "flops_scale_exec")},
        "phases_ms": {"ms_factorize": statistics.mean(fac_ms), "ms_preprocess": statistics.mean(pre_ms),
                      "ms_assembly_tail": statistics.mean(asm_ms),
                      "note": "each group's interface assembly + correction is captured right behind its "
                              "factorization in the group's step graph; ms_assembly_tail = past the last "
                              "group's factorization"},
        "apply": {"ms_per_iter": apply_ms, "kernel_ms_per_iter": apply_kernel_ms, "e2e_ms_per_iter": apply_e2e_ms,
                  "what": "ms_per_iter: local kernels + fused exchange (N > 1), max over ranks; kernel_ms_per_iter: "
                          "this rank's apply kernels alone; e2e: host p -> q through the public API",
                  "roofline": {"bound": "hbm", "kernel": "apply_kernel + reduce_kernel",
                               "achieved": app_bytes / (apply_kernel_ms / 1e3) / 1e9, "peak": hbm_peak,
                               "unit": "GB/s", "frac": app_bytes / (apply_kernel_ms / 1e3) / 1e9 / hbm_peak,
                               "peak_source": hbm_src, "algorithmic_bytes": app_bytes,
                               "traffic": (lambda t: (t.get("apply_kernel<8>", 0) + t.get("reduce_kernel", 0)) or None)(
                                   load_traffic(args.config, "sparse")) if world == 1 else None,
                               "traffic_note": "DRAM read+write per apply (apply_kernel + reduce_kernel, ncu "
                                               "dram__bytes_*.sum, profiles/ncu_traffic.json, r02_apply_traffic.md)"}},
        "e2e": {"value": pre_wall + apply_e2e_ms / 1e3, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": int(8 * prob.n_multipliers),
                "what": "preprocess through the drop-in (sparse K values + kernel basis H2D from page-locked host "
                        "buffers, device factorization, assembly, correction) + one apply with host p/q"},
        "prepare_s": t_prepare,
        "implicit_strategy": implicit,
        "solve": solve,
        "host_side_ms": {"stiffness_upload_per_step": statistics.mean(host_up) * 1e3,
                         "preprocess_wall_per_step": statistics.mean(walls) * 1e3},
        "device_bytes": {"persistent": st["bytes_persistent"], "temporary": st["bytes_temporary"]},
        "gpu_launches": int(args.steps * (st["launches_factorize"] + st["launches_assemble"])),
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline and args.config == "c5":
        ms = prob.m_per_subdomain()
        sample = int(np.argmax(ms))
        cpu = cpu_sparse_reference(prob, sample, os.cpu_count())
        line["cpu_baseline"] = {
            "value": cpu["assembly_total_s"], "unit": UNIT, "cores": cpu["threads"], "kind": "port",
            "sample": f"oracle sparse route (SuperLU of K_s' + Woodbury, F~ = B~ K_reg^-1 B~^T) on subdomain "
                      f"{sample} (m={cpu['sample_m']}): {cpu['threads']} concurrent copies = {cpu['sample_s']:.2f} s, "
                      f"x{cpu['waves']} waves for {prob.n_sub} subdomains; the reference's own dense path cannot "
                      f"run this config (4.4 GB factor per subdomain)"}
    return line


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2502_08382_b200 import _lib
    from paper_2502_08382_b200 import distributed as fd
    from harness import inputs
    from paper_2502_08382_b200 import dualop

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    multi = world > 1

    def barrier():
        if multi:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if not multi:
            return float(x)
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    prob = inputs.Problem(*inputs.CONFIGS[args.config], n_clusters=world)
    cons = prob.constraints()
    owned = fd.owned_subdomains(prob.layout, rank)
    n = prob.n_dofs
    cfg = dualop.DualOpConfig(strategy="explicit", path="syrk")

    def measure(ordering, keep_host=False):
        """Everything for one symbolic ordering: device-resident assembly,
        apply, end-to-end from pinned host factors."""
        perms = {s: (rcm_perm_dense(n) if ordering == "rcm" else interface_last_perm(n, prob.bcol[s]))
                 for s in owned}
        t0 = time.time()
        mask_cache = {}
        dev_factors, host_factors = {}, {}
        all_dense = True
        for s in owned:
            packed, dense_ok = device_factor(prob, s, perms[s], dev, mask_cache)
            all_dense &= dense_ok
            dev_factors[s] = packed
            pa = _lib.PinnedArray(packed.numel())
            torch.from_numpy(pa.array).copy_(packed)
            host_factors[s] = pa
        mask_cache.clear()
        torch.cuda.empty_cache()
        if not all_dense:
            raise RuntimeError("K_reg has exact zeros: reversed natural order is not the RCM ordering")
        log(f"[rank {rank}] {ordering}: factors for {len(owned)} subdomains in {time.time() - t0:.1f}s")
        mats = [inputs.ShapeOnly((n, n)) for _ in range(prob.n_sub)]
        op = dualop.DualOperator(mats, cons, prob.layout, cfg, device=local_rank, subdomains=owned, perms=perms)
        op.prepare()
        for s in owned:
            op.set_factor(s, dev_factors[s], on_device=True)
        # value: device-resident assembly, CUDA events on the launching stream
        for _ in range(args.warmup):
            op.assemble()
        barrier()
        sampler = ClockSampler(local_rank).start() if rank == 0 else None
        step_ms, stats = [], None
        for _ in range(args.steps):
            op.assemble()
            stats = op.stats()
            step_ms.append(stats["ms_assemble"])
        barrier()
        clocks = sampler.stop() if sampler else None
        ms_step = max_over_ranks(statistics.mean(step_ms))
        # apply: device-resident (kernels + NCCL all-reduce for N > 1)
        dco = fd.ClusterDualOperator(op, prob.n_multipliers, dev)
        p_dev = torch.from_numpy(np.random.default_rng(0).normal(size=prob.n_multipliers)).to(dev)
        q_dev = torch.empty_like(p_dev)
        for _ in range(10):
            dco.apply_device(p_dev, q_dev)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.applies):
            dco.apply_device(p_dev, q_dev)
        e1.record()
        e1.synchronize()
        apply_ms = max_over_ranks(e0.elapsed_time(e1) / args.applies)
        stream = torch.cuda.current_stream(dev).cuda_stream
        e0.record()
        for _ in range(args.applies):
            op.apply_device(p_dev, q_dev, stream)
        e1.record()
        e1.synchronize()
        apply_kernel_ms = e0.elapsed_time(e1) / args.applies
        # implicit strategy on the device through the same factor tiles
        n_impl = max(3, args.applies // 20)
        op.apply_implicit_device(p_dev, q_dev, stream)
        e0.record()
        for _ in range(n_impl):
            op.apply_implicit_device(p_dev, q_dev, stream)
        e1.record()
        e1.synchronize()
        implicit_ms = e0.elapsed_time(e1) / n_impl
        # e2e: pinned host factors -> H2D -> device assembly -> one host apply
        p_host = np.random.default_rng(1).normal(size=prob.n_multipliers)
        q_host = np.zeros(prob.n_multipliers)
        e2e = []
        for i in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            for s in owned:
                op.set_factor(s, host_factors[s].array)
            op.assemble()
            if multi:
                dco.apply(p_host if rank == 0 else None, out=q_host)
            else:
                op.apply(p_host, out=q_host)
            barrier()
            if i >= args.warmup:
                e2e.append(time.perf_counter() - t0)
        st_host = op.stats()
        e2e_s = max_over_ranks(statistics.mean(e2e))
        ta = []
        for _ in range(20):
            barrier()
            t0 = time.perf_counter()
            if multi:
                dco.apply(p_host if rank == 0 else None, out=q_host)
            else:
                op.apply(p_host, out=q_host)
            ta.append(time.perf_counter() - t0)
        apply_e2e_ms = max_over_ranks(statistics.median(ta) * 1e3)
        solve = None
        if world == 1 and args.solve:
            # GPU-resident PCPG on this operator; the host
            # factors handed over in the e2e loop serve solve_local for d
            from paper_2502_08382_b200.pcpg import DevicePCPG

            t0 = time.perf_counter()
            kernels, forces = [], []
            for s in range(prob.n_sub):
                _, f, qk = prob.subdomain_system(s)
                kernels.append(qk)
                forces.append(f)
            solver = DevicePCPG(op, kernels, forces, prob.c)
            t_setup = time.perf_counter() - t0
            solver.solve(tol=1e-9)                       # warm-up (lazy library init)
            lam, iters, t_loop = solver.solve(tol=1e-9)
            solve = {"pcpg_iterations": iters, "device_loop_s": t_loop, "ms_per_iteration": t_loop / max(iters, 1) * 1e3,
                     "dual_system_setup_s": t_setup, "lambda_norm": float(np.linalg.norm(lam)), "tol": 1e-9}
            log(f"[rank {rank}] {ordering}: device PCPG {iters} iterations in {t_loop * 1e3:.1f} ms")
        res = {"ordering": ordering, "ms_step": ms_step, "stats": stats, "clocks": clocks, "apply_ms": apply_ms,
               "implicit_ms": implicit_ms,
               "apply_kernel_ms": apply_kernel_ms, "e2e_s": e2e_s, "apply_e2e_ms": apply_e2e_ms,
               "h2d_bytes": int(st_host["factor_bytes"]) + 8 * prob.n_multipliers,
               "host_factors": host_factors if keep_host else None, "perms": perms, "solve": solve}
        op.close()
        del dev_factors, dco, p_dev, q_dev
        torch.cuda.empty_cache()
        return res

    def measure_device_factor():
        """The host factorization moved to the GPU: upload the sparse
        K + kernel basis, form K_reg and factor it on the device, then assemble."""
        ks, qs = {}, {}
        for s in owned:
            k, _, q = prob.subdomain_system(s)
            ks[s], qs[s] = k, q
        mats = [inputs.ShapeOnly((n, n)) for _ in range(prob.n_sub)]
        stiff = [ks.get(s) if s in ks else inputs.ShapeOnly((n, n)) for s in range(prob.n_sub)]
        kern = [qs.get(s) if s in qs else np.zeros((n, 1)) for s in range(prob.n_sub)]
        op = dualop.DualOperator(mats, cons, prob.layout, cfg, device=local_rank, subdomains=owned,
                                 ordering=args.ordering, factorization="device", stiffness=stiff, kernels=kern)
        op.prepare()
        walls, fac_ms, asm_ms = [], [], []
        for i in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            op.preprocess()
            barrier()
            if i >= args.warmup:
                walls.append(time.perf_counter() - t0)
                st = op.stats()
                fac_ms.append(st["ms_factorize"])
                asm_ms.append(st["ms_assemble"])
        flops = sum(float(n) ** 3 / 3.0 for _ in owned)
        res = {"preprocess_e2e_s": max_over_ranks(statistics.mean(walls)),
               "factorize_ms": max_over_ranks(statistics.mean(fac_ms)),
               "assemble_ms": max_over_ranks(statistics.mean(asm_ms)),
               "factorize_tflops": flops / (statistics.mean(fac_ms) / 1e3) / 1e12,
               "h2d_bytes_per_step": int(sum(ks[s].indptr[-1] * 8 + qs[s].size * 8 for s in owned)),
               "what": "sparse K + kernel basis uploaded, K_reg = P(K + rho Q Q^T)P^T formed and factored on the GPU "
                       "(blocked right-looking Cholesky on DMMA), then the assembly; replaces the host LAPACK "
                       "factorization and the factor upload"}
        op.close()
        torch.cuda.empty_cache()
        return res

    main_res = measure(args.ordering)
    alt = None
    if not args.single_ordering:
        alt = measure("interface_last" if args.ordering == "rcm" else "rcm")
    devfac = measure_device_factor() if args.device_factor else None
    if rank != 0:
        return None
    peak_f64 = dgemm_peak(dev)
    hbm_peak, hbm_src = load_peaks()

    def summarize(r):
        st = r["stats"]
        traffic = load_traffic(args.config, r["ordering"])
        trsm_s = st["ms_trsm"] / 1e3
        alg_trsm, alg_syrk = st["flops_trsm_alg"], st["flops_syrk_alg"]
        value = r["ms_step"] / 1e3
        roof_trsm = {"bound": "tensor", "kernel": "trsm_chain_kernel (FP64 DMMA)",
                     "achieved": alg_trsm / trsm_s / 1e12, "peak": peak_f64, "unit": "TFLOP/s",
                     "frac": alg_trsm / trsm_s / 1e12 / peak_f64,
                     "peak_source": "measured in-run: cuBLAS DGEMM 8192^3 f64 (torch.matmul), best of 5",
                     "traffic": traffic.get("trsm_chain_kernel"),
                     "algorithmic": "sum_j (n - r_j)^2 pruned forward-solve flops per launch",
                     "executed_flops": st["flops_trsm_exec"], "algorithmic_flops": alg_trsm}
        app_bytes = st["apply_bytes_alg"]
        roof_apply = {"bound": "hbm", "kernel": "apply_kernel + reduce_kernel",
                      "achieved": app_bytes / (r["apply_kernel_ms"] / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": app_bytes / (r["apply_kernel_ms"] / 1e3) / 1e9 / hbm_peak, "peak_source": hbm_src,
                      "traffic": traffic.get("apply_kernel"),
                      "algorithmic": "packed F~ (8 m(m+1)/2) + 28 m per subdomain + 16 n_mult bytes per apply",
                      "algorithmic_bytes": app_bytes}
        return value, {
            "roofline": roof_trsm,
            "phases_ms": {k: st[k] for k in ("ms_unpack", "ms_diag_inverse", "ms_block_scale", "ms_trsm",
                                             "ms_syrk")},
            "flops": {"trsm_alg": alg_trsm, "syrk_alg": alg_syrk, "trsm_exec": st["flops_trsm_exec"],
                      "syrk_exec": st["flops_syrk_exec"], "scale_exec": st["flops_scale_exec"],
                      "assembly_alg_tflops": (alg_trsm + alg_syrk) / value / 1e12,
                      "assembly_alg_frac_of_dgemm": (alg_trsm + alg_syrk) / value / 1e12 / peak_f64},
            "apply": {"ms_per_iter": r["apply_ms"], "kernel_ms_per_iter": r["apply_kernel_ms"],
                      "e2e_ms_per_iter": r["apply_e2e_ms"], "roofline": roof_apply,
                      "gpu_implicit_ms_per_iter": r["implicit_ms"],
                      "amortization_vs_gpu_implicit": amortization_point(
                          (0.0, r["implicit_ms"] / 1e3), (value, r["apply_kernel_ms"] / 1e3))},
            "e2e": {"value": r["e2e_s"], "unit": UNIT, "h2d_bytes_per_step": r["h2d_bytes"],
                    "d2h_bytes_per_step": int(8 * prob.n_multipliers),
                    "what": "pinned host factors (reference layout; the lib copies the suffix the pruned solve "
                            "reads) -> device assembly -> one apply with host p/q"},
            "device_bytes": {"persistent": st["bytes_persistent"], "temporary": st["bytes_temporary"]},
            "solve": r["solve"],
        }

    value, fields = summarize(main_res)
    st = main_res["stats"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main_res["ms_step"], "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's problem regenerated (inputs.py), factors computed in setup",
        "config": {"workload": f"{args.config}: {prob.physics} {prob.dim}D, {prob.n_sub} subdomains x {n} DOFs, "
                               f"{prob.n_multipliers} multipliers", "ordering": args.ordering,
                   "parallelism": f"cluster-per-gpu x{world}",
                   "l2": "inputs larger than L2 (factors 22 GB, packed F~ 1.1 GB per apply)"},
    }
    line.update(fields)
    line["gpu_launches"] = int(args.steps * st["launches_assemble"])
    if devfac is not None:
        line["device_factorization"] = devfac
    line["clocks"] = main_res["clocks"]
    if alt is not None:
        v2, f2 = summarize(alt)
        line[f"ordering_{alt['ordering']}"] = {"value": v2, **{k: f2[k] for k in
                                                              ("e2e", "phases_ms", "flops", "roofline", "apply",
                                                               "solve")}}
    if world == 1 and not args.no_cpu_baseline:
        ms = prob.m_per_subdomain()
        sample = int(np.argmax(ms))
        from paper_2502_08382_b200 import factor as fct

        t0 = time.perf_counter()
        kreg = inputs.DenseSym(prob.kreg_dense(sample))
        t_dense = time.perf_counter() - t0
        t0 = time.perf_counter()
        fct.numeric_factorize_dense(kreg, main_res["perms"][sample])
        t_fac = time.perf_counter() - t0
        del kreg
        cpu_ref = CpuReference(prob, log_fn=log)
        cpu_ref.choose_threading()
        total, per = cpu_ref.time_assembly()
        t_sparse, sp_info = cpu_ref.time_sparse_storage()
        t_expl, t_impl = cpu_ref.time_applies()
        cpu = {"assembly_total_s": total, "explicit_apply_s": t_expl, "implicit_apply_s": t_impl,
               "threads": cpu_ref.threads}
        line["cpu_baseline"] = {
            "value": total, "unit": UNIT, "cores": cpu_ref.threads, "kind": "port",
            "sample": f"CPU explicit SYRK assembly, the reference's dense-storage config as is (densify, "
                      f"factor_to_dense, dtrsm, dsyrk, zero_lower; dualop.py:427-501), one subdomain per "
                      f"multiplier-count class weighted by the class counts ({cpu_ref.describe(per)}), "
                      f"{cpu_ref.variant} threading on {cpu_ref.threads} host threads",
            "per_class_s": {str(k): v for k, v in per.items()},
            "threading_s": cpu_ref.threading,
            "default_sparse_storage_s": t_sparse, "default_sparse_storage_sample": sp_info,
            "explicit_apply_ms": t_expl * 1e3,
            "implicit_apply_ms": t_impl * 1e3,
            "implicit_sample": f"apply_implicit_local per m-class, {min(cpu_ref.threads, prob.n_sub)} concurrent, "
                               f"weighted by the class counts"}
        line["host_factorization"] = {
            "lapack_dpotrf_s_per_subdomain": t_fac, "dense_kreg_build_s": t_dense,
            "note": "host numeric factorization (before the path; common to implicit and explicit, cancels "
                    "in the amortization point)"}
        t_app_gpu = main_res["apply_e2e_ms"] / 1e3
        line["amortization"] = {
            "vs_cpu_implicit": amortization_point((0.0, cpu["implicit_apply_s"]), (main_res["e2e_s"], t_app_gpu)),
            "vs_cpu_explicit": amortization_point((cpu["assembly_total_s"], cpu["explicit_apply_s"]),
                                                  (main_res["e2e_s"], t_app_gpu)),
            "basis": "T_pre = factor upload + device assembly (e2e); t_app = host-vector apply; the host "
                     "factorization is common to both sides and cancels"}
        if devfac is not None:
            # whole preprocess incl. factorization: device path vs the CPU implicit
            # path, whose preprocess is the host factorization alone
            t_fac_host = t_fac * prob.n_sub
            line["amortization"]["with_factorization_vs_cpu_implicit"] = amortization_point(
                (t_fac_host, cpu["implicit_apply_s"]), (devfac["preprocess_e2e_s"], t_app_gpu))
            line["amortization"]["host_factorization_total_s_estimate"] = t_fac_host
    return line


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="c3", choices=("c1", "c2", "c3", "c4", "c5"))
    ap.add_argument("--route", default=None, choices=("dense", "sparse"),
                    help="factor route (default: sparse for c3-c5, dense for c1-c2)")
    ap.add_argument("--sparse-only", action="store_true",
                    help="sparse route: skip the reference-factor-path measurements")
    ap.add_argument("--ordering", default="rcm", choices=("rcm", "interface_last"))
    ap.add_argument("--assign", default="contiguous", choices=("contiguous", "lpt"),
                    help="subdomain -> rank: the reference's contiguous clusters or LPT by packed F~ bytes")
    ap.add_argument("--applies", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-device-factor", dest="device_factor", action="store_false",
                    help="skip the device-factorization measurement")
    ap.add_argument("--no-solve", dest="solve", action="store_false",
                    help="skip the GPU-resident PCPG solve measurement")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="gloo only to exercise N > 1 with several ranks sharing one GPU")
    ap.add_argument("--single-ordering", action="store_true",
                    help="skip the second (alternative ordering) measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        local_rank = local_rank % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:   # gloo: exercises the N > 1 code path with several ranks on one GPU
            dist.init_process_group("gloo")
    try:
        route = args.route or ("sparse" if args.config in ("c3", "c4", "c5") else "dense")
        line = None
        if route == "sparse":
            line = run_sparse(args, rank, world, local_rank)
            if args.config != "c5" and not args.sparse_only:
                # the reference-factor path on the same box: assembly from the
                # reference's own (dense-pattern RCM) factor, the CPU baseline
                dense = run_ours(args, rank, world, local_rank)
                if line is not None:
                    merge_reference_factor_path(line, dense)
        else:
            line = run_ours(args, rank, world, local_rank)
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

/*
 * feti_b200.h -- C-ABI of the B200-native explicit FETI local dual operator.
 *
 * This is the drop-in boundary for the explicit strategy of the reference's
 * `tfeti.dualop.DualOperator` (arXiv 2502.08382 reference, pkg/src/tfeti).
 * The reference is pure Python+numba and has no FFI of its own; the entry
 * points below are exactly the operations its object interface performs on
 * the hot path, so a ctypes binding can stand in for them.
 * Plain C types only: pointers, sizes, status codes.  No torch types.
 *
 * Status codes: 0 = ok, otherwise one of FETI_ERR_*; feti_last_error()
 * returns a thread-local message for the last failing call on this thread.
 *
 * Reference interface each entry replaces (file:line under pkg/src/tfeti/):
 *   feti_create            DualOperator.__init__            dualop.py:124-148
 *   feti_add_subdomain     prepare(), per subdomain: B~ permutation by the
 *                          factor's iperm, persistent buffers
 *                                                           dualop.py:233-248, 85-97
 *   feti_finalize          prepare(), capacity check / layout
 *                                                           dualop.py:250-269
 *   feti_set_factor        numeric refill target of CholFactor.values
 *                                                           dualop.py:313, sparse.py:287-299
 *   feti_assemble          assemble_explicit_local (SYRK path) for every
 *                          subdomain, inside preprocess     dualop.py:316-320, 427-501
 *   feti_local_operator    local_operator(i)                dualop.py:399-401
 *   feti_apply             apply(p, out)                    dualop.py:348-388
 *   feti_apply_device      apply on device-resident vectors (multi-GPU / solver on device)
 *   feti_destroy           close()                          dualop.py:198-208
 */
#ifndef FETI_B200_H
#define FETI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FETI_B200_ABI_VERSION 1

enum {
  FETI_OK = 0,
  FETI_ERR_ARG = 1,        /* maps to ValueError                         */
  FETI_ERR_LIFECYCLE = 2,  /* maps to dualop.LifecycleError              */
  FETI_ERR_CUDA = 3,       /* CUDA runtime failure (RuntimeError)        */
  FETI_ERR_CAPACITY = 4,   /* device memory too small: PoolCapacityError */
  FETI_ERR_SINGULAR = 5,   /* zero diagonal in the factor: SingularFactorError (sparse.py:491-492) */
  FETI_ERR_INTERNAL = 6,
  FETI_ERR_NOT_SPD = 7,    /* non-positive pivot in the device factorization: SpdError (sparse.py:297-298) */
  FETI_ERR_BREAKDOWN = 8,  /* PCPG: p^T F p <= 0, BreakdownError (solver.py:40-41, 246-247) */
  FETI_ERR_NOT_CONVERGED = 9 /* PCPG: iteration cap reached, ConvergenceError (solver.py:44-45, 263-267) */
};

enum { FETI_FACTOR_HOST = 0, FETI_FACTOR_DEVICE = 1 };

/* DualOpConfig.strategy (dualop.py:55-82): explicit F~ (default), or the
 * implicit strategy -- no F~, each apply runs two block triangular sweeps
 * over the factor (apply_implicit_local, dualop.py:504-521). */
enum { FETI_STRATEGY_EXPLICIT = 0, FETI_STRATEGY_IMPLICIT = 1 };
enum { FETI_PATH_SYRK = 0, FETI_PATH_TRSM = 1 };

typedef struct feti_ctx feti_ctx;

typedef struct feti_stats {
  /* device time of the last feti_assemble, per phase (CUDA events, ms) */
  double ms_wait_upload;  /* waiting for host->device factor copies     */
  double ms_unpack;
  double ms_diag_inverse;
  double ms_block_scale;
  double ms_trsm;
  double ms_syrk;
  double ms_assemble;     /* sum of the above device phases             */
  double ms_apply;        /* device time of the last apply (kernels)    */
  /* algorithmic work and what the kernels execute */
  double flops_trsm_alg;  /* sum_j (n - r_j)^2                          */
  double flops_syrk_alg;  /* sum_{a<=b} 2 (n - max(r_a, r_b))           */
  double flops_trsm_exec;
  double flops_syrk_exec;
  double flops_scale_exec;
  double apply_bytes_alg; /* packed F~ + index/vector traffic per apply */
  double apply_bytes_exec;
  double factor_bytes;    /* host->device factor values per assemble   */
  int64_t bytes_persistent;
  int64_t bytes_temporary;
  int64_t n_subdomains;
  int64_t n_multipliers;
  int32_t launches_assemble; /* kernel launches of the last assemble */
  int32_t launches_apply;    /* kernel launches per apply             */
  double ms_factorize;       /* device time of the last feti_factorize  */
  double ms_correct;         /* sparse-factor route: rank-2r update of F~ */
  double flops_factor_exec;  /* sparse-factor route: tile flops executed by feti_factorize */
  int32_t launches_factorize;
  int32_t pad_;
  double ms_preprocess;      /* sparse-factor route: factorize start -> assemble end (device) */
  double flops_factor_alg;   /* sparse-factor route: scalar Cholesky flops of K_s in the chosen ordering
                                (sum_j c_j (c_j + 3) from the exact column counts, + the y = L^-1 P Q solve) */
  double ms_pcpg;            /* device time of the last feti_pcpg_solve iteration loop */
  int64_t pcpg_iterations;   /* its iteration count */
} feti_stats;

int feti_abi_version(void);
const char* feti_last_error(void);

/* Create a context on CUDA device `device`. */
int feti_create(int device, feti_ctx** out);
int feti_destroy(feti_ctx* ctx);

/* Register one subdomain (call in the reference's gather order: ascending
 * cluster, then ascending subdomain, dualop.py:375-379).
 *   n, m       local DOFs and local multipliers (rows of B~_i)
 *   first_row  length m: r_j = iperm[dof_j], the factor row of the single
 *              nonzero of B~_i row j (decomposition.py:184-207 gives exactly
 *              one nonzero per row)
 *   sign       length m: the value of that nonzero (+-1)
 *   gids       length m: global multiplier ids (multiplier_ids, ascending)
 *   up, ui     CSR-of-U factor pattern (CholSymbolic.up/ui, sparse.py:240-241);
 *              pass NULL for a dense pattern, i.e. values are LAPACK packed
 *              column-major lower of L = U^T (length n(n+1)/2)
 *   nnz        number of factor values
 *   out_slot   the slot index used by the other calls */
int feti_add_subdomain(feti_ctx* ctx, int64_t n, int64_t m, const int64_t* first_row, const double* sign,
                       const int64_t* gids, const int64_t* up, const int64_t* ui, int64_t nnz,
                       int64_t* out_slot);

/* Choose the strategy before feti_finalize (replaces the branch on
 * config.strategy in DualOperator.preprocess/_apply_local, dualop.py:317-322,
 * 382-388).  Implicit: feti_assemble only prepares the block-scaled factor
 * (no TRSM/SYRK, no F~ memory) and feti_apply/feti_apply_device run the
 * implicit sweeps; feti_local_operator is unavailable (the reference's
 * local_operator returns None, dualop.py:399-401).  On the sparse-factor
 * route the apply adds the rank-2r correction (U2 solved once per assembly). */
int feti_set_strategy(feti_ctx* ctx, int strategy);

/* Choose the explicit assembly's path before feti_finalize (config.path,
 * assemble_explicit_local, dualop.py:470-479): FETI_PATH_SYRK (default)
 * F = X^T X; FETI_PATH_TRSM the second triangular solve Y = L^-T X and the
 * row gather F = B~ Y (spmm_rows), as the reference's "trsm" path -- the
 * same F~ to roundoff, about twice the flops, extra U/Y panels and a
 * transposed copy of the trailing factor tiles. */
int feti_set_path(feti_ctx* ctx, int path);

/* Allocate persistent and temporary device memory; n_multipliers is the
 * global dual-vector length. */
int feti_finalize(feti_ctx* ctx, int64_t n_multipliers);

/* Hand over the numeric factor of one subdomain.
 *   where == FETI_FACTOR_HOST:   async host->device copy (pinned memory
 *                                recommended; keep alive until assemble returns)
 *   where == FETI_FACTOR_DEVICE: `values` is a device pointer used in place */
int feti_set_factor(feti_ctx* ctx, int64_t slot, const double* values, int64_t nnz, int where);

/* Assemble every F~_i on the device (TRSM + SYRK); returns when done. */
int feti_assemble(feti_ctx* ctx);

/* Copy F~_i back: m x m row-major, upper triangle, strictly lower = 0. */
int feti_local_operator(feti_ctx* ctx, int64_t slot, double* out);

/* q = sum_i B~_i^T F~_i B~_i p over this context's subdomains.
 * Host vectors of length n_multipliers; q is overwritten. */
int feti_apply(feti_ctx* ctx, const double* p, double* q);

/* Same on device vectors, enqueued on `stream` (a cudaStream_t used
 * verbatim: NULL is the legacy default stream).  Does not synchronise; the
 * caller orders it after feti_assemble (which returns synchronised).  The
 * other direction is the library's: the next feti_factorize/feti_assemble
 * waits (cudaStreamWaitEvent) for the last apply enqueued on any stream
 * before it rewrites the factor tiles or F~. */
int feti_apply_device(feti_ctx* ctx, const double* d_p, double* d_q, void* stream);

/* Coarse space for a GPU-resident PCPG (solver.py:117-123, 195-272): the
 * projector P x = x - G (G^T G)^-1 G^T x with G = B R block sparse.
 *   kdim        per slot: kernel dimension r_s (1 heat, 3/6 elasticity)
 *   G           per slot, concatenated: m_s x r_s row-major, original local
 *               multiplier order, G_s[a][c] = B~_s[a] R_s[dof_a][c]
 *   coarse_inv  nk x nk row-major (G^T G)^-1, nk = sum r_s                  */
int feti_coarse_setup(feti_ctx* ctx, const int64_t* kdim, const double* G, const double* coarse_inv, int64_t nk);
/* out = P x on device vectors (out may alias x), enqueued on `stream`. */
int feti_project_device(feti_ctx* ctx, const double* d_x, double* d_out, void* stream);
/* out = G (G^T G)^-1 v for v of length nk (feasible start G (G^T G)^-1 e). */
int feti_coarse_apply_device(feti_ctx* ctx, const double* d_v, double* d_out, void* stream);

/* Device-native PCPG (pcpg, solver.py:195-272) on this context's explicit
 * operator (which must own every subdomain) after feti_coarse_setup: the
 * whole iteration -- apply, projections, inner products, the stopping test
 * -- runs on the device (CUDA graph of several iterations, the host polls a
 * status word per graph launch).  d (n_multipliers) and e (nk) host vectors
 * of the dual system (solver.py:125-148); precond 0 = none, 1 = lumped
 * (feti_set_preconditioner); lam (host, n_multipliers) receives the
 * multipliers.  The reference's feasible start, roundoff guard and stopping
 * test (||w_k|| <= tol ||w_0||); maxit <= 0 means n_multipliers.  Returns
 * FETI_ERR_BREAKDOWN / FETI_ERR_NOT_CONVERGED as the reference raises. */
int feti_pcpg_solve(feti_ctx* ctx, const double* d, const double* e, double tol, int64_t maxit, int precond,
                    double* lam, int64_t* iterations, double* rel_residual);

/* Implicit strategy on the device (apply_implicit_local, dualop.py:504-521):
 * q = sum_i B~_i^T K_reg,i^-1 B~_i p through two block triangular sweeps over
 * the scaled factor the last feti_assemble left in HBM (same result as
 * feti_apply to rounding; reads the factor tiles instead of F~). */
int feti_apply_implicit(feti_ctx* ctx, const double* p, double* q);
int feti_apply_implicit_device(feti_ctx* ctx, const double* d_p, double* d_q, void* stream);

/* Device numeric factorization (replaces the host numeric stage,
 * sparse.py:418-424 + regularize sparse.py:427-454): call
 * feti_enable_device_factorization before feti_finalize, then per step
 * feti_set_stiffness for every slot (the UNregularized sparse K as CSR, the
 * orthonormal kernel basis Q (n x r row-major), rho = trace(K)/n and the
 * symbolic ordering perm), feti_factorize, feti_assemble.  K_reg = P (K +
 * rho Q Q^T) P^T is formed and factored on the device; feti_set_factor is not
 * used.  All subdomains must have the same size. */
int feti_enable_device_factorization(feti_ctx* ctx);
int feti_set_stiffness(feti_ctx* ctx, int64_t slot, int64_t n, const int64_t* indptr, const int64_t* indices,
                       const double* data, int64_t nnz, const double* Q, int64_t r, double rho,
                       const int64_t* perm);
int feti_factorize(feti_ctx* ctx);

/* Sparse-factor route (SURVEY.md §7 hard part 4): the reference's dense
 * K_reg is never formed.  K_s = K + rho E E^T (E = r fixing DOFs, E^T Q
 * nonsingular) keeps K's pattern and is factored on the device into a
 * block-sparse pool of 128x128 tiles; F~_i is recovered exactly by the
 * rank-2r correction F~ = B K_s^-1 B^T - U1 U2^T - U2 U1^T + U1 (Q^T W + I/rho)
 * U1^T (W = K_s^-1 Q, U1 = B~ Q, U2 = B~ W), which feti_assemble applies.
 * Replaces regularize (sparse.py:427-454) + symbolic_factorize
 * (sparse.py:340-415) + numeric_factorize (sparse.py:418-424) for
 * assemble_explicit_local (dualop.py:427-501).
 * Call feti_enable_sparse_factorization and, per slot, feti_set_sparse_pattern
 * (K's CSR pattern, the ordering -- constrained DOFs last -- and the fixing
 * DOFs) before feti_finalize; then per step feti_set_stiffness (values, Q,
 * same ordering; rho = trace(K)/n, sparse.py:450, is computed on the device
 * in this mode and the argument is ignored) -- or, after the first step,
 * the batched feti_set_stiffness_values -- then feti_factorize,
 * feti_assemble.  In this mode the K values are copied asynchronously
 * (overlapping the zeroing of the tile pool): keep `data` alive and
 * unchanged until feti_assemble returns.
 * The implicit apply is not available in this mode. */
int feti_enable_sparse_factorization(feti_ctx* ctx);
int feti_set_sparse_pattern(feti_ctx* ctx, int64_t slot, int64_t n, const int64_t* indptr, const int64_t* indices,
                            const int64_t* perm, int64_t r, const int64_t* fix_dofs);
/* Per-step numeric hand-over of the sparse route over a frozen pattern (the
 * refill of CholFactor over its symbolic stage, sparse.py:287-299, without
 * re-validating the pattern): for each listed slot, nnz[i] values of K in
 * the CSR order of its first feti_set_stiffness, and Q[i] its n x r kernel
 * basis or NULL when unchanged (Q may itself be NULL: all unchanged).
 * Copies are queued asynchronously; keep the buffers alive until
 * feti_assemble returns. */
int feti_set_stiffness_values(feti_ctx* ctx, int64_t nslots, const int64_t* slots, const double* const* data,
                              const int64_t* nnz, const double* const* Q);
/* Device dual right-hand side of the sparse route (replaces the solve_local
 * calls of assemble_dual_system, solver.py:141-143, for d = B~ K_reg^-1 f - c):
 * feti_enable_dual_rhs before feti_finalize appends a force row to every
 * slot's (P Q)^T block row; per step feti_set_forces hands over
 * f' = (I - Q Q^T) f (n) and Q^T f (r) per slot before feti_factorize (same
 * asynchronous rules as the stiffness values); after feti_assemble,
 * feti_dual_rhs writes d = sum_i B~_i K_reg,i^-1 f_i - c (c may be NULL) to
 * the host.  With K_reg^-1 = Pi K_s^-1 Pi + rho^-1 Q Q^T:
 * B~ K_reg^-1 f = X^T y_f - U1 (y^T y_f) + rho^-1 U1 Q^T f, y_f = L^-1 P f'. */
int feti_enable_dual_rhs(feti_ctx* ctx);
int feti_set_forces(feti_ctx* ctx, int64_t nslots, const int64_t* slots, const double* const* fproj,
                    const double* const* qtf);
int feti_dual_rhs(feti_ctx* ctx, const double* c, double* d);
/* x = K_reg^-1 b for the listed slots (host vectors concatenated in list
 * order), through the device factor (CholFactor.solve, sparse.py:324-337):
 * the dense device factor, or the sparse route's block-sparse factor of
 * K_s = K + rho E E^T (K_reg^-1 = Pi K_s^-1 Pi + rho^-1 Q Q^T, one CTA per
 * right-hand side; needs an assembled context, repeated slots allowed). */
int feti_solve_many(feti_ctx* ctx, int64_t nslots, const int64_t* slots, const double* b, double* x);

/* Lumped preconditioner (make_preconditioner("lumped"), solver.py:155-175):
 * M w = sum_i B~_i K_i B~_i^T w.  P is P_i = B~_i K_i B~_i^T as an m x m
 * row-major (full, symmetric) array in the slot's original multiplier order;
 * it is stored in the apply's packed tile layout and applied by the same
 * fused gather/SYMV/scatter kernels (deterministic, like feti_apply). */
int feti_set_preconditioner(feti_ctx* ctx, int64_t slot, const double* P);
int feti_precond_apply(feti_ctx* ctx, const double* w, double* out);
int feti_precond_apply_device(feti_ctx* ctx, const double* d_w, double* d_out, void* stream);

/* Multi-GPU apply with the exchange fused into the reduction (one process
 * per GPU, this context = this rank's cluster, decomposition.py:227-243).
 * The reduction kernel stores its per-multiplier sums straight into every
 * rank's receive slab over NVLink (CUDA IPC peer memory) and publishes an
 * epoch flag; a second kernel waits for all ranks and sums the slabs in rank
 * order, so q is identical on every rank and deterministic.  Replaces the
 * apply + all-reduce pair.  Setup: feti_exchange_setup returns this rank's
 * IPC handle (FETI_IPC_HANDLE_BYTES), the caller all-gathers the handles
 * (rank order) and passes them to feti_exchange_connect.  Every rank must
 * issue the same number of exchange applies; a rank that waits ~10 s for a
 * peer gives up, writes NaN into q (never stale values) and sets a sticky
 * error that feti_exchange_status reports (FETI_ERR_CUDA): the context's
 * exchange is unusable after that.  Successive calls may use different
 * streams: each call waits for the previous call's sum (slab reuse). */
#define FETI_IPC_HANDLE_BYTES 64
int feti_exchange_setup(feti_ctx* ctx, int rank, int world, char* handle_out);
int feti_exchange_connect(feti_ctx* ctx, const char* handles);
int feti_apply_exchange_device(feti_ctx* ctx, const double* d_p, double* d_q, void* stream);
int feti_exchange_status(feti_ctx* ctx);

int feti_get_stats(feti_ctx* ctx, feti_stats* out);

/* Diagnostics: per-kernel register / thread limits as text. */
int feti_debug_kernel_attributes(char* buf, int len);

/* Pinned host memory for factor staging. */
int feti_host_alloc(size_t bytes, void** out);
int feti_host_free(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* FETI_B200_H */

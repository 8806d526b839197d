// Sparse-factor route: block-sparse device Cholesky of K_s = K + rho E E^T
// plus the rank-2r correction that recovers the reference's F~ (see
// feti_sparse.cu and paper_2502_08382_b200/sparse_route.py).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "feti_common.cuh"

namespace feti {

// Per-subdomain data of the block-sparse factor (device pointers).
struct SpSub {
  double* pool;             // every stored 128x128 tile of the subdomain
  const int* tmap;          // Tq x Tq: tile (K, L) -> slot in pool, -1 if structurally zero
  const int64_t* perm;      // permuted position -> original DOF
  const int64_t* iperm;     // original DOF -> permuted position
  const int64_t* kptr;      // K (unregularized) CSR, original numbering
  const int64_t* kind;
  const double* kdata;
  const double* Q;          // n x r kernel basis, row-major
  const int64_t* kdiag;     // n: position of K's diagonal entry of each row in kdata
  const int64_t* fix;       // fixing DOFs (original numbering), nfix = r
  const double* U1;         // P*128 x r: sign_a * Q[dof_a], sorted column order
  double* U2W;              // P*128 x 2r: U2 = X^T y_b, then W = C U1 - U2
  double* rho;              // device scalar: trace(K) / n (sparse.py:450), written by sp_trace_kernel
  const double* fproj;      // n: f' = (I - Q Q^T) f, factored along as row `frow` of the (P Q)^T block row
  const double* qtf;        // r: Q^T f
  double* U2f;              // P*128: X^T y_f = B~ K_s^-1 f' (sorted column order)
  int frow;                 // -1, or the block-row-T row holding f' (= r)
  int T;                    // block rows of K_s (the Q block row is T when r > 0)
  int Tq;                   // T + (r > 0)
  int n, r, nfix;           // n: DOFs (rows of K)
  int npos;                 // positions (>= n; perm[p] = -1 marks a padding position)
};

// One tile of the left-looking factorization:
//   accumulate (flags 0):  C -= sum_p A_p B_p^T
//   panel      (flags 1):  C  = C B^T  (B = inv(L_jj), one pair (C, B))
//   flags & 2: C is a tile of the (P Q)^T block row (rows >= 8 are zero)
// one 32-deep k-slice of a tile product: A and B point at the slice (tiles
// are stored k-slice major, SLICE doubles per slice); k-slices where either
// operand is structurally zero in the scalar factor are not listed
struct SpPair {
  const double* A;
  const double* B;
};
struct SpTask {
  double* C;
  int64_t pair0;
  int npairs;     // k-slices (SpPair entries) of this task
  int flags;
};
struct SpDiag {
  double* C;       // tile (j, j): A_jj in, L_jj out
  double* D;       // inv(L_jj) scratch
  int sub;
  int rowbase;     // j * 128 (for the pivot report)
};
struct SpInit {
  double* tile;
  int K, L, sub, pad_;
};

// Host-side block symbolic factorization of one subdomain (the sparse
// analogue of symbolic_factorize, sparse.py:340-415, at 128-row tiles).
struct SpPlan {
  int T = 0, Tq = 0, smin = 0;
  int64_t ntiles = 0;                 // tiles in the pool
  int64_t trail_base = 0;             // slot of tile (smin, smin); the
                                      // trailing triangle follows in tri_index order
  std::vector<int> tmap;              // Tq x Tq -> slot or -1
  // per block column j in [0, Tq): accumulation targets (C slot, (A, B) slot pairs)
  std::vector<std::vector<std::pair<int, std::vector<std::pair<int, int>>>>> acc;
  std::vector<std::vector<int>> panel;  // per column j < T: slots of L_ij, i in struct(j)
  // per slot: bit s set when the tile's k-slice s (columns [32 s, 32 s + 32)
  // of its block column) holds a nonzero of the scalar factor in the tile's
  // rows (the (P Q)^T row: all slices).  A product's slice s is needed only
  // when both operands have bit s: the others add exact zeros.
  std::vector<uint8_t> slot_mask;
  double flops_exec = 0.0;            // tile flops the factorization executes
  double flops_scalar = 0.0;          // scalar Cholesky flops of K_s in this ordering (+ the y = L^-1 P Q solve)
  int64_t nnz_l = 0;                  // nonzeros of the scalar factor
};
// indptr/indices: symmetric pattern of K (original numbering); iperm: DOF ->
// position; r: kernel dimension (adds the (P Q)^T block row T when > 0);
// smin: first block row of the dense trailing triangle.
// n DOFs (rows of K); positions live in [0, npos) (npos >= n: tile-aligned
// orderings leave padding positions, which hold identity rows)
// extra_row: keep the appended block row T even when r = 0 (it then carries
// only the force row of the device dual right-hand side)
void sp_symbolic(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* iperm, int64_t npos,
                 int r, int smin, SpPlan* out, bool extra_row = false);

cudaError_t configure_sparse();
void launch_sp_init(const SpInit* w, int nw, const SpSub* ss, cudaStream_t st);
void launch_sp_scatter(const SpSub* ss, int sub0, int nsub, int max_n, cudaStream_t st);
// rho = trace(K) / n per subdomain on the device (fixed-order reduction)
void launch_sp_trace(const SpSub* ss, int nsub, cudaStream_t st);
void launch_sp_gemm(const SpTask* tasks, int ntasks, const SpPair* pairs, cudaStream_t st);
void launch_sp_potrf(const SpDiag* d, int nd, int* bad, cudaStream_t st);
// d[g] = sum over (sub, a) contributions of B~ K_reg^-1 f, minus c[g]
// (assemble_dual_system, solver.py:141-143), from U2f, U1, y^T y_f, rho, Q^T f
void launch_sp_dual_rhs(const SpSub* ss, int n_mult, const int* cptr, const int4* cent, const double* c, double* d,
                        cudaStream_t st);
// U2/W (and U2f) per (sub, panel) from the X panels
// max_cols >= every panel's subdomain's r (+ 1 with the device dual rhs)
void launch_sp_u2(const SubDev* subs, const SpSub* ss, const int2* panels, int npanels, int max_cols,
                  cudaStream_t st);
// after the assembly: U2/W per (sub, panel), then the rank-2r update of F~
void launch_sp_correct(const SubDev* subs, const SpSub* ss, const int2* panels, int npanels, int sub0, int nsub,
                       int max_T32, int max_cols, cudaStream_t st);

// device solve_local (feti_spsolve.cu): one right-hand side per item, b/x at
// `off` (n values), scratch at `scr` (3 x T*128 values)
struct SpSolveItem {
  int sub, pad_;
  int64_t off, scr;
};
size_t sp_solve_smem();
cudaError_t configure_sp_solve();
void launch_sp_solve(const SubDev* subs, const SpSub* ss, const SpSolveItem* items, int nitems, const double* b,
                     double* x, double* scratch, cudaStream_t st);

}  // namespace feti

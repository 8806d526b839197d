/*
 * CPU oracle kernels -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's numba inner loops on the explicit
 * dual-operator path (pkg/src/tfeti/_kernels.py).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl
 * reference leg may load this library, and only as the checker or the CPU
 * baseline; the product path never does.
 *
 * Each function cites the reference function it restates.  int64 indices and
 * float64 values throughout, row-major (C order) dense blocks.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* _kernels.py:23-42 etree */
void ora_etree(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* parent) {
  int64_t* ancestor = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  for (int64_t i = 0; i < n; ++i) parent[i] = -1, ancestor[i] = -1;
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t p = indptr[k]; p < indptr[k + 1]; ++p) {
      int64_t i = indices[p];
      while (i != -1 && i < k) {
        int64_t inext = ancestor[i];
        ancestor[i] = k;
        if (inext == -1) parent[i] = k;
        i = inext;
      }
    }
  }
  free(ancestor);
}

/* _kernels.py:45-66 factor_row_counts (counts has length n+1, counts[0]=0) */
void ora_factor_row_counts(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* parent,
                           int64_t* counts) {
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  for (int64_t i = 0; i < n; ++i) mark[i] = -1;
  counts[0] = 0;
  for (int64_t k = 0; k < n; ++k) {
    mark[k] = k;
    int64_t cnt = 0;
    for (int64_t p = indptr[k]; p < indptr[k + 1]; ++p) {
      int64_t i = indices[p];
      if (i >= k) continue;
      while (mark[i] != k) {
        mark[i] = k;
        ++cnt;
        i = parent[i];
      }
    }
    counts[k + 1] = cnt;
  }
  free(mark);
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* _kernels.py:69-86 factor_row_pattern */
void ora_factor_row_pattern(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* parent,
                            const int64_t* rowptr, int64_t* rowind) {
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  for (int64_t i = 0; i < n; ++i) mark[i] = -1;
  for (int64_t k = 0; k < n; ++k) {
    mark[k] = k;
    int64_t nxt = rowptr[k];
    for (int64_t p = indptr[k]; p < indptr[k + 1]; ++p) {
      int64_t i = indices[p];
      if (i >= k) continue;
      while (mark[i] != k) {
        mark[i] = k;
        rowind[nxt++] = i;
        i = parent[i];
      }
    }
    qsort(rowind + rowptr[k], (size_t)(rowptr[k + 1] - rowptr[k]), sizeof(int64_t), cmp_i64);
  }
  free(mark);
}

/* _kernels.py:89-104 factor_column_pattern */
void ora_factor_column_pattern(int64_t n, const int64_t* rowptr, const int64_t* rowind, const int64_t* colptr,
                               int64_t* colind) {
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  memcpy(fill, colptr, sizeof(int64_t) * n);
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t q = rowptr[k]; q < rowptr[k + 1]; ++q) {
      int64_t j = rowind[q];
      colind[fill[j]++] = k;
    }
    colind[fill[k]++] = k;
  }
  free(fill);
}

/* _kernels.py:107-140 chol_numeric: up-looking Cholesky; returns -1 or the bad row */
int64_t ora_chol_numeric(int64_t n, const int64_t* aptr, const int64_t* aind, const int64_t* asrc,
                         const double* avals, const int64_t* rowptr, const int64_t* rowind, const int64_t* up,
                         const int64_t* ui, double* ux) {
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  double* x = (double*)calloc((size_t)(n ? n : 1), sizeof(double));
  memcpy(fill, up, sizeof(int64_t) * n);
  int64_t bad = -1;
  for (int64_t k = 0; k < n; ++k) {
    double d = 0.0;
    for (int64_t p = aptr[k]; p < aptr[k + 1]; ++p) {
      int64_t j = aind[p];
      double v = avals[asrc[p]];
      if (j == k)
        d = v;
      else
        x[j] = v;
    }
    for (int64_t q = rowptr[k]; q < rowptr[k + 1]; ++q) {
      int64_t j = rowind[q];
      double lkj = x[j] / ux[up[j]];
      x[j] = 0.0;
      for (int64_t p = up[j] + 1; p < fill[j]; ++p) x[ui[p]] -= ux[p] * lkj;
      d -= lkj * lkj;
      ux[fill[j]] = lkj;
      fill[j] += 1;
    }
    if (d <= 0.0) {
      bad = k;
      break;
    }
    ux[fill[k]] = sqrt(d);
    fill[k] += 1;
  }
  free(fill);
  free(x);
  return bad;
}

/* _kernels.py:168-181 utsolve_rows: U^T X = B in place, X row-major n x k */
void ora_utsolve_rows(int64_t n, int64_t k, const int64_t* up, const int64_t* ui, const double* ux, double* X) {
  for (int64_t j = 0; j < n; ++j) {
    const double d = ux[up[j]];
    double* xj = X + j * k;
    for (int64_t c = 0; c < k; ++c) xj[c] /= d;
    for (int64_t p = up[j] + 1; p < up[j + 1]; ++p) {
      double* xi = X + ui[p] * k;
      const double v = ux[p];
      for (int64_t c = 0; c < k; ++c) xi[c] -= v * xj[c];
    }
  }
}

/* _kernels.py:152-165 usolve_rows: U X = B in place */
void ora_usolve_rows(int64_t n, int64_t k, const int64_t* up, const int64_t* ui, const double* ux, double* X) {
  for (int64_t i = n - 1; i >= 0; --i) {
    double* xi = X + i * k;
    for (int64_t p = up[i] + 1; p < up[i + 1]; ++p) {
      const double* xj = X + ui[p] * k;
      const double v = ux[p];
      for (int64_t c = 0; c < k; ++c) xi[c] -= v * xj[c];
    }
    const double d = ux[up[i]];
    for (int64_t c = 0; c < k; ++c) xi[c] /= d;
  }
}

/* _kernels.py:222-229 spmv_rows */
void ora_spmv_rows(int64_t rows, const int64_t* indptr, const int64_t* indices, const double* data, const double* x,
                   double* out) {
  for (int64_t i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) acc += data[p] * x[indices[p]];
    out[i] = acc;
  }
}

/* _kernels.py:232-239 spmv_rows_t (out has length cols) */
void ora_spmv_rows_t(int64_t rows, int64_t cols, const int64_t* indptr, const int64_t* indices, const double* data,
                     const double* x, double* out) {
  for (int64_t c = 0; c < cols; ++c) out[c] = 0.0;
  for (int64_t i = 0; i < rows; ++i) {
    const double xi = x[i];
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) out[indices[p]] += data[p] * xi;
  }
}

/* _kernels.py:274-287 symv_upper: out = F x reading the upper triangle of row-major F */
void ora_symv_upper(int64_t n, const double* F, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = F[i * n + i] * x[i];
  for (int64_t i = 0; i < n; ++i) {
    const double xi = x[i];
    double acc = 0.0;
    for (int64_t j = i + 1; j < n; ++j) {
      const double f = F[i * n + j];
      acc += f * x[j];
      out[j] += f * xi;
    }
    out[i] += acc;
  }
}

/* _kernels.py:290-296 zero_lower */
void ora_zero_lower(int64_t n, double* F) {
  for (int64_t i = 1; i < n; ++i)
    for (int64_t j = 0; j < i; ++j) F[i * n + j] = 0.0;
}

/* _kernels.py:299-305 densify_transposed: Z (rows_of_bt x cols) = B^T, row-major */
void ora_densify_transposed(int64_t brows, int64_t zcols, int64_t zrows, const int64_t* bptr, const int64_t* bind,
                            const double* bval, double* Z) {
  memset(Z, 0, sizeof(double) * (size_t)(zrows * zcols));
  for (int64_t r = 0; r < brows; ++r)
    for (int64_t p = bptr[r]; p < bptr[r + 1]; ++p) Z[bind[p] * zcols + r] = bval[p];
}

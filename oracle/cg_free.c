/* TEST INFRASTRUCTURE (oracle), not product code.
 *
 * CPU conjugate gradients on A_free for the configs[4] oracle:
 * the reference factors A_free densely (dynamics.py:413-414, linalg.py:23-40,
 * cho_factor / cho_solve), which is infeasible at 12 M dofs, so the oracle
 * replaces only `sysfact.solve` (linalg.py:57-59, used by solvers.py:116,134)
 * with Jacobi-preconditioned CG run to a relative residual far tighter than the
 * GPU's 1e-10 (1e-13 by default), so that the oracle's own solve error does not
 * confound the comparison.  Every other step of the frame stays the reference's
 * (oracle/qnsim_oracle.py).
 *
 * The three coordinates are three independent CG runs over the same matrix
 * (A is the same scalar matrix for x, y and z); they run in lockstep so each
 * matrix entry is loaded once per iteration, and each column stops at
 * ||r_c||_2 <= tol ||b_c||_2 (the GPU's criterion, qn_solver.cu k_pcg_update).
 * Reductions are chunked in a fixed order (chunk partials summed
 * sequentially), so results do not depend on the thread count.
 *
 *   gcc -O3 -fopenmp -fPIC -shared -o oracle/_build/libcg_free.so oracle/cg_free.c
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CHUNK 65536

static void spmv3(int64_t n, const int64_t* ptr, const int32_t* idx, const double* val, const double* x,
                  double* y) {
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      const double v = val[k];
      const double* xr = x + 3 * (int64_t)idx[k];
      a += v * xr[0];
      b += v * xr[1];
      c += v * xr[2];
    }
    y[3 * i] = a;
    y[3 * i + 1] = b;
    y[3 * i + 2] = c;
  }
}

/* out[c] = sum_i u[3i+c] v[3i+c], fixed chunk order */
static void dot3(int64_t n, const double* u, const double* v, double* out) {
  const int64_t nch = (n + CHUNK - 1) / CHUNK;
  double* part = (double*)calloc((size_t)nch * 3, sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int64_t lo = ch * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t i = lo; i < hi; ++i) {
      a += u[3 * i] * v[3 * i];
      b += u[3 * i + 1] * v[3 * i + 1];
      c += u[3 * i + 2] * v[3 * i + 2];
    }
    part[3 * ch] = a;
    part[3 * ch + 1] = b;
    part[3 * ch + 2] = c;
  }
  out[0] = out[1] = out[2] = 0.0;
  for (int64_t ch = 0; ch < nch; ++ch)
    for (int c = 0; c < 3; ++c) out[c] += part[3 * ch + c];
  free(part);
}

/* Solve A X = B for B, X of shape (n, 3) row-major; X starts at zero.
 * iters[c] = CG iterations of column c, relres[c] = final true relative
 * residual ||b - A x|| / ||b||.  Returns 0, or 1 if a column hit maxit. */
int oracle_cg3(int64_t n, const int64_t* ptr, const int32_t* idx, const double* val, const double* B, double* X,
               double tol, int32_t maxit, int32_t* iters, double* relres) {
  double* dinv = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * 3 * n);
  double* z = (double*)malloc(sizeof(double) * 3 * n);
  double* p = (double*)malloc(sizeof(double) * 3 * n);
  double* q = (double*)malloc(sizeof(double) * 3 * n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double d = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
      if (idx[k] == i) d = val[k];
    dinv[i] = 1.0 / d;
  }
  memset(X, 0, sizeof(double) * 3 * n);
  memcpy(r, B, sizeof(double) * 3 * n);
  double bb[3], rz[3], rr[3], pq[3];
  int done[3] = {0, 0, 0};
  dot3(n, B, B, bb);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < 3 * n; ++i) {
    z[i] = dinv[i / 3] * r[i];
    p[i] = z[i];
  }
  dot3(n, r, z, rz);
  for (int c = 0; c < 3; ++c) {
    iters[c] = 0;
    if (bb[c] == 0.0) done[c] = 1;
  }
  int it = 0;
  while (!(done[0] && done[1] && done[2]) && it < maxit) {
    ++it;
    spmv3(n, ptr, idx, val, p, q);
    dot3(n, p, q, pq);
    double al[3];
    for (int c = 0; c < 3; ++c) al[c] = done[c] ? 0.0 : rz[c] / pq[c];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) {
        X[3 * i + c] += al[c] * p[3 * i + c];
        r[3 * i + c] -= al[c] * q[3 * i + c];
      }
    dot3(n, r, r, rr);
    for (int c = 0; c < 3; ++c)
      if (!done[c]) {
        iters[c] = it;
        if (rr[c] <= tol * tol * bb[c]) done[c] = 1;
      }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < 3 * n; ++i) z[i] = dinv[i / 3] * r[i];
    double rzn[3], be[3];
    dot3(n, r, z, rzn);
    for (int c = 0; c < 3; ++c) {
      be[c] = done[c] ? 0.0 : rzn[c] / rz[c];
      rz[c] = rzn[c];
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c)
        if (!done[c]) p[3 * i + c] = z[3 * i + c] + be[c] * p[3 * i + c];
  }
  /* true residual */
  spmv3(n, ptr, idx, val, X, q);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < 3 * n; ++i) r[i] = B[i] - q[i];
  dot3(n, r, r, rr);
  for (int c = 0; c < 3; ++c) relres[c] = bb[c] > 0.0 ? sqrt(rr[c] / bb[c]) : 0.0;
  free(dinv);
  free(r);
  free(z);
  free(p);
  free(q);
  return (done[0] && done[1] && done[2]) ? 0 : 1;
}

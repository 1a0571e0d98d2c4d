// Host-only check of the supernodal factor data structures (TEST ONLY).
// Builds libqnsim_b200's host factorisation (qn_factor.cpp) and replays the
// device solve algorithm of qn_sptrsv.cuh sequentially on the CPU, so the
// ordering / symbolic / numeric / relative-index logic is verified in the
// GPU-less build container.  Not linked into the product library.
#include <cstring>
#include <string>
#include <vector>

#include "qn_factor.h"

namespace qn {
static std::string g_err;
void set_error(const std::string& m) { g_err = m; }
const char* get_error() { return g_err.c_str(); }
void count_launch(int) {}
}  // namespace qn

extern "C" {
const char* hc_last_error() { return qn::get_error(); }

// X = A^-1 B (B: n x 3) for batch instance `b`; returns QN_* code.
int hc_factor_solve(int64_t n, const int64_t* indptr, const int32_t* indices, const double* values, int64_t nbatch,
                    const double* coords, int64_t b, const double* B, double* X, int64_t* stats) {
  qn_factor f;
  int rc = qn::factor_build_host(&f, n, indptr, indices, values, nbatch, coords);
  if (rc) return rc;
  const double* vals = f.vals.data() + (size_t)b * f.nvals;
  std::vector<double> y(n * 3), x(n * 3), u(std::max<int64_t>(f.nupd, 1) * 3);
  for (int s = 0; s < f.nsup; ++s) {
    const int c0 = f.sup_col[s], nc = f.sup_col[s + 1] - c0;
    const int64_t r0 = f.sup_row_ptr[s];
    const int nr = (int)(f.sup_row_ptr[s + 1] - r0), mb = nr - nc;
    std::vector<double> acc(nr * 3, 0.0), ys(nc * 3);
    for (int q = f.child_ptr[s]; q < f.child_ptr[s + 1]; ++q) {
      const int c = f.child_idx[q];
      const int mc = (int)(f.rel_ptr[c + 1] - f.rel_ptr[c]);
      for (int i = 0; i < mc; ++i)
        for (int a = 0; a < 3; ++a) acc[3 * f.rel[f.rel_ptr[c] + i] + a] += u[(f.sup_upd_ptr[c] + i) * 3 + a];
    }
    for (int i = 0; i < nc; ++i)
      for (int a = 0; a < 3; ++a) acc[3 * i + a] = B[3 * f.perm[c0 + i] + a] - acc[3 * i + a];
    const double* Xv = vals + f.sup_val_ptr[s];
    for (int i = 0; i < nc; ++i)
      for (int a = 0; a < 3; ++a) {
        double v = 0;
        for (int k = 0; k <= i; ++k) v += Xv[i + k * nc] * acc[3 * k + a];
        ys[3 * i + a] = v;
        y[3 * (c0 + i) + a] = v;
      }
    if (mb > 0 && f.parent[s] >= 0) {
      const double* Lb = Xv + nc * nc;
      for (int r = 0; r < mb; ++r)
        for (int a = 0; a < 3; ++a) {
          double v = acc[3 * (nc + r) + a];
          for (int k = 0; k < nc; ++k) v += Lb[r + k * mb] * ys[3 * k + a];
          u[(f.sup_upd_ptr[s] + r) * 3 + a] = v;
        }
    }
  }
  for (int s = f.nsup - 1; s >= 0; --s) {
    const int c0 = f.sup_col[s], nc = f.sup_col[s + 1] - c0;
    const int64_t r0 = f.sup_row_ptr[s];
    const int nr = (int)(f.sup_row_ptr[s + 1] - r0), mb = nr - nc;
    const double* Xv = vals + f.sup_val_ptr[s];
    const double* Lb = Xv + nc * nc;
    std::vector<double> t(nc * 3);
    for (int k = 0; k < nc; ++k)
      for (int a = 0; a < 3; ++a) {
        double v = 0;
        for (int r = 0; r < mb; ++r) v += Lb[r + k * mb] * x[3 * f.sup_rows[r0 + nc + r] + a];
        t[3 * k + a] = y[3 * (c0 + k) + a] - v;
      }
    for (int k = 0; k < nc; ++k)
      for (int a = 0; a < 3; ++a) {
        double v = 0;
        for (int i = k; i < nc; ++i) v += Xv[i + k * nc] * t[3 * i + a];
        x[3 * (c0 + k) + a] = v;
        X[3 * f.perm[c0 + k] + a] = v;
      }
  }
  if (stats) {
    stats[0] = f.nsup;
    stats[1] = f.nnz_l;
    stats[2] = f.depth;
    stats[3] = f.max_rows;
  }
  return 0;
}
}

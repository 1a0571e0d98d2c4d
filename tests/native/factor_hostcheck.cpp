// Host-only check of the supernodal factor data structures (TEST ONLY).
// Builds libqnsim_b200's host factorisation (qn_factor.cpp) and replays the
// device solve algorithm of qn_sptrsv.cuh sequentially on the CPU (Z blocks,
// pull-style extend-add lists, task decomposition), so the ordering /
// symbolic / numeric / task logic is verified in the GPU-less build
// container.  Not linked into the product library.
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
// stats: nsup, nnz_l, depth, max_rows, n_forward_tasks, n_backward_tasks
int hc_factor_solve(int64_t n, const int64_t* indptr, const int32_t* indices, const double* values, int64_t nbatch,
                    const double* coords, int64_t b, const double* B, double* X, int64_t* stats) {
  qn_factor f;
  int rc = qn::factor_build_host(&f, n, indptr, indices, values, nbatch, coords);
  if (rc) return rc;
  const double* vals = f.vals.data() + (size_t)b * f.nvals;
  std::vector<double> y(n * 3), x(n * 3), u(std::max<int64_t>(f.nupd, 1) * 3);
  std::vector<int> done_f(f.nsup, 0), done_b(f.nsup, 0);
  // forward tasks in ticket order; every dependency must already be complete
  // forward descriptors / relative lists must describe exactly the cptr/cidx structure
  if (f.fdesc.size() != f.ftask.size()) return 93;
  for (size_t i = 0; i < f.ftask.size(); ++i) {
    const int4& t = f.ftask[i];
    const qn_fdesc& d = f.fdesc[i];
    const int s = t.x;
    const int64_t R0 = f.sup_row_ptr[s];
    const int nc = f.sup_col[s + 1] - f.sup_col[s];
    if (d.lo != t.y || d.hi != t.z || d.nc != nc || d.c0 != f.sup_col[s] || d.zoff != f.sup_val_ptr[s] + t.y ||
        d.upd0 != f.sup_upd_ptr[s] || d.dep0 != f.fdep_ptr[s] || d.dep1 != f.fdep_ptr[s + 1])
      return 93;
    const int32_t* sp_top = f.fblob.data() + d.blob;
    const int nptr_bot = d.blo < d.hi ? d.hi - d.blo + 1 : 0;
    const int32_t* sp_bot = sp_top + nc + 1;
    const int32_t* si_top = sp_bot + nptr_bot;
    const int32_t* si_bot = si_top + d.ntop;
    for (int p = 0; p < nc; ++p)
      for (int q = sp_top[p]; q < sp_top[p + 1]; ++q)
        if (si_top[q] != f.cidx[f.cptr[R0 + p] + (q - sp_top[p])]) return 93;
    for (int r = d.blo; r < d.hi; ++r)
      for (int q = sp_bot[r - d.blo]; q < sp_bot[r - d.blo + 1]; ++q)
        if (si_bot[q] != f.cidx[f.cptr[R0 + r] + (q - sp_bot[r - d.blo])]) return 93;
  }
  if (f.bdesc.size() != f.btask.size()) return 92;
  for (size_t i = 0; i < f.btask.size(); ++i) {
    const int4& t = f.btask[i];
    const qn_bdesc& d = f.bdesc[i];
    const int s = t.x, p = f.parent[s];
    const int nr = (int)(f.sup_row_ptr[s + 1] - f.sup_row_ptr[s]);
    if (d.k0 != t.y || d.k1 != t.z || d.c0 != f.sup_col[s] || d.nr != nr || d.rows != f.sup_row_ptr[s] ||
        d.zoff != f.sup_val_ptr[s] + (int64_t)t.y * nr || d.nwait != (p >= 0 ? f.bcount[p] : 0) ||
        (p >= 0 && d.wait0 != f.bfirst[p]) || d.fwd0 != f.ffirst[s] || d.nfwd != f.fcount[s])
      return 92;
  }
  for (const int4& t : f.ftask) {
    const int s = t.x;
    for (int q = f.child_ptr[s]; q < f.child_ptr[s + 1]; ++q)
      if (done_f[f.child_idx[q]] != f.fcount[f.child_idx[q]]) return 99;
    const int c0 = f.sup_col[s], nc = f.sup_col[s + 1] - c0;
    const int64_t R0 = f.sup_row_ptr[s];
    const int nr = (int)(f.sup_row_ptr[s + 1] - R0);
    std::vector<double> fv(nc * 3);
    for (int p = 0; p < nc; ++p)
      for (int a = 0; a < 3; ++a) {
        double acc = 0;
        for (int64_t q = f.cptr[R0 + p]; q < f.cptr[R0 + p + 1]; ++q) acc += u[3 * f.cidx[q] + a];
        fv[3 * p + a] = B[3 * f.perm[c0 + p] + a] - acc;
      }
    const double* Z = vals + f.sup_val_ptr[s];
    for (int r = t.y; r < t.z; ++r)
      for (int a = 0; a < 3; ++a) {
        double v = 0;
        for (int k = 0; k < nc; ++k) v += Z[r + (int64_t)k * nr] * fv[3 * k + a];
        if (r < nc) {
          y[3 * (c0 + r) + a] = v;
        } else {
          double e = 0;
          for (int64_t q = f.cptr[R0 + r]; q < f.cptr[R0 + r + 1]; ++q) e += u[3 * f.cidx[q] + a];
          u[3 * (f.sup_upd_ptr[s] + r - nc) + a] = e + v;
        }
      }
    done_f[s]++;
  }
  if (f.ktop > 0) {  // dense top: x_T = S^-1 (b_T - updates of the subtrees below T)
    const int K = f.ktop;
    std::vector<double> g(3 * K);
    for (int k = 0; k < K; ++k)
      for (int a = 0; a < 3; ++a) {
        double acc = 0;
        for (int q = f.tg_ptr[k]; q < f.tg_ptr[k + 1]; ++q) acc += u[3 * f.tg_idx[q] + a];
        g[3 * k + a] = B[3 * f.perm[f.tcols[k]] + a] - acc;
      }
    for (int k = 0; k < K; ++k)
      for (int a = 0; a < 3; ++a) {
        double v = 0;
        for (int c = 0; c < K; ++c) v += f.sinv[(size_t)k * K + c] * g[3 * c + a];
        x[3 * f.tcols[k] + a] = v;
        X[3 * f.perm[f.tcols[k]] + a] = v;
      }
  }
  for (const int4& t : f.btask) {
    const int s = t.x;
    if (f.parent[s] >= 0 && done_b[f.parent[s]] != f.bcount[f.parent[s]]) return 98;
    const int c0 = f.sup_col[s], nc = f.sup_col[s + 1] - c0;
    const int64_t R0 = f.sup_row_ptr[s];
    const int nr = (int)(f.sup_row_ptr[s + 1] - R0);
    const double* Z = vals + f.sup_val_ptr[s];
    for (int k = t.y; k < t.z; ++k)
      for (int a = 0; a < 3; ++a) {
        double v = 0;
        for (int r = k; r < nr; ++r) {
          const double w = r < nc ? y[3 * (c0 + r) + a] : -x[3 * f.sup_rows[R0 + r] + a];
          v += Z[r + (int64_t)k * nr] * w;
        }
        x[3 * (c0 + k) + a] = v;
        X[3 * f.perm[c0 + k] + a] = v;
      }
    done_b[s]++;
  }
  if (stats) {
    stats[0] = f.nsup;
    stats[1] = f.nnz_l;
    stats[2] = f.depth;
    stats[3] = f.max_rows;
    stats[4] = (int64_t)f.ftask.size();
    stats[5] = (int64_t)f.btask.size();
    stats[6] = f.ktop;
  }
  return 0;
}
}

// Symbolic structure of the host factor (diagnostics / kernel design):
// sup[s] = {parent, col0, nc, nr, is_top}, sizes[] = {n, nsup, ktop, nvals, n_ftask, n_btask, nnz_l}.
// Call with sup == nullptr first to get nsup.
extern "C" int hc_factor_structure(int64_t n, const int64_t* indptr, const int32_t* indices, const double* values,
                                   const double* coords, int64_t* sizes, int32_t* sup, int64_t cap) {
  qn_factor f;
  const int64_t nbatch = sizes[7] > 0 ? sizes[7] : 1;  // in: instances (values = nbatch x nnz)
  int rc = qn::factor_build_host(&f, n, indptr, indices, values, nbatch, coords);
  if (rc) return rc;
  sizes[0] = f.n;
  sizes[1] = f.nsup;
  sizes[2] = f.ktop;
  sizes[3] = f.nvals;
  sizes[4] = (int64_t)f.ftask.size();
  sizes[5] = (int64_t)f.btask.size();
  sizes[6] = f.nnz_l;
  if (!sup || cap < f.nsup) return 0;
  for (int s = 0; s < f.nsup; ++s) {
    sup[5 * s + 0] = f.parent[s];
    sup[5 * s + 1] = f.sup_col[s];
    sup[5 * s + 2] = f.sup_col[s + 1] - f.sup_col[s];
    sup[5 * s + 3] = (int32_t)(f.sup_row_ptr[s + 1] - f.sup_row_ptr[s]);
    sup[5 * s + 4] = f.is_top.empty() ? 0 : f.is_top[s];
  }
  return 0;
}

// ---- AMG hierarchy (qn_amg.cpp) + host reference PCG (TEST ONLY) ----
#include "qn_amg.h"
extern "C" int hc_amg_solve(int64_t n, const int64_t* indptr, const int32_t* indices, const double* values,
                            const double* B, double* X, double tol, int maxit, int64_t* stats) {
  qn::AmgHierarchy h;
  int rc = qn::amg_build(n, indptr, indices, values, &h);
  if (rc) return rc;
  const int it = qn::amg_pcg_host(h, B, X, tol, maxit);
  stats[0] = it;
  stats[1] = (int64_t)h.lv.size();
  for (size_t l = 0; l < h.lv.size() && l < 6; ++l) stats[2 + l] = h.lv[l].A.n;
  if (stats[8] == -1)  // caller asks for nnz per level too: A, P in stats[9 + 2l], stats[10 + 2l]
    for (size_t l = 0; l < h.lv.size() && l < 6; ++l) {
      stats[9 + 2 * l] = h.lv[l].A.ptr.empty() ? 0 : h.lv[l].A.ptr.back();
      stats[10 + 2 * l] = h.lv[l].P.ptr.empty() ? 0 : h.lv[l].P.ptr.back();
    }
  return 0;
}

// Smoothed-aggregation AMG setup (host) — see qn_amg.h.
//
// Per level: strong connections |a_ij| >= theta sqrt(a_ii a_jj) (for the
// Freudenthal FEM operators this selects the 6 axis neighbours and drops the
// near-zero diagonal-edge couplings), greedy three-phase aggregation, the
// filtered operator A_F (weak entries lumped into the diagonal), the
// prolongator P = (I - w D_F^-1 A_F) P_tent with w = 4 / (3 rho(D_F^-1 A_F)),
// R = P^T and the Galerkin product A_c = R A P.  The coarsest operator
// (<= kAmgCoarsest rows) is inverted densely.
#include "qn_amg.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <numeric>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "qn_common.cuh"

namespace qn {
namespace {

Csr transpose(const Csr& a) {
  Csr t;
  t.n = a.m;
  t.m = a.n;
  t.ptr.assign(t.n + 1, 0);
  for (int64_t e = 0; e < a.ptr[a.n]; ++e) t.ptr[a.col[e] + 1]++;
  for (int64_t i = 0; i < t.n; ++i) t.ptr[i + 1] += t.ptr[i];
  t.col.resize(a.ptr[a.n]);
  t.val.resize(a.ptr[a.n]);
  std::vector<int64_t> fill(t.ptr.begin(), t.ptr.end() - 1);
  for (int64_t i = 0; i < a.n; ++i)  // rows in order -> columns of t sorted
    for (int64_t e = a.ptr[i]; e < a.ptr[i + 1]; ++e) {
      const int64_t w = fill[a.col[e]]++;
      t.col[w] = (int32_t)i;
      t.val[w] = a.val[e];
    }
  return t;
}

// C = A B (row-parallel, dense accumulator per thread, columns sorted)
Csr spgemm(const Csr& a, const Csr& b) {
  Csr c;
  c.n = a.n;
  c.m = b.m;
  c.ptr.assign(c.n + 1, 0);
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  const int64_t chunk = std::max<int64_t>(1, (c.n + nt - 1) / nt);
  std::vector<std::vector<int32_t>> tcol(nt);
  std::vector<std::vector<double>> tval(nt);
  std::vector<std::vector<int64_t>> tcnt(nt);
#pragma omp parallel num_threads(nt)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    const int64_t r0 = std::min<int64_t>(c.n, t * chunk), r1 = std::min<int64_t>(c.n, r0 + chunk);
    std::vector<int64_t> mark(b.m, -1);
    std::vector<double> acc(b.m, 0.0);
    std::vector<int32_t> cols;
    auto& oc = tcol[t];
    auto& ov = tval[t];
    auto& cnt = tcnt[t];
    for (int64_t i = r0; i < r1; ++i) {
      cols.clear();
      for (int64_t e = a.ptr[i]; e < a.ptr[i + 1]; ++e) {
        const int32_t k = a.col[e];
        const double av = a.val[e];
        for (int64_t f = b.ptr[k]; f < b.ptr[k + 1]; ++f) {
          const int32_t j = b.col[f];
          if (mark[j] != i) {
            mark[j] = i;
            acc[j] = 0.0;
            cols.push_back(j);
          }
          acc[j] += av * b.val[f];
        }
      }
      std::sort(cols.begin(), cols.end());
      for (int32_t j : cols) {
        oc.push_back(j);
        ov.push_back(acc[j]);
      }
      cnt.push_back((int64_t)cols.size());
    }
  }
  int64_t w = 0;
  for (int t = 0; t < nt; ++t)
    for (int64_t k = 0; k < (int64_t)tcnt[t].size(); ++k) {
      const int64_t row = t * chunk + k;
      c.ptr[row + 1] = tcnt[t][k];
      w += tcnt[t][k];
    }
  for (int64_t i = 0; i < c.n; ++i) c.ptr[i + 1] += c.ptr[i];
  c.col.reserve(w);
  c.val.reserve(w);
  for (int t = 0; t < nt; ++t) {
    c.col.insert(c.col.end(), tcol[t].begin(), tcol[t].end());
    c.val.insert(c.val.end(), tval[t].begin(), tval[t].end());
  }
  return c;
}

void spmv3(const Csr& a, const double* x, double* y) {  // y = A x, 3 RHS
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < a.n; ++i) {
    double s0 = 0, s1 = 0, s2 = 0;
    for (int64_t e = a.ptr[i]; e < a.ptr[i + 1]; ++e) {
      const double v = a.val[e];
      const double* xj = x + 3 * (size_t)a.col[e];
      s0 += v * xj[0];
      s1 += v * xj[1];
      s2 += v * xj[2];
    }
    y[3 * i + 0] = s0;
    y[3 * i + 1] = s1;
    y[3 * i + 2] = s2;
  }
}

// largest eigenvalue of D^-1 A (power iteration, deterministic start); the
// row loop is parallel and the norms are summed over fixed 64 k-row chunks in
// chunk order, so the result does not depend on the thread count
double rho_dinv_a(const Csr& a, const std::vector<double>& dinv, int its = 15) {
  const int64_t n = a.n;
  constexpr int64_t kChunk = 65536;
  const int64_t nch = (n + kChunk - 1) / kChunk;
  std::vector<double> x(n), y(n), part(2 * nch);
  for (int64_t i = 0; i < n; ++i) x[i] = 1.0 + 0.1 * std::sin(0.7 * (double)i);
  double lam = 1.0;
  for (int k = 0; k < its; ++k) {
#pragma omp parallel for schedule(static)
    for (int64_t ch = 0; ch < nch; ++ch) {
      double ny = 0.0, nx = 0.0;
      for (int64_t i = ch * kChunk; i < std::min(n, (ch + 1) * kChunk); ++i) {
        double s = 0.0;
        for (int64_t e = a.ptr[i]; e < a.ptr[i + 1]; ++e) s += a.val[e] * x[a.col[e]];
        y[i] = dinv[i] * s;
        ny += y[i] * y[i];
        nx += x[i] * x[i];
      }
      part[2 * ch] = ny;
      part[2 * ch + 1] = nx;
    }
    double nrm = 0.0, xn = 0.0;
    for (int64_t ch = 0; ch < nch; ++ch) {
      nrm += part[2 * ch];
      xn += part[2 * ch + 1];
    }
    nrm = std::sqrt(nrm);
    lam = nrm / std::max(std::sqrt(xn), 1e-300);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) x[i] = y[i] / std::max(nrm, 1e-300);
  }
  return lam;
}

}  // namespace

int amg_build(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, AmgHierarchy* h) {
  const auto t0 = std::chrono::steady_clock::now();
  const bool verbose = std::getenv("QN_AMG_VERBOSE") != nullptr;  // diagnostics: per-phase setup times
  auto tp = t0;
  auto phase = [&](const char* what, int lev) {
    if (!verbose) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "amg setup L%d %-12s %8.3f s\n", lev, what, std::chrono::duration<double>(t - tp).count());
    tp = t;
  };
  h->lv.clear();
  h->omega_l.clear();
  AmgLevel L0;
  L0.A.n = L0.A.m = n;
  L0.A.ptr.assign(ptr, ptr + n + 1);
  L0.A.col.assign(col, col + ptr[n]);
  L0.A.val.assign(val, val + ptr[n]);
  h->lv.push_back(std::move(L0));
  for (int lev = 0; lev < kAmgMaxLevels; ++lev) {
    AmgLevel& L = h->lv.back();
    const Csr& A = L.A;
    const int64_t nl = A.n;
    std::vector<double> diag(nl, 0.0);
    for (int64_t i = 0; i < nl; ++i)
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
        if (A.col[e] == i) diag[i] = A.val[e];
    L.dinv.resize(nl);
    for (int64_t i = 0; i < nl; ++i) {
      QN_REQUIRE(diag[i] > 0.0, QN_ERR_NOT_SPD, "amg: non-positive diagonal");
      L.dinv[i] = 1.0 / diag[i];
    }
    h->omega_l.push_back(4.0 / (3.0 * rho_dinv_a(A, L.dinv)));
    phase("diag+rho", lev);
    if (nl <= kAmgCoarsest || lev == kAmgMaxLevels - 1) break;
    // ---- strength + filtered operator ----
    std::vector<uint8_t> strong(A.ptr[nl], 0);
    std::vector<double> fdiag(diag);
    for (int64_t i = 0; i < nl; ++i)
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        const int32_t j = A.col[e];
        if (j == i) continue;
        if (std::fabs(A.val[e]) >= kAmgStrength * std::sqrt(diag[i] * diag[j]))
          strong[e] = 1;
        else
          fdiag[i] += A.val[e];  // lump the weak coupling (row sums preserved)
      }
    phase("strength", lev);
    // ---- greedy aggregation ----
    std::vector<int32_t> agg(nl, -1);
    int32_t na = 0;
    for (int64_t i = 0; i < nl; ++i) {  // phase 1: whole strong neighbourhoods
      if (agg[i] >= 0) continue;
      bool free_nb = true;
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1] && free_nb; ++e)
        if (strong[e] && agg[A.col[e]] >= 0) free_nb = false;
      if (!free_nb) continue;
      agg[i] = na;
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
        if (strong[e]) agg[A.col[e]] = na;
      ++na;
    }
    std::vector<int32_t> agg1(agg);
    for (int64_t i = 0; i < nl; ++i) {  // phase 2: join the strongest aggregated neighbour
      if (agg1[i] >= 0) continue;
      double best = -1.0;
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
        if (strong[e] && agg1[A.col[e]] >= 0 && std::fabs(A.val[e]) > best) {
          best = std::fabs(A.val[e]);
          agg[i] = agg1[A.col[e]];
        }
    }
    for (int64_t i = 0; i < nl; ++i) {  // phase 3: leftovers with their free neighbours
      if (agg[i] >= 0) continue;
      agg[i] = na;
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
        if (strong[e] && agg[A.col[e]] < 0) agg[A.col[e]] = na;
      ++na;
    }
    if (na >= nl || na < 1) break;  // no coarsening possible
    phase("aggregate", lev);
    // ---- smoothed prolongator P = (I - w D_F^-1 A_F) P_tent ----
    Csr Af;
    Af.n = Af.m = nl;
    Af.ptr.assign(nl + 1, 0);
    for (int64_t i = 0; i < nl; ++i) {
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
        if (strong[e] || A.col[e] == i) {
          Af.col.push_back(A.col[e]);
          Af.val.push_back(A.col[e] == i ? fdiag[i] : A.val[e]);
        }
      Af.ptr[i + 1] = (int64_t)Af.col.size();
    }
    std::vector<double> fdinv(nl);
    for (int64_t i = 0; i < nl; ++i) fdinv[i] = fdiag[i] > 0 ? 1.0 / fdiag[i] : L.dinv[i];
    const double wp = 4.0 / (3.0 * rho_dinv_a(Af, fdinv));
    Csr P;
    P.n = nl;
    P.m = na;
    P.ptr.assign(nl + 1, 0);
    {  // rows are independent: per-thread row ranges, concatenated in row order
      int nt = 1;
#ifdef _OPENMP
      nt = omp_get_max_threads();
#endif
      const int64_t chunk = std::max<int64_t>(1, (nl + nt - 1) / nt);
      std::vector<std::vector<int32_t>> tcol(nt);
      std::vector<std::vector<double>> tval(nt);
#pragma omp parallel num_threads(nt)
      {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        std::vector<int32_t> cols;
        std::vector<double> vals;
        for (int64_t i = t * chunk; i < std::min<int64_t>(nl, (t + 1) * chunk); ++i) {
          cols.clear();
          vals.clear();
          auto add = [&](int32_t c, double v) {
            for (size_t k = 0; k < cols.size(); ++k)
              if (cols[k] == c) {
                vals[k] += v;
                return;
              }
            cols.push_back(c);
            vals.push_back(v);
          };
          add(agg[i], 1.0);
          for (int64_t e = Af.ptr[i]; e < Af.ptr[i + 1]; ++e) add(agg[Af.col[e]], -wp * fdinv[i] * Af.val[e]);
          std::vector<int32_t> ord(cols.size());
          std::iota(ord.begin(), ord.end(), 0);
          std::sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return cols[x] < cols[y]; });
          for (int32_t k : ord) {
            tcol[t].push_back(cols[k]);
            tval[t].push_back(vals[k]);
          }
          P.ptr[i + 1] = (int64_t)ord.size();
        }
      }
      for (int64_t i = 0; i < nl; ++i) P.ptr[i + 1] += P.ptr[i];
      P.col.reserve(P.ptr[nl]);
      P.val.reserve(P.ptr[nl]);
      for (int t = 0; t < nt; ++t) {
        P.col.insert(P.col.end(), tcol[t].begin(), tcol[t].end());
        P.val.insert(P.val.end(), tval[t].begin(), tval[t].end());
      }
    }
    L.P = std::move(P);
    phase("prolongator", lev);
    L.R = transpose(L.P);
    AmgLevel next;
    next.A = spgemm(L.R, spgemm(L.A, L.P));
    phase("galerkin", lev);
    {  // exact symmetry (the products round differently per side): A_c = (A_c + A_c^T) / 2
      const Csr t = transpose(next.A);
      for (int64_t e = 0; e < next.A.ptr[next.A.n]; ++e) next.A.val[e] = 0.5 * (next.A.val[e] + t.val[e]);
    }
    h->lv.push_back(std::move(next));
    phase("symmetrise", lev);
  }
  // ---- dense inverse of the coarsest operator (Cholesky, then columns) ----
  if (!h->skip_coarse_inverse) {
    const Csr& A = h->lv.back().A;
    const int64_t nc = A.n;
    std::vector<double> M((size_t)nc * nc, 0.0);
    for (int64_t i = 0; i < nc; ++i)
      for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e) M[(size_t)i * nc + A.col[e]] = A.val[e];
    for (int64_t j = 0; j < nc; ++j) {  // in-place lower Cholesky
      double d = M[(size_t)j * nc + j];
      for (int64_t k = 0; k < j; ++k) d -= M[(size_t)j * nc + k] * M[(size_t)j * nc + k];
      QN_REQUIRE(d > 0.0, QN_ERR_NOT_SPD, "amg: coarsest operator is not positive definite");
      d = std::sqrt(d);
      M[(size_t)j * nc + j] = d;
#pragma omp parallel for schedule(static)
      for (int64_t i = j + 1; i < nc; ++i) {
        double s = M[(size_t)i * nc + j];
        for (int64_t k = 0; k < j; ++k) s -= M[(size_t)i * nc + k] * M[(size_t)j * nc + k];
        M[(size_t)i * nc + j] = s / d;
      }
    }
    h->coarse_inv.assign((size_t)nc * nc, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t c = 0; c < nc; ++c) {  // column c of A^-1: L L^T x = e_c
      std::vector<double> z(nc, 0.0);
      for (int64_t i = c; i < nc; ++i) {
        double s = i == c ? 1.0 : 0.0;
        for (int64_t k = c; k < i; ++k) s -= M[(size_t)i * nc + k] * z[k];
        z[i] = s / M[(size_t)i * nc + i];
      }
      for (int64_t i = nc - 1; i >= 0; --i) {
        double s = z[i];
        for (int64_t k = i + 1; k < nc; ++k) s -= M[(size_t)k * nc + i] * z[k];
        z[i] = s / M[(size_t)i * nc + i];
      }
      for (int64_t i = 0; i < nc; ++i) h->coarse_inv[(size_t)i * nc + c] = z[i];
    }
  }
  phase("coarse inv", (int)h->lv.size() - 1);
  h->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return QN_OK;
}

// ---- host reference V(1,1) cycle and PCG (mirror the device kernels) ----
namespace {
void vcycle_level(const AmgHierarchy& h, size_t l, const double* b, double* x) {
  const AmgLevel& L = h.lv[l];
  const int64_t n = L.A.n;
  if (l + 1 == h.lv.size()) {
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += h.coarse_inv[(size_t)i * n + j] * b[3 * j + a];
        x[3 * i + a] = s;
      }
    return;
  }
  const double w = h.omega_l[l];
  std::vector<double> r(3 * n), ax(3 * n);
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) x[3 * i + a] = w * L.dinv[i] * b[3 * i + a];  // pre-smooth from 0
  spmv3(L.A, x, ax.data());
  for (int64_t k = 0; k < 3 * n; ++k) r[k] = b[k] - ax[k];
  const int64_t nc = L.R.n;
  std::vector<double> bc(3 * nc), xc(3 * nc);
  spmv3(L.R, r.data(), bc.data());
  vcycle_level(h, l + 1, bc.data(), xc.data());
  std::vector<double> px(3 * n);
  spmv3(L.P, xc.data(), px.data());
  for (int64_t k = 0; k < 3 * n; ++k) x[k] += px[k];
  spmv3(L.A, x, ax.data());  // post-smooth
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) x[3 * i + a] += w * L.dinv[i] * (b[3 * i + a] - ax[3 * i + a]);
}
}  // namespace

void amg_vcycle_host(const AmgHierarchy& h, const double* b, double* x) { vcycle_level(h, 0, b, x); }

int amg_pcg_host(const AmgHierarchy& h, const double* b, double* x, double tol, int maxit) {
  const Csr& A = h.lv[0].A;
  const int64_t n = A.n;
  std::vector<double> r(b, b + 3 * n), z(3 * n), p(3 * n), q(3 * n);
  std::fill(x, x + 3 * n, 0.0);
  amg_vcycle_host(h, r.data(), z.data());
  p = z;
  double rz[3] = {0, 0, 0}, bb[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      rz[a] += r[3 * i + a] * z[3 * i + a];
      bb[a] += b[3 * i + a] * b[3 * i + a];
    }
  int it = 0;
  bool conv[3] = {!(bb[0] > 0), !(bb[1] > 0), !(bb[2] > 0)};
  while (it < maxit && !(conv[0] && conv[1] && conv[2])) {
    spmv3(A, p.data(), q.data());
    double pq[3] = {0, 0, 0}, rr[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) pq[a] += p[3 * i + a] * q[3 * i + a];
    for (int a = 0; a < 3; ++a) {
      const double al = conv[a] ? 0.0 : rz[a] / pq[a];
      for (int64_t i = 0; i < n; ++i) {
        x[3 * i + a] += al * p[3 * i + a];
        r[3 * i + a] -= al * q[3 * i + a];
        rr[a] += r[3 * i + a] * r[3 * i + a];
      }
    }
    ++it;
    for (int a = 0; a < 3; ++a)
      if (rr[a] <= tol * tol * bb[a]) conv[a] = true;
    amg_vcycle_host(h, r.data(), z.data());
    for (int a = 0; a < 3; ++a) {
      if (conv[a]) continue;
      double rzn = 0.0;
      for (int64_t i = 0; i < n; ++i) rzn += r[3 * i + a] * z[3 * i + a];
      const double be = rzn / rz[a];
      rz[a] = rzn;
      for (int64_t i = 0; i < n; ++i) p[3 * i + a] = z[3 * i + a] + be * p[3 * i + a];
    }
  }
  return it;
}

}  // namespace qn

// Per-tetrahedron device math: fp64 rotation-variant 3x3 SVD, Valanis-Landel
// energy / principal stress, PK1 stress and corner forces.
//
// Reference semantics restated here:
//   svd_rv_batch          linalg.py:86-110  (sign rule, ordering, 1e-10 clamp)
//   PolyFn/LogFn/HermiteFn materials.py:40-133
//   vl_energy/vl_stress   materials.py:181-207
//   elem_gradient         dynamics.py:50-55 (P = U diag(tau) V^T, vol * P G^T)
#pragma once

#include "qn_common.cuh"

namespace qn {

constexpr double kSigmaClamp = 1e-10;  // linalg.py:13

// ---------------------------------------------------------------------------
// scalar functions

__device__ __forceinline__ void poly_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  // numpy polyval = Horner from the highest coefficient (materials.py:48-51)
  const int n = f.n;
  double a = f.c[n - 1];
  for (int i = n - 2; i >= 0; --i) a = fma(a, x, f.c[i]);
  v = a;
  if (n > 1) {
    double d = f.dc[n - 2];
    for (int i = n - 3; i >= 0; --i) d = fma(d, x, f.dc[i]);
    dv = d;
  } else {
    dv = 0.0;
  }
}

// fp64 1/x for |x| in the fp32 normal range: SFU seed + two Newton steps (~1 ulp)
__device__ __forceinline__ double rcp_nr(double x) {
  double y = (double)__frcp_rn((float)x);
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

__device__ __forceinline__ void log_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  // materials.py:57-80: core for x > eps, quadratic Taylor continuation below
  const bool core = x > f.eps;
  const double xs = core ? x : 1.0;
  const double lx = log(xs);
  const double d = x - f.eps;
  v = core ? f.alpha * lx + 0.5 * f.beta * lx * lx : f.f0 + f.f1 * d + 0.5 * f.f2 * d * d;
  dv = core ? (f.alpha + f.beta * lx) * rcp_nr(xs) : f.f1 + f.f2 * d;
}

__device__ __forceinline__ void hermite_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  // materials.py:99-133: segment = searchsorted(xs, x, 'right') - 1 clipped to
  // [0, K-2]; linear extrapolation outside [xs0, xsK-1].
  const int K = f.n;
  if (x < f.xs[0]) {
    v = f.ys[0] + f.ts[0] * (x - f.xs[0]);
    dv = f.ts[0];
    return;
  }
  if (x > f.xs[K - 1]) {
    v = f.ys[K - 1] + f.ts[K - 1] * (x - f.xs[K - 1]);
    dv = f.ts[K - 1];
    return;
  }
  int i = 0;
  for (int k = 1; k < K - 1; ++k) i += (f.xs[k] <= x) ? 1 : 0;
  const double h = f.xs[i + 1] - f.xs[i];
  const double ih = rcp_nr(h);
  const double u = (x - f.xs[i]) * ih;
  const double u2 = u * u, u3 = u2 * u;
  const double y0 = f.ys[i], y1 = f.ys[i + 1], t0 = f.ts[i], t1 = f.ts[i + 1];
  v = (2 * u3 - 3 * u2 + 1) * y0 + (u3 - 2 * u2 + u) * h * t0 + (-2 * u3 + 3 * u2) * y1 + (u3 - u2) * h * t1;
  dv = ((6 * u2 - 6 * u) * y0 + (-6 * u2 + 6 * u) * y1) * ih + (3 * u2 - 4 * u + 1) * t0 + (3 * u2 - 2 * u) * t1;
}

// c0 (x - c1)^2 evaluated on the deviation (no cancellation near x = c1)
__device__ __forceinline__ void sqdev_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  const double u = x - f.c[1];
  v = f.c[0] * (u * u);
  dv = (2.0 * f.c[0]) * u;
}

__device__ __forceinline__ void fn_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  switch (f.kind) {
    case QN_FN_POLY: poly_eval(f, x, v, dv); break;
    case QN_FN_SQDEV: sqdev_eval(f, x, v, dv); break;
    case QN_FN_LOG: log_eval(f, x, v, dv); break;
    case QN_FN_HERMITE: hermite_eval(f, x, v, dv); break;
    default: v = 0.0; dv = 0.0; break;
  }
}

// f and f' at N points with one dispatch (the function kind is uniform across a
// warp); a polynomial's coefficients are loaded once for all N Horner chains.
template <int N>
__device__ __forceinline__ void fn_eval_n(const qn_scalar_fn& f, const double (&x)[N], double (&v)[N],
                                          double (&dv)[N]) {
  const int kind = f.kind;
  if (kind == QN_FN_POLY) {
    const int n = f.n;
    double a[N], d[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      a[j] = f.c[n - 1];
      d[j] = n > 1 ? f.dc[n - 2] : 0.0;
    }
    for (int i = n - 2; i >= 0; --i) {
      const double ci = f.c[i];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = fma(a[j], x[j], ci);
    }
    for (int i = n - 3; i >= 0; --i) {
      const double di = f.dc[i];
#pragma unroll
      for (int j = 0; j < N; ++j) d[j] = fma(d[j], x[j], di);
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      v[j] = a[j];
      dv[j] = d[j];
    }
  } else if (kind == QN_FN_LOG) {
#pragma unroll
    for (int j = 0; j < N; ++j) log_eval(f, x[j], v[j], dv[j]);
  } else if (kind == QN_FN_HERMITE) {
#pragma unroll
    for (int j = 0; j < N; ++j) hermite_eval(f, x[j], v[j], dv[j]);
  } else if (kind == QN_FN_SQDEV) {
#pragma unroll
    for (int j = 0; j < N; ++j) sqdev_eval(f, x[j], v[j], dv[j]);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = dv[j] = 0.0;
  }
}

// Psi(s) - shift and tau = dPsi/ds  (materials.py:181-207)
__device__ __forceinline__ double vl_eval(const qn_material& M, const double s[3], double tau[3]) {
  double a[3], da[3], b[3], db[3], c[1], dc[1];
  const double xa[3] = {s[0], s[1], s[2]};
  const double xb[3] = {s[0] * s[1], s[1] * s[2], s[0] * s[2]};  // b01, b12, b02
  const double xc[1] = {s[0] * s[1] * s[2]};
  fn_eval_n<3>(M.a, xa, a, da);
  fn_eval_n<3>(M.b, xb, b, db);
  fn_eval_n<1>(M.c, xc, c, dc);
  tau[0] = da[0] + db[0] * s[1] + db[2] * s[2] + dc[0] * s[1] * s[2];
  tau[1] = da[1] + db[0] * s[0] + db[1] * s[2] + dc[0] * s[0] * s[2];
  tau[2] = da[2] + db[1] * s[1] + db[2] * s[0] + dc[0] * s[0] * s[1];
  return a[0] + a[1] + a[2] + b[0] + b[1] + b[2] + c[0] - M.shift;
}

// ---------------------------------------------------------------------------
// fp64 rotation-variant SVD.
// 1) cyclic Jacobi on the symmetric A = F^T F gives V (a proper rotation);
// 2) columns sorted by eigenvalue (swap + negate keeps det V = +1);
// 3) Givens QR of B = F V gives U (product of rotations, det U = +1) and
//    R with R00, R11 >= 0; sigma = diag(R), so sigma2 carries sign(det F) and
//    has the smallest magnitude — the reference's rule (linalg.py:95-103).
// Matrices are row-major m[r*3+c].

// fp64 1/sqrt(x) for x in the fp32 normal range: SFU seed + two Newton steps
// (relative error ~1e-16, no library slow paths or branches).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = (double)rsqrtf((float)x);
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// One Jacobi rotation in the (p,q) plane.  The angle only needs to be
// approximate (it is computed in fp32 on the SFU); the rotation itself is an
// exact fp64 rotation (c^2 + s^2 = 1 to rounding) applied as a full
// similarity transform, so A stays symmetric-similar and V orthogonal, and
// the next sweep removes what the approximate angle left (~1e-7 relative).
// Branch-free (lanes never diverge): a converged pair gets t = 0, i.e. the
// identity rotation c = 1, s = 0, which leaves A and V bit-identical.
// Returns whether the pair needed a rotation that was not tiny (|t| >= 1e-12):
// after a sweep of tiny rotations the off-diagonal is ~1e-7 |t| (the fp32
// angle's error) below the diagonal, under the 1e-18 rotation threshold, so
// the sweep that would only confirm convergence is skipped.
__device__ __forceinline__ bool jacobi_rot(double (&A)[3][3], double (&V)[3][3], int p, int q) {
  const double apq = A[p][q];
  const double app = A[p][p], aqq = A[q][q];
  const float d = (float)(aqq - app), a = (float)apq;
  // tan of the Jacobi angle, stable form: t = 2a sign(d) / (|d| + sqrt(d^2 + 4a^2))
  const float den = fabsf(d) + sqrtf(fmaf(d, d, 4.f * a * a));
  // rotate unless apq is below the fp64 resolution of the diagonal (or of fp32)
  const bool need = apq * apq > 1e-36 * fabs(app * aqq) && den > 0.f;
  const float tf = __fdividef(2.f * a, need ? den : 1.f) * (d >= 0.f ? 1.f : -1.f);
  const double t = need ? (double)tf : 0.0;
  const double c = rsqrt_nr(fma(t, t, 1.0));
  const double s = t * c;
  const double cc = c * c, ss = s * s, cs = c * s;
  A[p][p] = fma(cc, app, fma(ss, aqq, -2.0 * cs * apq));
  A[q][q] = fma(ss, app, fma(cc, aqq, 2.0 * cs * apq));
  A[p][q] = A[q][p] = fma(cc - ss, apq, cs * (app - aqq));
  const int r = 3 - p - q;
  const double arp = A[r][p], arq = A[r][q];
  A[r][p] = A[p][r] = c * arp - s * arq;
  A[r][q] = A[q][r] = s * arp + c * arq;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double vkp = V[k][p], vkq = V[k][q];
    V[k][p] = c * vkp - s * vkq;
    V[k][q] = s * vkp + c * vkq;
  }
  return need && fabs(t) >= 1e-12;
}

// swap eigenpairs i <-> j when A[i][i] < A[j][j] (branch-free); the swapped
// column is negated so det V stays +1
__device__ __forceinline__ void sort_pair(double (&A)[3][3], double (&V)[3][3], int i, int j) {
  const bool sw = A[i][i] < A[j][j];
  const double ai = A[i][i], aj = A[j][j];
  A[i][i] = sw ? aj : ai;
  A[j][j] = sw ? ai : aj;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double vi = V[k][i], vj = V[k][j];
    V[k][i] = sw ? vj : vi;
    V[k][j] = sw ? -vi : vj;
  }
}

// Givens rotation acting on rows (p,q) of R, accumulated into the columns of U.
__device__ __forceinline__ void givens_qr(double (&R)[3][3], double (&U)[3][3], int p, int q, int col) {
  // c = a / r, s = b / r makes the new pivot r >= 0 (for b = 0, a < 0 this is
  // the rotation by pi); r = 0 keeps the identity.  Branch-free except for
  // pivots outside the fp32 range of the rsqrt seed.
  const double a = R[p][col], b = R[q][col];
  const double r2 = fma(a, a, b * b);
  double inv;
  if (r2 > 1e-36 && r2 < 1e36) {
    inv = rsqrt_nr(r2);
  } else {
    inv = r2 > 0.0 ? rsqrt(r2) : 0.0;
  }
  const double c = r2 > 0.0 ? a * inv : 1.0;
  const double s = b * inv;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double rp = R[p][k], rq = R[q][k];
    R[p][k] = c * rp + s * rq;
    R[q][k] = -s * rp + c * rq;
    const double up = U[k][p], uq = U[k][q];
    U[k][p] = c * up + s * uq;
    U[k][q] = -s * up + c * uq;
  }
  R[q][col] = 0.0;
}

__device__ __forceinline__ void svd_rv3(const double (&F)[3][3], double (&U)[3][3], double (&sig)[3],
                                        double (&V)[3][3]) {
  double A[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) A[i][j] = F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  // cyclic sweeps until no pair needs a rotation; the exit is a warp vote so
  // the loop stays convergent across lanes (callers keep all 32 lanes active)
  for (int sweep = 0; sweep < 12; ++sweep) {
    bool rot = jacobi_rot(A, V, 0, 1);
    rot |= jacobi_rot(A, V, 0, 2);
    rot |= jacobi_rot(A, V, 1, 2);
    if (!__any_sync(0xffffffffu, rot)) break;
  }
  // sort eigenvalues descending
  sort_pair(A, V, 0, 1);
  sort_pair(A, V, 0, 2);
  sort_pair(A, V, 1, 2);
  // B = F V
  double R[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) R[i][j] = F[i][0] * V[0][j] + F[i][1] * V[1][j] + F[i][2] * V[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) U[i][j] = (i == j) ? 1.0 : 0.0;
  givens_qr(R, U, 0, 1, 0);
  givens_qr(R, U, 0, 2, 0);
  givens_qr(R, U, 1, 2, 1);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double s = R[i][i];
    if (fabs(s) < kSigmaClamp) s = (s < 0.0) ? -kSigmaClamp : kSigmaClamp;  // linalg.py:105-109
    sig[i] = s;
  }
}

// Energy density and corner forces of one tet.
//   x[v][a]: corner positions; Dminv[j][c] = G[j+1][c] (mesh.py:212-215)
//   forces[v][a] = vol * sum_c P[a][c] G[v][c]  with G[0] = -(Dminv rows summed)
// Returns vol * (Psi - shift).
template <bool kForces>
__device__ __forceinline__ double tet_eval(const qn_material& M, const double (&x)[4][3],
                                           const double (&Dm)[3][3], double vol, double (&f)[4][3]) {
  double F[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double e0 = x[1][a] - x[0][a], e1 = x[2][a] - x[0][a], e2 = x[3][a] - x[0][a];
#pragma unroll
    for (int c = 0; c < 3; ++c) F[a][c] = e0 * Dm[0][c] + e1 * Dm[1][c] + e2 * Dm[2][c];
  }
  double U[3][3], s[3], V[3][3], tau[3];
  svd_rv3(F, U, s, V);
  const double psi = vl_eval(M, s, tau);
  if (kForces) {
    double P[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        P[a][c] = vol * (U[a][0] * tau[0] * V[c][0] + U[a][1] * tau[1] * V[c][1] + U[a][2] * tau[2] * V[c][2]);
    double G0[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) G0[c] = -(Dm[0][c] + Dm[1][c] + Dm[2][c]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      f[0][a] = P[a][0] * G0[0] + P[a][1] * G0[1] + P[a][2] * G0[2];
#pragma unroll
      for (int v = 1; v < 4; ++v) f[v][a] = P[a][0] * Dm[v - 1][0] + P[a][1] * Dm[v - 1][1] + P[a][2] * Dm[v - 1][2];
    }
  }
  return vol * psi;
}

// anisotropic fibre (dynamics.py:154-193): u = F d, energy w/2 (|u| - 1)^2 with
// w = vol kappa, P = w (|u|' - 1)/|u|' u d^T with |u|' = max(|u|, 1e-12)
__device__ __forceinline__ double aniso_eval(const qn_material& M, const double (&x)[4][3],
                                             const double (&Dm)[3][3], double vol, double (&f)[4][3]) {
  const double d[3] = {M.a.c[0], M.a.c[1], M.a.c[2]};
  const double w = vol * M.a.c[3];
  double u[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double e0 = x[1][a] - x[0][a], e1 = x[2][a] - x[0][a], e2 = x[3][a] - x[0][a];
    double Fa[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) Fa[c] = e0 * Dm[0][c] + e1 * Dm[1][c] + e2 * Dm[2][c];
    u[a] = Fa[0] * d[0] + Fa[1] * d[1] + Fa[2] * d[2];
  }
  const double nu = sqrt((u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]);
  const double nuc = fmax(nu, 1e-12);
  const double coef = w * (nuc - 1.0) / nuc;
  double G0[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) G0[c] = -(Dm[0][c] + Dm[1][c] + Dm[2][c]);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double pa = coef * u[a];
    f[0][a] = pa * (d[0] * G0[0] + d[1] * G0[1] + d[2] * G0[2]);
#pragma unroll
    for (int v = 1; v < 4; ++v) f[v][a] = pa * (d[0] * Dm[v - 1][0] + d[1] * Dm[v - 1][1] + d[2] * Dm[v - 1][2]);
  }
  return 0.5 * w * ((nu - 1.0) * (nu - 1.0));
}

}  // namespace qn

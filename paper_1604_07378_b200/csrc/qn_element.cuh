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

__device__ __forceinline__ void log_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  // materials.py:57-80: core for x > eps, quadratic Taylor continuation below
  if (x > f.eps) {
    const double lx = log(x);
    v = f.alpha * lx + 0.5 * f.beta * lx * lx;
    dv = (f.alpha + f.beta * lx) / x;
  } else {
    const double d = x - f.eps;
    v = f.f0 + f.f1 * d + 0.5 * f.f2 * d * d;
    dv = f.f1 + f.f2 * d;
  }
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
  const double u = (x - f.xs[i]) / h;
  const double u2 = u * u, u3 = u2 * u;
  const double y0 = f.ys[i], y1 = f.ys[i + 1], t0 = f.ts[i], t1 = f.ts[i + 1];
  v = (2 * u3 - 3 * u2 + 1) * y0 + (u3 - 2 * u2 + u) * h * t0 + (-2 * u3 + 3 * u2) * y1 + (u3 - u2) * h * t1;
  dv = (6 * u2 - 6 * u) * y0 / h + (3 * u2 - 4 * u + 1) * t0 + (-6 * u2 + 6 * u) * y1 / h + (3 * u2 - 2 * u) * t1;
}

__device__ __forceinline__ void fn_eval(const qn_scalar_fn& f, double x, double& v, double& dv) {
  switch (f.kind) {
    case QN_FN_POLY: poly_eval(f, x, v, dv); break;
    case QN_FN_LOG: log_eval(f, x, v, dv); break;
    case QN_FN_HERMITE: hermite_eval(f, x, v, dv); break;
    default: v = 0.0; dv = 0.0; break;
  }
}

// Psi(s) - shift and tau = dPsi/ds  (materials.py:181-207)
__device__ __forceinline__ double vl_eval(const qn_material& M, const double s[3], double tau[3]) {
  double a0, a1, a2, da0, da1, da2;
  fn_eval(M.a, s[0], a0, da0);
  fn_eval(M.a, s[1], a1, da1);
  fn_eval(M.a, s[2], a2, da2);
  double b01 = 0, b12 = 0, b02 = 0, db01 = 0, db12 = 0, db02 = 0;
  if (M.b.kind != QN_FN_ZERO) {
    fn_eval(M.b, s[0] * s[1], b01, db01);
    fn_eval(M.b, s[1] * s[2], b12, db12);
    fn_eval(M.b, s[0] * s[2], b02, db02);
  }
  double c = 0, dc = 0;
  if (M.c.kind != QN_FN_ZERO) fn_eval(M.c, s[0] * s[1] * s[2], c, dc);
  tau[0] = da0 + db01 * s[1] + db02 * s[2] + dc * s[1] * s[2];
  tau[1] = da1 + db01 * s[0] + db12 * s[2] + dc * s[0] * s[2];
  tau[2] = da2 + db12 * s[1] + db02 * s[0] + dc * s[0] * s[1];
  return a0 + a1 + a2 + b01 + b12 + b02 + c - M.shift;
}

// ---------------------------------------------------------------------------
// fp64 rotation-variant SVD.
// 1) cyclic Jacobi on the symmetric A = F^T F gives V (a proper rotation);
// 2) columns sorted by eigenvalue (swap + negate keeps det V = +1);
// 3) Givens QR of B = F V gives U (product of rotations, det U = +1) and
//    R with R00, R11 >= 0; sigma = diag(R), so sigma2 carries sign(det F) and
//    has the smallest magnitude — the reference's rule (linalg.py:95-103).
// Matrices are row-major m[r*3+c].

__device__ __forceinline__ void jacobi_rot(double (&A)[3][3], double (&V)[3][3], int p, int q) {
  const double apq = A[p][q];
  const double app = A[p][p], aqq = A[q][q];
  // skip rotations below the fp64 resolution of the diagonal (and apq == 0)
  if (fabs(apq) <= 1e-18 * sqrt(fabs(app * aqq))) return;
  const double theta = (aqq - app) / (2.0 * apq);
  double t;
  if (fabs(theta) > 1e150) {
    t = 0.5 / theta;
  } else {
    t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
  }
  const double c = rsqrt(t * t + 1.0);
  const double s = t * c;
  A[p][p] = app - t * apq;
  A[q][q] = aqq + t * apq;
  A[p][q] = A[q][p] = 0.0;
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
}

__device__ __forceinline__ void swap_cols(double (&A)[3][3], double (&V)[3][3], int i, int j) {
  // swap eigenpairs i <-> j; negate one column so det V stays +1
  double t = A[i][i];
  A[i][i] = A[j][j];
  A[j][j] = t;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double a = V[k][i];
    V[k][i] = V[k][j];
    V[k][j] = -a;
  }
}

// Givens rotation acting on rows (p,q) of R, accumulated into the columns of U.
__device__ __forceinline__ void givens_qr(double (&R)[3][3], double (&U)[3][3], int p, int q, int col) {
  const double a = R[p][col], b = R[q][col];
  double c, s;
  if (b == 0.0) {
    if (a >= 0.0) return;
    c = -1.0;  // rotation by pi in the (p,q) plane makes the pivot non-negative
    s = 0.0;
  } else {
    const double inv = rsqrt(a * a + b * b);
    c = a * inv;
    s = b * inv;
  }
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
  for (int sweep = 0; sweep < 8; ++sweep) {
    jacobi_rot(A, V, 0, 1);
    jacobi_rot(A, V, 0, 2);
    jacobi_rot(A, V, 1, 2);
    const double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    const double dia = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
    if (off <= 1e-17 * dia) break;
  }
  // sort eigenvalues descending
  if (A[0][0] < A[1][1]) swap_cols(A, V, 0, 1);
  if (A[0][0] < A[2][2]) swap_cols(A, V, 0, 2);
  if (A[1][1] < A[2][2]) swap_cols(A, V, 1, 2);
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

}  // namespace qn

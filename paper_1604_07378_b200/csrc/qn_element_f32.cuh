// fp32 variant of the per-tet math (the optional fp32 mode of configs[2],
// BASELINE.json; tolerance 1e-4 on positions).  Same algorithm as the fp64
// path in qn_element.cuh — cyclic Jacobi on F^T F for V, descending sort,
// Givens QR of F V for U with the sign rule of linalg.py:95-103, the 1e-10
// clamp, Valanis-Landel energy / principal stresses, PK1 and corner forces —
// the SVD, PK1 and corner forces in single precision.  Positions and Dm^-1
// are read in fp64 and rounded once; energies and forces return to fp64 for the
// deterministic fp64 gather and reductions; the material functions run in
// fp64 on the fp32 stretches (cheap next to the SVD, and free of the fp32
// cancellation of expanded polynomials).  The fp64 path is untouched.
#pragma once

#include "qn_element.cuh"

namespace qn {

__device__ __forceinline__ bool jacobi_rot_f(float (&A)[3][3], float (&V)[3][3], int p, int q) {
  const float apq = A[p][q], app = A[p][p], aqq = A[q][q];
  const float d = aqq - app;
  const float den = fabsf(d) + sqrtf(fmaf(d, d, 4.f * apq * apq));
  const bool need = apq * apq > 1e-13f * fabsf(app * aqq) && den > 0.f;
  const float t = need ? __fdividef(2.f * apq, den) * (d >= 0.f ? 1.f : -1.f) : 0.f;
  const float c = rsqrtf(fmaf(t, t, 1.f));
  const float s = t * c;
  const float cc = c * c, ss = s * s, cs = c * s;
  A[p][p] = fmaf(cc, app, fmaf(ss, aqq, -2.f * cs * apq));
  A[q][q] = fmaf(ss, app, fmaf(cc, aqq, 2.f * cs * apq));
  A[p][q] = A[q][p] = fmaf(cc - ss, apq, cs * (app - aqq));
  const int r = 3 - p - q;
  const float arp = A[r][p], arq = A[r][q];
  A[r][p] = A[p][r] = c * arp - s * arq;
  A[r][q] = A[q][r] = s * arp + c * arq;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float vkp = V[k][p], vkq = V[k][q];
    V[k][p] = c * vkp - s * vkq;
    V[k][q] = s * vkp + c * vkq;
  }
  return need;
}

__device__ __forceinline__ void sort_pair_f(float (&A)[3][3], float (&V)[3][3], int i, int j) {
  const bool sw = A[i][i] < A[j][j];
  const float ai = A[i][i], aj = A[j][j];
  A[i][i] = sw ? aj : ai;
  A[j][j] = sw ? ai : aj;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float vi = V[k][i], vj = V[k][j];
    V[k][i] = sw ? vj : vi;
    V[k][j] = sw ? -vi : vj;
  }
}

__device__ __forceinline__ void givens_qr_f(float (&R)[3][3], float (&U)[3][3], int p, int q, int col) {
  const float a = R[p][col], b = R[q][col];
  const float r2 = fmaf(a, a, b * b);
  const float inv = r2 > 0.f ? rsqrtf(r2) : 0.f;
  const float c = r2 > 0.f ? a * inv : 1.f;
  const float s = b * inv;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float rp = R[p][k], rq = R[q][k];
    R[p][k] = c * rp + s * rq;
    R[q][k] = -s * rp + c * rq;
    const float up = U[k][p], uq = U[k][q];
    U[k][p] = c * up + s * uq;
    U[k][q] = -s * up + c * uq;
  }
  R[q][col] = 0.f;
}

__device__ __forceinline__ void svd_rv3_f(const float (&F)[3][3], float (&U)[3][3], float (&sig)[3],
                                          float (&V)[3][3]) {
  float A[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) A[i][j] = F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.f : 0.f;
  for (int sweep = 0; sweep < 12; ++sweep) {
    bool rot = jacobi_rot_f(A, V, 0, 1);
    rot |= jacobi_rot_f(A, V, 0, 2);
    rot |= jacobi_rot_f(A, V, 1, 2);
    if (!__any_sync(0xffffffffu, rot)) break;
  }
  sort_pair_f(A, V, 0, 1);
  sort_pair_f(A, V, 0, 2);
  sort_pair_f(A, V, 1, 2);
  float R[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) R[i][j] = F[i][0] * V[0][j] + F[i][1] * V[1][j] + F[i][2] * V[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) U[i][j] = (i == j) ? 1.f : 0.f;
  givens_qr_f(R, U, 0, 1, 0);
  givens_qr_f(R, U, 0, 2, 0);
  givens_qr_f(R, U, 1, 2, 1);
  const float clamp = (float)kSigmaClamp;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float s = R[i][i];
    if (fabsf(s) < clamp) s = (s < 0.f) ? -clamp : clamp;
    sig[i] = s;
  }
}

// energy (vol (Psi - shift)) and corner forces in fp32, returned in fp64
__device__ __forceinline__ double tet_eval_f32(const qn_material& M, const double (&x)[4][3],
                                               const double (&Dmd)[3][3], double vold, double (&f)[4][3]) {
  float Dm[3][3], F[3][3];
  const float vol = (float)vold;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Dm[r][c] = (float)Dmd[r][c];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float e0 = (float)(x[1][a] - x[0][a]), e1 = (float)(x[2][a] - x[0][a]), e2 = (float)(x[3][a] - x[0][a]);
#pragma unroll
    for (int c = 0; c < 3; ++c) F[a][c] = e0 * Dm[0][c] + e1 * Dm[1][c] + e2 * Dm[2][c];
  }
  float U[3][3], s[3], V[3][3], tau[3];
  svd_rv3_f(F, U, s, V);
  // the material in fp64 on the fp32 stretches: expanded polynomials (StVK,
  // cubic terms) cancel to ~1e-7 of their magnitude at rest, which fp32 would
  // turn into an energy offset the Armijo test cannot see through
  const double sd[3] = {(double)s[0], (double)s[1], (double)s[2]};
  double taud[3];
  const double psi = vl_eval(M, sd, taud);
  for (int i = 0; i < 3; ++i) tau[i] = (float)taud[i];
  float P[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      P[a][c] = vol * (U[a][0] * tau[0] * V[c][0] + U[a][1] * tau[1] * V[c][1] + U[a][2] * tau[2] * V[c][2]);
  float G0[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) G0[c] = -(Dm[0][c] + Dm[1][c] + Dm[2][c]);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    f[0][a] = (double)(P[a][0] * G0[0] + P[a][1] * G0[1] + P[a][2] * G0[2]);
#pragma unroll
    for (int v = 1; v < 4; ++v)
      f[v][a] = (double)(P[a][0] * Dm[v - 1][0] + P[a][1] * Dm[v - 1][1] + P[a][2] * Dm[v - 1][2]);
  }
  return vold * psi;
}

}  // namespace qn

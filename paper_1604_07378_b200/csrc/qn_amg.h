// Smoothed-aggregation algebraic multigrid hierarchy for the PCG solve of
// configs[4] (A_free = M/h^2 + L, scalar, SPD; SURVEY.md §8 c5 "distributed
// PCG on A to relative residual 1e-10").  Built once on the host (C++/OpenMP);
// the device runs a symmetric V(1,1) cycle (weighted Jacobi smoothing,
// Galerkin coarse operators, dense inverse on the coarsest level) as the CG
// preconditioner.  Any SPD preconditioner leaves the CG solution defined by
// the same residual tolerance, so the frame results stay within the PCG
// tolerance of the direct solve (tests/test_gpu_parity.py).
#pragma once

#include <cstdint>
#include <vector>

namespace qn {

struct Csr {
  int64_t n = 0, m = 0;  // rows, cols
  std::vector<int64_t> ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};

struct AmgLevel {
  Csr A;                    // level operator (n x n)
  std::vector<double> dinv; // 1 / diag(A)
  Csr P;                    // prolongator (n x n_coarse), empty on the coarsest level
  Csr R;                    // restriction = P^T (n_coarse x n)
};

struct AmgHierarchy {
  std::vector<AmgLevel> lv;
  std::vector<double> coarse_inv;  // dense inverse of the coarsest operator (row-major)
  bool skip_coarse_inverse = false;  // caller inverts the coarsest operator itself (device: cuSOLVER)
  std::vector<double> omega_l;     // Jacobi smoothing weight per level: 4 / (3 rho(D^-1 A))
  double setup_seconds = 0.0;
};

constexpr int64_t kAmgCoarsest = 3072;    // stop coarsening at or below this many rows (dense inverse <= 75 MB)
constexpr int kAmgMaxLevels = 10;
constexpr double kAmgStrength = 0.08;     // |a_ij| >= theta sqrt(a_ii a_jj)

// Build the hierarchy for the CSR matrix (rows sorted, both triangles).
int amg_build(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, AmgHierarchy* h);

// Host reference of the device V-cycle / PCG (tests only): x = B b for 3 RHS
// ([n][3]), and a full PCG solve returning the iteration count.
void amg_vcycle_host(const AmgHierarchy& h, const double* b, double* x);
int amg_pcg_host(const AmgHierarchy& h, const double* b, double* x, double tol, int maxit);

}  // namespace qn

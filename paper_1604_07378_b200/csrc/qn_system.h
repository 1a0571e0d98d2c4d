// Device-resident simulation system (SimSystem + SimState + solver workspace).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "qn_factor.h"
#include "qnsim_b200.h"

namespace qn {

// per-instance solver phase (one body pass of the frame graph advances every
// instance by one step of this machine; see qn_solver.cu)
enum Phase : int32_t {
  PH_FIRST = 0,  // evaluate g0 and corner forces at x = y
  PH_GRAD = 1,   // gather gradient, L-BFGS push, zeta's
  PH_DIR = 2,    // triangular solves, eta's, direction, first trial formed
  PH_ALPHA = 3,  // backtracking trial x + alpha d
  PH_COPY = 4,   // re-evaluate corner forces at the current x (after slope early-out)
  PH_DONE = 5,
};

constexpr int kMaxM = QN_MAX_M;
constexpr int kVertexThreads = 128;     // vertex kernels of batched systems: small blocks so every SM gets work
constexpr int kVertexThreadsMax = 256;
constexpr int kTetThreads = 128;  // per-tet kernel block (qn_kernels.cuh kTT; the grid is mt / kTetThreads)  // vertex kernels of single systems (swept on configs[1]: 256 > 128)
constexpr int kNG = 5 + 2 * kMaxM;  // gradient-kernel dot products per block

struct InstCtl {
  int32_t phase, k, trials, status;
  int32_t xs_cur, xs_prev, xs_trial, gs_cur;
  int32_t npairs, have_prev, fallbacks, cheb_fb;  // chebyshev: fallbacks so far, this direction fell back
  int32_t ring[kMaxM + 1];
  double g0, g_x, alpha, slope;
  double e_base, e_col;  // colliders: objective without the collision term at x; collision term at the trial
  double omega;          // chebyshev weight of the current direction (solvers.py:154-164)
  unsigned long long t0;
  double rho[kMaxM + 1];
  double tt[kMaxM + 1];  // <t, t> per slot (lbfgs_init = scaled_identity)
  double sg[kMaxM + 1];
  double gram[kMaxM + 1][kMaxM + 1];  // gram[i][j] = <s_i, t_j> (slot ids), i older than j
  double zeta[kMaxM];                 // by ring position
  double coef[kMaxM];                 // zeta - eta by ring position
};

// Preconditioned CG on A_free (3 right-hand sides solved in lockstep), the
// solve used for meshes too large to factor (configs[4]).
// PCG kernel shapes: SpMV = one warp per 32-row slice, grid-stride over slices;
// the vector update = one thread per (row, coordinate), grid-stride with a
// stride that is a multiple of 3 so a thread keeps its coordinate.
constexpr int kSpmvThreads = 256, kSpmvWarps = kSpmvThreads / 32, kSpmvBlocksPerSm = 4;
constexpr int kUpdThreads = 384, kUpdBlocksPerSm = 3;


// A sparse matrix as SELL-32 on the device (see SysView::sell_* below)
struct SellDev {
  const int64_t* ptr;  // [nslice + 1]
  const int32_t* col;
  const double* val;
  int32_t nslice, nrows;
};

// SELL-32 with fp32 coefficients: the AMG V-cycle operators.  The cycle is
// only the CG preconditioner, so rounding its coefficients changes the
// (still fixed, symmetric) preconditioner, not the system CG solves to 1e-10.
struct SellDevF {
  const int64_t* ptr;   // SELL: [nslice + 1] slice offsets; CSR (kl > 0): [nrows + 1] row offsets
  const int32_t* col;
  const float* val;
  int32_t nslice, nrows;
  int32_t kl;           // 0 = SELL-32 (lane per row); K = CSR with K lanes per row
  int32_t nblk;         // grid of the kernels applying this operator
};

// One level of the AMG V-cycle (solver QN_SOLVE_AMG; n_inst == 1)
struct AmgDevLevel {
  SellDevF A, P, R;     // operator (n x n), prolongator (n x n_coarse), restriction (n_coarse x n)
  const double* dinv;   // [n]
  // V-cycle vectors: fp32, one 16-byte (x, y, z, 0) entry per row, so the column gather of every
  // operator product is ONE 128-bit load per matrix entry (the cycle is a preconditioner: the CG
  // recurrences, its residual and the convergence test stay fp64)
  float4* xf;           // [n] pre-smoothed (+ prolonged) iterate
  float4* rf;           // [n] residual after pre-smoothing
  float4* bf;           // [n] right-hand side, levels >= 1
  float4* tf;           // [n] post-smoothed result, levels >= 1
  double* t;            // level 0: z [n][3]
  double* b;            // level 0: the CG residual [n][3]
  double omega;         // Jacobi weight 4 / (3 rho(D^-1 A))
  int32_t n, nblk;      // rows, grid of the level's SELL kernels
};

struct PcgCtl {
  double rz[3], alpha[3], beta[3], bb[3], rr[3];
  int32_t iter, conv, total, pad1;  // conv: bit c = column c converged; total: CG iterations this frame
};

struct DevConfig {
  int32_t kind, iterations, m, line_search;
  double gamma, alpha_init, shrink, grad_tol;
  int32_t has_targets, use_graph, max_passes, cheb_S;
  double cheb_rho;
  int32_t lbfgs_init, fault;  // fault: test-only injection, mode | (first iteration << 4)
};

struct SysView {
  int32_t n, mt, n_inst, n_mat, n_fixed, nblk_v, nblk_t, rec_cap;
  int32_t vt, pad_vt;     // vertex-kernel block size (kVertexThreads or kVertexThreadsMax)
  int32_t spring, aniso;  // elements are edge springs (a, b, -1, -1), vols = rest lengths; fibre materials present
  int32_t f32, pad_f;     // optional fp32 element pass (VL tets; fp64 storage, gather and reductions)
  double h;
  double grav[3];
  const int4* tets;
  const double* dminv;  // SoA [9][mt]
  const double* vols;
  const int32_t* tet_mat;
  const qn_material* mats;
  const double* masses;
  const double* w_in;        // masses / h^2 (dynamics.py:472), precomputed on the host
  const uint8_t* is_fixed;
  const int32_t* fixed_pos;  // vertex -> index into the fixed list, -1 if free
  const int32_t* v2e_ptr;
  const int32_t* v2e;        // slots 4 t + c, increasing
  const int32_t* slot_pos;   // [4 mt] gather position of slot 4 t + c (forces are stored in v2e order), -1 if absent
  const int32_t* fact_vtx;   // factor row -> vertex
  double* q_l;
  double* q_prev;
  double* y;
  double* X;       // [3][inst][n][3]
  double* Gr;      // [2][inst][n][3]
  double* S;       // [kMaxM+1][inst][n][3]
  double* T;
  double* R0;      // [inst][n][3]
  double* qf;      // [inst][n_free][3] solve right-hand side in factor order (direct solver, non-batched)
  double* D;       // [inst][n][3]
  double* forces;  // [inst][4 mt][3] corner forces in gather (v2e) order
  const double* targets;  // [inst][n_fixed][3]
  double* part_v;  // [inst][nblk_v][kNG]
  double* part_t;  // [inst][nblk_t]
  unsigned* cnt;   // [4][inst] last-block counters + [global]
  InstCtl* ctl;
  const DevConfig* cfg;
  double* rec_g;          // the record arrays are sub-ranges of one allocation (one D2H per frame):
  int32_t* rec_trials;    // [g | alpha | ms : ni x cap doubles][g0 : ni doubles][trials : ni x cap int32]
  double* rec_alpha;      // [status | fallbacks : ni int32 each]
  double* rec_ms;
  double* rec_g0;         // filled by k_finish from the control blocks
  int32_t* rec_status;
  int32_t* rec_fb;
  int32_t* active;     // instances not yet done
  unsigned long long* passes;
  unsigned long long* ktl;  // diagnostics timeline [kTimelinePasses][kTimelineKernels][2] ns, or null
  cudaGraphConditionalHandle handle;
  // ---- PCG solve mode (pcg: 0 = direct, 1 = Jacobi-PCG, 2 = AMG-PCG) ----
  int32_t pcg, n_free, nblk_p, pcg_maxit;
  int32_t nslice, nblk_spmv, nblk_upd, pad_p;
  double pcg_tol;
  // A_free (free-vertex order) as SELL-32: slice s holds rows 32s..32s+31,
  // entry k of lane l at sell_ptr[s] + 32k + l (zero-padded to the slice's
  // longest row), so every warp load of the matrix is coalesced
  const int64_t* sell_ptr;  // [nslice + 1]
  const int32_t* sell_col;
  const double* sell_val;   // [inst][sell_ptr[nslice]]
  int64_t sell_nnz;
  const double* dinv;     // [inst][n_free] Jacobi preconditioner
  double* px;             // [inst][n_free][3] iterate
  double* pr;             // residual (z = dinv r is recomputed where needed)
  double* pp;             // [2][inst][n_free][3] search directions (double buffered)
  double* pq;             // A p
  double* part_p;         // [inst][max(nblk_p, nblk_spmv, nblk_upd)][8]
  unsigned* cnt_p;        // [4][inst] (init, spmv, update, rz) + [global]
  PcgCtl* pctl;           // [inst]
  int32_t* pcg_active;    // instances still iterating
  cudaGraphConditionalHandle pcg_handle;
  // ---- AMG-preconditioned CG (pcg == 2) ----
  int32_t amg_levels, ncoarse;
  const AmgDevLevel* alev;  // [amg_levels] (device)
  const float* cinv;        // dense inverse of the coarsest operator [ncoarse][ncoarse], fp32 (preconditioner only)
  double* pz;               // z = B r (the V-cycle output on level 0)
  unsigned* amg_bar;        // grid barrier of k_amg_tail: [0] arrivals (monotonic), [1] count at kernel entry
  float4* pzf;              // single-system AMG: z rounded to fp32 rows of 16 B (replaces pz; null: fp64 pz)
  // ---- colliders (dynamics.py:199-285, 446-457, 486-516) ----
  int32_t n_col, nblk_c;
  double w_col;
  const qn_collider* cols;  // [n_col]
  uint8_t* col_act;         // [inst][n][n_col] active constraint of (vertex, collider)
  double* col_t;            // [inst][n][n_col][3] surface point
  double* col_n;            // [inst][n][n_col][3] outward normal
  double* col_g;            // [inst][n][3] collision gradient at the current iterate
  double* part_c;           // [inst][nblk_c]
  unsigned* cnt_c;          // [inst]
  // ---- lbfgs_init = rest_pose_hessian (solvers.py:142-146, 401-407) ----
  int32_t nf3, pad_r;       // free dofs
  const int32_t* free3;     // [nf3] dof = 3 vertex + coordinate
  const double* hrest_inv;  // [nf3][nf3] inverse of the rest-pose Hessian (dense, symmetric)
  double* qbuf;             // [nf3] first-loop vector q on the free dofs
};

}  // namespace qn

struct qn_system {
  int64_t n = 0, mt = 0, n_inst = 1, n_mat = 1, n_fixed = 0, n_free = 0;
  double h = 0, grav[3] = {0, 0, 0}, scale = 1, max_mass = 0;
  qn_factor* factor = nullptr;
  cudaStream_t stream = nullptr;
  // device buffers (owned)
  std::vector<void*> allocs;
  qn::SysView v{};
  qn::DevConfig* d_cfg = nullptr;
  qn::DevConfig h_cfg{};
  double* d_targets = nullptr;
  int rec_cap = 0;
  // pinned host staging
  double* h_stage = nullptr;
  void* h_rec = nullptr;  // pinned mirror of the packed record arrays
  size_t rec_bytes = 0;
  size_t h_stage_bytes = 0;
  // graph
  bool use_graph = true;
  bool pdl = false;  // programmatic dependent launch between the body kernels (QN_PDL=1; measured neutral inside the frame graph)
  int32_t fault = 0;  // qn_system_set_fault
  int graph_m_bound = 0;  // history bound the captured graph's kernels are specialised on
  int graph_init = 0;     // lbfgs_init the captured graph's direction step was built for
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int64_t last_passes = 0;
  int64_t kernels_per_pass = 0, kernels_per_cg = 0;  // kernel nodes of the captured frame graph
  bool pcg_rec = false;  // AMG-PCG SpMV in recurrence form (k_pcg_spmv_rec)
  int amg_tail_level = 0, amg_tail_grid = 0;  // V-cycle levels >= amg_tail_level run in one kernel (0: none)
  // element-seam workspace
  double* d_part_plain = nullptr;
  double* scratch[3] = {nullptr, nullptr, nullptr};  // n x 3 vectors of the objective / elements seams
  std::vector<int32_t> h_tet_mat;
  // AMG (host copy of the level table, for launch sizes and diagnostics)
  std::vector<qn::AmgDevLevel> h_alev;
  std::vector<int64_t> amg_nnz;  // per level: nnz(A), nnz(P), nnz(R) of the host hierarchy
  double amg_setup_s = 0.0;
};

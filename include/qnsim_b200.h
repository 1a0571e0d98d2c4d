/*
 * qnsim_b200 — C-ABI of the B200 (sm_100a) per-timestep quasi-Newton / L-BFGS
 * hyperelastic solver (arXiv 1604.07378).  Plain pointers and sizes only.
 *
 * The reference (`/root/reference/pkg/src/qnsim`, pure Python) has no FFI; each
 * entry point below replaces one reference call site, cited as file:line.  The
 * Python host package `paper_1604_07378_b200` binds these through ctypes
 * (`_lib.py`); INTEGRATION.md shows the binding a qnsim maintainer would add.
 *
 * Conventions
 *   - every function returns QN_OK (0) or a QN_ERR_* code; qn_last_error()
 *     returns a message for the calling thread's last failure;
 *   - arrays are C-contiguous row-major, float64 unless stated (int32 indices);
 *   - `mem` selects where caller buffers live: QN_MEM_HOST (pageable or pinned
 *     host memory; pageable inputs are staged through the library's own
 *     pinned buffer, page-locked ones are copied by DMA directly) or
 *     QN_MEM_DEVICE (device pointers on the current CUDA device);
 *   - `stream` is a cudaStream_t (NULL = the library's own stream); every call
 *     is stream-ordered and the call returns after the stream work completes
 *     unless stated otherwise.
 */
#ifndef QNSIM_B200_H
#define QNSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QN_OK 0
#define QN_ERR_ARG 1          /* bad argument (shape, range, null)            */
#define QN_ERR_CUDA 2         /* CUDA runtime failure                         */
#define QN_ERR_NOT_SPD 3      /* FactorizationError (linalg.py:20-21,31-34)   */
#define QN_ERR_ALLOC 4        /* device or host allocation failed             */
#define QN_ERR_ASCENT 5       /* SolverError: non-descent direction (solvers.py:244-246) */
#define QN_ERR_UNSUPPORTED 6  /* option outside the B200 hot path             */

#define QN_MEM_HOST 0
#define QN_MEM_DEVICE 1

/* Valanis-Landel scalar-function kinds (materials.py:32-133) */
#define QN_FN_ZERO 0
#define QN_FN_POLY 1
#define QN_FN_LOG 2
#define QN_FN_HERMITE 3
#define QN_FN_SQDEV 4    /* c[0] (x - c[1])^2: the ARAP tet energy (w/2)||F - R||^2 = vol k/2 sum (s_i - 1)^2
                            of dynamics.ARAPGroup (dynamics.py:73-108) as a Valanis-Landel a(x) */
#define QN_FN_ANISO 5    /* material a of an anisotropic-fibre element (dynamics.AnisoGroup,
                            dynamics.py:154-193): c[0..2] = unit fibre d, c[3] = kappa;
                            energy vol kappa/2 (|F d| - 1)^2, no SVD                    */

#define QN_MAX_COEF 12   /* polynomial coefficients (ascending)  */
#define QN_MAX_KNOTS 12  /* cubic Hermite control points          */
#define QN_MAX_M 16      /* L-BFGS history window                 */

/* One univariate function a, b or c of Psi = sum a(si) + sum b(si sj) + c(s1 s2 s3). */
typedef struct qn_scalar_fn {
  int32_t kind;                 /* QN_FN_*                                        */
  int32_t n;                    /* poly: #coefficients; hermite: #knots            */
  double c[QN_MAX_COEF];        /* poly: ascending coefficients (PolyFn, :40-51)  */
  double dc[QN_MAX_COEF];       /* poly: polyder(c), n-1 entries                   */
  double xs[QN_MAX_KNOTS];      /* hermite knots, strictly increasing (:83-133)   */
  double ys[QN_MAX_KNOTS];
  double ts[QN_MAX_KNOTS];
  double alpha, beta, eps;      /* log: alpha ln x + beta/2 ln^2 x, x > eps (:54-80) */
  double f0, f1, f2;            /* log: value/slope/curvature at eps (Taylor)    */
} qn_scalar_fn;

/* MaterialModel (materials.py:146-159): shift = 3a(1) + 3b(1) + c(1). */
typedef struct qn_material {
  qn_scalar_fn a, b, c;
  double shift;
} qn_material;

/* Collider (dynamics.py:199-270): keeps vertices outside a solid.  Penalty
 * w_col (depth . n)^2 per active constraint (dynamics.py:446-457), active set
 * rebuilt at the start of every iteration (update_collisions, :486-516). */
#define QN_COL_HALFSPACE 0  /* p = point, n = unit normal                 */
#define QN_COL_SPHERE 1     /* p = center, r0 = radius                    */
#define QN_COL_TORUS 2      /* p = center, r0 = major, r1 = minor radius  */
#define QN_MAX_COLLIDERS 4
typedef struct qn_collider {
  int32_t kind, pad;
  double p[3], n[3];
  double r0, r1;
} qn_collider;

/* ------------------------------------------------------------------------ */
/* library                                                                  */

const char* qn_last_error(void);
int qn_version(void);
/* number of CUDA devices visible; 0 without a GPU (no compute calls then) */
int qn_device_count(int32_t* count);
/* kernels launched by this library since load (for launch-count evidence) */
int qn_launch_count(int64_t* count);

/* ------------------------------------------------------------------------ */
/* rotation-variant 3x3 SVD — replaces linalg.svd_rv_batch (linalg.py:86-110)
 * F: (m,3,3); U, V: (m,3,3) proper rotations; sigma: (m,3), s0 >= s1 >= |s2|,
 * s2 < 0 iff det F < 0, |s| < 1e-10 clamped to +-1e-10. */
int qn_svd_rv_batch(int64_t m, const double* F, double* U, double* sigma, double* V, int32_t mem,
                    void* stream);

/* ------------------------------------------------------------------------ */
/* material point evaluation — replaces vl_energy_batch / vl_stress_batch
 * (materials.py:181-207) on the device.  sigma: (k,3) -> psi (k), tau (k,3). */
int qn_material_eval(const qn_material* mat, int64_t k, const double* sigma, double* psi, double* tau,
                     int32_t mem, void* stream);

/* ------------------------------------------------------------------------ */
/* Prefactored SPD solve — replaces linalg.Factorization / factorize_spd /
 * solve_prefactored (linalg.py:23-59) and the dense cho_factor of
 * dynamics.py:413-414.  Supernodal Cholesky (host, geometric nested
 * dissection on `coords`) + level-free dependency-driven supernodal
 * triangular solves on the device.  A: symmetric CSR (both triangles),
 * `nbatch` numeric instances sharing one pattern (values: nbatch x nnz). */
typedef struct qn_factor qn_factor;

typedef struct qn_factor_info {
  int64_t n, nnz_a, nnz_l, n_supernodes, max_front, tree_depth, nbatch;
  double factor_seconds, flops;
  int64_t dense_top;  /* columns solved by the dense top block S^-1 (0 = none) */
  int64_t nnz_l_sparse; /* entries of L in the supernodes solved by the sparse sweeps (not the dense top) */
  int64_t sinv_stored;  /* entries of S^-1 the top apply reads (lower-triangle tiles, padded) */
} qn_factor_info;

int qn_factor_create(int64_t n, const int64_t* indptr, const int32_t* indices, const double* values,
                     int64_t nbatch, const double* coords, qn_factor** out);
int qn_factor_info_get(const qn_factor* f, qn_factor_info* info);
/* X = A^-1 B for instance `batch`; B, X: (n, nrhs) row-major */
int qn_factor_solve(qn_factor* f, int64_t batch, const double* B, double* X, int64_t nrhs, int32_t mem,
                    void* stream);
int qn_factor_destroy(qn_factor* f);
/* diagnostics: one traced solve (instance 0, current staging RHS); stamps =
 * globaltimer ns at (ticket taken, staging issued, dependencies ready), then
 * SM clock64 at (ready, data staged, computed, published) per forward then
 * backward work item; tasks = {supernode, lo, hi, 0} per forward then
 * backward task.  Sizes: 7 (n_ftask + n_btask) nbatch and 4 (n_ftask + n_btask). */
int qn_factor_task_counts(const qn_factor* f, int64_t* n_ftask, int64_t* n_btask);
int qn_factor_trace_solve(qn_factor* f, uint64_t* stamps, int32_t* tasks);

/* ------------------------------------------------------------------------ */
/* Device setup assembly — replaces the numpy part of dynamics.build_system
 * (dynamics.py:351-414) with mesh.tet_diff_operators (mesh.py:200-216) and
 * mesh.lumped_masses (mesh.py:178-197) for tet meshes: per tet G (m x 4 x 3)
 * and rest volume, lumped vertex masses, L = sum w G G^T (w = vol k_of_tet)
 * as CSR with sorted columns, and A_free = (L + M/h^2)[free][:, free].
 * Tets with volume < vol_eps raise QN_ERR_ARG (MeshError in the reference).
 * Summation orders are the reference's (masses corner-major then element
 * order, L entries in element order); the 3x3 inverse is the adjugate, so
 * values agree with the reference to rounding.  qn_setup_copy writes host
 * arrays (any pointer may be NULL to skip that output). */
typedef struct qn_setup qn_setup;
int qn_setup_create(int64_t n, const double* verts, int64_t m, const int32_t* tets, double density,
                    const double* k_of_tet, double h, int64_t n_fixed, const int32_t* fixed, double vol_eps,
                    qn_setup** out);
int qn_setup_sizes(const qn_setup* s, int64_t* nnz_l, int64_t* n_free, int64_t* nnz_a);
int qn_setup_copy(const qn_setup* s, double* G, double* vols, double* masses, int64_t* l_indptr,
                  int32_t* l_indices, double* l_values, int64_t* a_indptr, int32_t* a_indices,
                  double* a_values);
int qn_setup_destroy(qn_setup* s);

/* ------------------------------------------------------------------------ */
/* Simulation system — replaces dynamics.build_system (dynamics.py:351-434)
 * for Valanis-Landel tet groups, plus the per-frame solver
 * solvers.simulate_frame (solvers.py:260-352).  `n_inst` independent
 * instances share one mesh (topology, rest shape, fixed set) and may differ in
 * material and in the numeric factor (configs[3] batch); n_inst = 1 is a
 * plain SimSystem. */
typedef struct qn_system qn_system;

typedef struct qn_system_desc {
  int64_t n_verts;            /* n                                              */
  int64_t n_tets;             /* m (may be 0: no elastic groups)                */
  int64_t n_inst;             /* instances (>= 1)                               */
  int64_t n_mat;              /* materials per instance (VL groups)             */
  const int32_t* tets;        /* (m,4), group-major order (dynamics.py:332-348) */
  const double* Dm_inv;       /* (m,3,3): G[:,1:] of mesh.tet_diff_operators    */
  const double* vols;         /* (m)                                            */
  const int32_t* tet_mat;     /* (m) material index in [0,n_mat) or NULL        */
  const qn_material* mats;    /* (n_inst * n_mat)                               */
  const double* masses;       /* (n) lumped masses (mesh.py:178-197)            */
  int64_t n_fixed;
  const int32_t* fixed;       /* sorted fixed vertex ids                        */
  double h;
  double gravity[3];
  double scale;               /* rest bbox diagonal (dynamics.py:416-417)      */
  /* A_free = (L + M/h^2)[free][free], CSR over free rows, values per instance */
  int64_t a_nnz;
  const int64_t* a_indptr;    /* (n_free+1)                                     */
  const int32_t* a_indices;   /* (a_nnz)                                        */
  const double* a_values;     /* (n_inst * a_nnz)                               */
  const double* free_coords;  /* (n_free,3) rest positions for the ordering     */
  /* solve of A_free d = q: QN_SOLVE_DIRECT (prefactored, linalg.py:23-59) or
   * QN_SOLVE_PCG (Jacobi-preconditioned CG to ||r|| <= pcg_tol ||b|| per
   * coordinate, for meshes too large to factor; configs[4]) */
  int32_t solver;
  int32_t pcg_maxit;
  double pcg_tol;
  /* colliders (shared by all instances); w_col = collision_weight or 10 max w */
  int64_t n_colliders;        /* <= QN_MAX_COLLIDERS                             */
  const qn_collider* colliders;
  double w_col;
  /* QN_ELEM_TET (default) or QN_ELEM_SPRING: spring networks (SpringGroup,
   * dynamics.py:111-151): tets rows are (a, b, -1, -1), vols = rest lengths,
   * Dm_inv unused, material a.c[0] = k (PDMaterial mass_spring)          */
  int32_t element_kind;
  int32_t pad_e;
  int64_t dminv_stride;       /* doubles between consecutive tets' Dm_inv (0 = 9; 12 when Dm_inv points
                                 at row 1 of a full (m,4,3) G array)          */
} qn_system_desc;

#define QN_ELEM_TET 0
#define QN_ELEM_SPRING 1

#define QN_SOLVE_DIRECT 0
#define QN_SOLVE_PCG 1
#define QN_SOLVE_AMG 2  /* CG preconditioned by a smoothed-aggregation AMG V(1,1) cycle (single instance) */

typedef struct qn_solver_config {  /* SolverConfig (solvers.py:43-68)          */
  int32_t kind;                    /* 0 = pd_qn, 1 = lbfgs (lbfgs_init=system_matrix),
                                      2 = chebyshev (solvers.py:154-164, 306-311) */
  int32_t iterations;
  int32_t m;
  int32_t line_search;
  double gamma, alpha_init, alpha_shrink;
  double rho;                      /* chebyshev: spectral radius estimate         */
  int32_t S;                       /* chebyshev: iterations before acceleration   */
  int32_t lbfgs_init;              /* lbfgs: 0 = system_matrix (A^-1), 1 = scaled_identity
                                      (rho/<t,t> of the newest pair, solvers.py:136-141),
                                      2 = rest_pose_hessian (qn_system_rest_hessian first) */
} qn_solver_config;

typedef struct qn_frame_record {   /* ConvergenceRecord (solvers.py:71-80), per instance */
  double* g0;        /* (n_inst)                 */
  double* g;         /* (n_inst, iterations)     */
  int32_t* ls_trials;/* (n_inst, iterations)     */
  double* alphas;    /* (n_inst, iterations)     */
  double* cum_ms;    /* (n_inst, iterations)     */
  int32_t* status;   /* (n_inst): bit0 stagnated, bit1 ascent error */
  int32_t* fallbacks;/* (n_inst) or NULL: chebyshev non-descent fallbacks (rec.fallbacks) */
} qn_frame_record;

int qn_system_create(const qn_system_desc* desc, qn_system** out);
int qn_system_destroy(qn_system* s);
int qn_system_factor(qn_system* s, qn_factor** out);  /* borrowed handle */

/* Device-resident state (SimState q_l / q_prev, dynamics.py:314-329), (n_inst,n,3). */
int qn_state_set(qn_system* s, const double* q_l, const double* q_prev, int32_t mem, void* stream);
int qn_state_get(qn_system* s, double* q_l, double* q_prev, double* y, int32_t mem, void* stream);

/* Advance the resident state one frame: y = inertia target, minimise g(x) by
 * `cfg`, then q_prev <- q_l, q_l <- x.  fixed_targets: (n_inst, n_fixed, 3) or
 * NULL (= q_l rows, dynamics.py:441-442).  rec: NULL or output record
 * (host pointers if mem == QN_MEM_HOST).  sync = 0 returns without waiting
 * (record then must be NULL).  Whole frame = one CUDA-graph launch. */
int qn_frame_step(qn_system* s, const qn_solver_config* cfg, const double* fixed_targets,
                  qn_frame_record* rec, int32_t mem, int32_t sync, void* stream);

/* Stateless wrapper = simulate_frame(system, state, config, fixed_targets):
 * uploads q_l/q_prev, steps, downloads x (next q_l) and y. */
int qn_simulate_frame(qn_system* s, const qn_solver_config* cfg, const double* q_l, const double* q_prev,
                      const double* fixed_targets, double* x_out, double* y_out, qn_frame_record* rec,
                      int32_t mem, void* stream);

/* objective g(x) and gradient (dynamics.py:460-478) at x for target y,
 * per instance: g_out (n_inst), grad_out (n_inst,n,3) or NULL. */
int qn_system_objective(qn_system* s, const double* x, const double* y, double* g_out, double* grad_out,
                        int32_t mem, void* stream);

/* Element-group seam (dynamics.VLGroup.energy / add_gradient, :57-67):
 * energy of the tets of material group `mat` of instance `inst` (all tets if
 * mat < 0) and their corner forces scattered, element-major, into out. */
int qn_system_elements(qn_system* s, int64_t inst, int64_t mat, const double* x, double* energy,
                       double* grad_accum, int32_t mem, void* stream);

/* Optional fp32 element pass (configs[2] "optional fp32 run"; tolerance 1e-4
 * on positions): the per-tet SVD / material / PK1 math in single precision,
 * positions, forces, gather, L-BFGS and the solve stay fp64.  VL / ARAP tets. */
int qn_system_set_precision(qn_system* s, int32_t fp32);
/* Execution mode for debugging: 1 = CUDA graph with conditional nodes
 * (default), 0 = host-driven loop (one host sync per line-search trial). */
int qn_system_set_graph_mode(qn_system* s, int32_t use_graph);
/* Device-only records of the last qn_frame_step, enqueued on `stream` (no host
 * sync, for the torch op boundary): g_out[b][k] = per-iteration objective
 * (rec.g, solvers.py:71-80) of instance b for k < iterations, and
 * status_out[b] = bit 0 stagnated, bit 1 ascent (SolverError); both device
 * pointers. */
int qn_frame_records_device(qn_system* s, int32_t iterations, double* g_out, int32_t* status_out, void* stream);
/* device time (ms) of the last qn_frame_step measured with CUDA events */
int qn_system_last_frame_ms(qn_system* s, double* ms);
/* body passes (line-search trials + re-evaluations) of the last frame */
int qn_system_last_frame_passes(qn_system* s, int64_t* passes);
/* diagnostics: per body pass, globaltimer ns at the entry of block 0 and at
 * the end of the finalising block / last CTA of k_grad, k_eta, k_vec (entry
 * only), k_tet, sptrsv_forward, sptrsv_backward; out = [512 passes][6
 * kernels][2] (0 = not reached).  Enabling rebuilds the frame graph. */
int qn_system_set_timeline(qn_system* s, int32_t enable);
/* Test-only fault injection into the device line search, from L-BFGS iteration
 * `iteration` (1-based) on: mode 1 negates the direction (slope >= 0, the
 * ascent -> SolverError branch of solvers.py:244-246); mode 2 steps along -d
 * while the Armijo test uses the slope of d (every trial increases g: the
 * StagnationError branch, solvers.py:250-252 and the record padding of
 * :329-336, as pkg/tests/test_solvers.py:318-337 provoke on the host).
 * mode 0 = off (the default). */
int qn_system_set_fault(qn_system* s, int32_t mode, int32_t iteration);
int qn_system_timeline(qn_system* s, uint64_t* out, int64_t cap);
/* diagnostics: task trace of the last in-graph solve (direct solver, timeline
 * enabled), same layout as qn_factor_trace_solve */
int qn_system_solve_trace(qn_system* s, uint64_t* stamps, int32_t* tasks);
/* PCG mode: conjugate-gradient iterations of the last frame, summed over
 * instances (0 in direct mode) */
int qn_system_last_frame_cg_iterations(qn_system* s, int64_t* iters);
/* AMG systems: out = [levels, rows of level 0..levels-1, setup ms]; cap >= 12 */
int qn_system_amg_info(qn_system* s, int64_t* out, int64_t cap);

/* Stand-alone timing of one hot kernel with CUDA events on `stream` (after a
 * warm-up launch), over every instance: kernel 0 = per-tet pass at the
 * resident q_l, kernel 1 = forward + backward supernodal solve (3 RHS),
 * kernel 2 = the CG's SpMV q = A_free x (PCG / AMG systems).  avg_ms = mean
 * launch time. */
int qn_system_time_kernel(qn_system* s, int32_t kernel, int32_t reps, double* avg_ms, void* stream);

/* Newton direction (solvers.py:167-234): d = -H^-1 g on the free dofs, H =
 * sum of per-element central-difference Hessian blocks of the corner forces
 * (step = fd step, e.g. 1e-6 scale) with eigenvalues clamped at eig_floor
 * (project_psd) + M/h^2, dense, Cholesky-factored (QN_ERR_NOT_SPD when not
 * SPD).  x, grad, d: (n,3); fixed rows of d are zero.  Single instance, no
 * colliders; for the small meshes the reference runs Newton on. */
int qn_newton_direction(qn_system* s, const double* x, const double* grad, double step, double eig_floor, double* d,
                        int32_t mem, void* stream);
/* lbfgs_init = "rest_pose_hessian" (solvers.py:142-146, 401-407): the Newton
 * Hessian at the rest positions `rest` (n,3) (y = rest), factored and inverted
 * once on the device; frames with that init then apply the dense inverse in
 * their direction step.  Single instance, <= 20000 free dofs. */
int qn_system_rest_hessian(qn_system* s, const double* rest, double step, double eig_floor);
/* free the Newton workspace of a system (also freed with the process) */
int qn_newton_release(qn_system* s);

/* Slab decomposition of one mesh across ranks (configs[4]):
 * the per-rank stages of simulate_frame (solvers.py:260-352) with the
 * reference's gradient (dynamics.py:470-478), objective (:460-467),
 * two-loop direction (solvers.py:120-151) with A_free solved by CG, and the
 * Armijo trial (:241-257).  The reference is single-process; these entry
 * points are new API under the same semantics.  A rank owns a contiguous
 * range of its local vertices and a suffix of its local tets; `local` is a
 * qn_system built (QN_SOLVE_PCG or QN_SOLVE_AMG) on the rank's own plus
 * ghost cells with the ghost and pinned vertices as its fixed set, so its
 * free rows are the owned free vertices and its A_free (= the preconditioner
 * block) is A restricted to them.  Each stage writes this rank's
 * fixed-order partial sums to the SEND buffer; the host all-gathers SEND into
 * every rank's GATHER buffer ([n_ranks][32]) and exchanges the boundary
 * planes of P / R0 between neighbours before the stages that read them. */
typedef struct qn_slab qn_slab;

typedef struct qn_slab_desc {
  qn_system* local;        /* borrowed; must outlive the slab                  */
  int64_t own_lo, own_hi;  /* owned local vertex range                         */
  int64_t tet_own_lo;      /* local tets [tet_own_lo, m) count in the energy   */
  const uint8_t* pinned;   /* (n) reference fixed vertices (gradient rows 0)   */
  /* A = L + M/h^2 on the owned free rows (local free order), columns = local
   * vertex ids of the non-pinned vertices (ghost columns included)          */
  int64_t a_nnz;
  const int64_t* a_indptr;
  const int32_t* a_indices;
  const double* a_values;
  int32_t n_ranks;
  int32_t pcg_maxit;
  double pcg_tol;          /* ||r|| <= pcg_tol ||b|| per coordinate           */
} qn_slab_desc;

#define QN_SLAB_SEND 0      /* [32] this rank's partial sums of the last stage   */
#define QN_SLAB_GATHER 1    /* [n_ranks][32] all-gathered SEND                   */
#define QN_SLAB_P 2         /* (n,3) CG search vector, vertex layout (halo)      */
#define QN_SLAB_R0 3        /* (n,3) A_free^-1 q, vertex layout (halo)           */
#define QN_SLAB_QL 4        /* (n,3) state q_l                                   */
#define QN_SLAB_QPREV 5     /* (n,3) state q_prev                                */
#define QN_SLAB_Y 6         /* (n,3) inertia target                              */
#define QN_SLAB_X 7         /* (2,n,3) current / trial iterate                   */
#define QN_SLAB_G 8         /* (n,3) gradient (owned rows complete)              */
#define QN_SLAB_CSEND 9     /* (nc,3) this rank's P_c^T r (coarse correction)     */
#define QN_SLAB_CGATHER 10  /* [n_ranks](nc,3) all-gathered CSEND                 */

#define QN_SLAB_INIT 0        /* y, x = y                                          */
#define QN_SLAB_EVAL 1        /* objective at X[xs]: SEND[0] elastic, [1] inertia sum m|x-y|^2 */
#define QN_SLAB_GRAD 2        /* gradient at X[xs], L-BFGS pair, dots (see qn_slab.cu) */
#define QN_SLAB_PCG_SETUP 3   /* q = -g - sum zeta t, CG start; SEND [bb, rz]     */
#define QN_SLAB_PCG_P 4       /* p = z + beta p from GATHER (first: [bb, rz], else [rr, rz]) */
#define QN_SLAB_PCG_SPMV 5    /* q = A p; SEND [pq]                                */
#define QN_SLAB_PCG_UPDATE 6  /* x += alpha p, r -= alpha q, z = B r; SEND [rr, rz] */
#define QN_SLAB_STORE 7       /* R0 = CG solution in vertex layout                 */
#define QN_SLAB_ETA 8         /* SEND[j] = <t_j, r0>                               */
#define QN_SLAB_DIR 9         /* d = r0 + sum (zeta - eta) s; SEND[0] = <g, d>     */
#define QN_SLAB_TRIAL 10      /* X[xs_to] = X[xs] + alpha d                        */
#define QN_SLAB_FINISH 11     /* q_prev <- q_l, q_l <- X[xs]                       */
#define QN_SLAB_PCG_RZ 12     /* SEND[3..5] = <r, z> after the preconditioner      */
#define QN_SLAB_COARSE_R 13   /* CSEND = P_c^T r                                   */
#define QN_SLAB_COARSE_APPLY 14 /* z += P_c A_c^-1 (sum over ranks of CGATHER)     */

int qn_slab_create(const qn_slab_desc* d, qn_slab** out);
int qn_slab_destroy(qn_slab* s);
int qn_slab_buffer(qn_slab* s, int32_t which, void** ptr, int64_t* count);
/* args (doubles): [xs, xs_to, have_prev, new_slot, nring, first, alpha,
 * ring[9] (slot ids oldest -> newest), coef[9]]; asynchronous on `stream` */
int qn_slab_stage(qn_slab* s, int32_t stage, const double* args, int32_t nargs, void* stream);
/* Two-level preconditioner z = B_slab r + P_c A_c^-1 P_c^T r for a grid bar
 * (grid = cells per dimension, vertex id (i (ny+1) + j)(nz+1) + k): P_c = the
 * trilinear hat functions of a coarse grid (coarse_dims nodes per dimension),
 * given per dimension d and fine index i by hat_first (first coarse node of
 * its cell) and hat_w (weights of that node and the next), concatenated over
 * d = x, y, z; node_pos = fine index of each coarse node (concatenated).  The
 * rank owns the x-planes [i_lo, i_lo + n_planes); v0 = global id of its
 * local vertex 0; cinv = A_c^-1 (nc x nc, identical on every rank). */
int qn_slab_set_coarse(qn_slab* s, const int32_t* grid, const int32_t* coarse_dims, int64_t v0, int64_t i_lo,
                       int64_t n_planes, const int32_t* hat_first, const double* hat_w, const int32_t* node_pos,
                       const double* cinv);
/* CG status after the last update (synchronises `stream`): conv bits (bit 3 =
 * finished), CG iterations of the current solve */
int qn_slab_pcg_status(qn_slab* s, int32_t* conv, int32_t* iters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QNSIM_B200_H */

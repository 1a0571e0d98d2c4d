// Per-frame quasi-Newton / L-BFGS solver on the device (solvers.py:260-352).
//
// One frame = one CUDA graph: [init] -> WHILE(any instance active){ body } -> [finish].
// The body is six kernels; every instance advances one step of its phase
// machine (qn_system.h) per body pass, so batched instances with different
// line-search trial counts proceed independently and the host never syncs
// inside a frame:
//   k_grad   (PH_GRAD)   gradient gather (inertia + corner forces in the
//                        reference's element order, fixed rows zeroed),
//                        L-BFGS push dots + Gram entries + <s_i, g>, then the
//                        last block finalises: curvature guard, ring update,
//                        ||g|| early-out, zeta recursion.
//   fwd/bwd  (PH_DIR)    supernodal solves r0 = A^-1 q', q' = -g - sum zeta t
//                        formed on the fly (qn_sptrsv.cuh).
//   k_eta    (PH_DIR)    <t_i, r0>, then eta recursion -> coef = zeta - eta.
//   k_vec    (PH_DIR)    d = r0 + sum coef s, slope partials, first trial x + a1 d
//            (PH_ALPHA)  trial x + alpha d;  all eval phases: inertia partials.
//   k_tet    (eval)      per-tet F, SVD, VL energy + PK1 corner forces; the last
//                        block per instance finalises: Armijo / early-outs /
//                        stagnation / records; the last block overall sets
//                        the WHILE condition.
//
// The L-BFGS two-loop (solvers.py:120-151) is evaluated with the Gram-matrix
// form of the same recursion: zeta_i = (<s_i, q> - sum_{j newer} zeta_j <s_i, t_j>)/rho_i
// and eta_i = (<t_i, r0> + sum_{j older} (zeta_j - eta_j) <s_j, t_i>)/rho_i,
// which needs one batched reduction per loop instead of one per pair; the
// vector updates q -= zeta t and r += s (zeta - eta) are applied in the
// reference's order with the reference's rounding (mul, then add).
#include <cstring>
#include <mutex>

#include "qn_common.cuh"
#include "qn_element.cuh"
#include "qn_kernels.cuh"
#include "qn_sptrsv.cuh"
#include "qn_system.h"

namespace qn {

constexpr int kVT = kVertexThreads;     // vertex-kernel block of the small kernels (k_col, k_rest_rhs)
constexpr int kVTB = kVertexThreadsMax;  // launch bound of the per-(vertex, coordinate) kernels (block = v.vt)
constexpr int kBodyUnroll = 3;  // body passes per WHILE iteration of the frame graph (direct solver)
constexpr int kGatherFast = 24;  // vertex valences up to this gather in two round trips (Freudenthal: <= 24)
#ifndef QN_GATHER_LD
#define QN_GATHER_LD __ldg  // corner-force loads of the gradient gather (read-only path: L1 catches the
                            // neighbouring 24-byte entries of a vertex run; __ldcg measured 1-7 % slower)
#endif

constexpr double kCurvatureGuard = 1e-12;  // solvers.py:28
constexpr double kAlphaFloor = 1e-12;      // solvers.py:29

__device__ __forceinline__ size_t vec_off(const SysView& v, int slot, int b) {
  return ((size_t)slot * v.n_inst + b) * (size_t)v.n * 3;
}
__device__ __forceinline__ size_t inst_off(const SysView& v, int b) { return (size_t)b * v.n * 3; }

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ void record(const SysView& v, int b, InstCtl& c, double g, int trials, double alpha) {
  const int it = v.cfg->iterations;
  if (c.k < it && c.k < v.rec_cap) {
    const size_t o = (size_t)b * v.rec_cap + c.k;
    v.rec_g[o] = g;
    v.rec_trials[o] = trials;
    v.rec_alpha[o] = alpha;
    v.rec_ms[o] = (double)(global_ns() - c.t0) * 1e-6;
  }
  c.k += 1;
}

__device__ __forceinline__ int free_slot(int cur, int prev) {
  if (prev < 0 || prev == cur) return (cur + 1) % 3;
  return 3 - cur - prev;
}

// ---------------------------------------------------------------------------
// frame init: y = 2 q_l - q_prev + h^2 g, fixed rows = targets | q_l (dynamics.py:437-443)
__global__ void k_init(SysView v) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < v.n) {
    const size_t o = inst_off(v, b) + (size_t)i * 3;
    double y[3];
    if (v.is_fixed[i]) {
      if (v.cfg->has_targets) {
        const double* t = v.targets + ((size_t)b * v.n_fixed + v.fixed_pos[i]) * 3;
        y[0] = t[0];
        y[1] = t[1];
        y[2] = t[2];
      } else {
        y[0] = v.q_l[o];
        y[1] = v.q_l[o + 1];
        y[2] = v.q_l[o + 2];
      }
    } else {
      const double hh = __dmul_rn(v.h, v.h);
#pragma unroll
      for (int a = 0; a < 3; ++a)
        y[a] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, v.q_l[o + a]), v.q_prev[o + a]), __dmul_rn(hh, v.grav[a]));
    }
    double* X0 = v.X + vec_off(v, 0, b) + (size_t)i * 3;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      v.y[o + a] = y[a];
      X0[a] = y[a];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    InstCtl& c = v.ctl[b];
    c.phase = PH_FIRST;
    c.k = 0;
    c.trials = 0;
    c.status = 0;
    c.fallbacks = 0;
    c.cheb_fb = 0;
    c.omega = 1.0;  // solvers.py:272
    c.xs_cur = 0;
    c.xs_prev = -1;
    c.xs_trial = 0;
    c.gs_cur = 0;
    c.npairs = 0;
    c.have_prev = 0;
    for (int r = 0; r <= kMaxM; ++r) c.ring[r] = r;
    c.g0 = c.g_x = 0.0;
    c.alpha = 0.0;
    c.slope = 0.0;
    c.t0 = global_ns();
    if (v.pcg) v.pctl[b].total = 0;
    if (b == 0) {
      *v.active = v.n_inst;
      v.passes[0] = 0;
      v.passes[1] = 0;  // error bits of this frame
    }
  }
}

// The finalisers run their scalar logic on a shared-memory copy of the
// instance's control block (one cooperative round trip in, one out) instead
// of chains of dependent global loads.
static_assert(sizeof(InstCtl) % 8 == 0, "InstCtl must be a whole number of 8-byte words");
__device__ __forceinline__ void ctl_load(const InstCtl* g, InstCtl* s) {
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(g);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(s);
  for (int w = threadIdx.x; w < (int)(sizeof(InstCtl) / 8); w += blockDim.x) dst[w] = __ldcg(src + w);
  __syncthreads();
}
__device__ __forceinline__ void ctl_store(InstCtl* g, const InstCtl* s) {
  __syncthreads();
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(s);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(g);
  for (int w = threadIdx.x; w < (int)(sizeof(InstCtl) / 8); w += blockDim.x) __stcg(dst + w, src[w]);
}

__device__ void grad_finalize(const SysView& v, int b, InstCtl& c, const double* tot, bool push, int np, int cand,
                              int gnew);
__device__ void eta_finalize(InstCtl& c, const double* tot, int np);

// diagnostics timeline: slot 0 = entry of block (0,0), slot 1 = end of the
// finalising block (only when v.ktl is set)
__device__ __forceinline__ void tl_mark(const SysView& v, int kid, int slot) {
  if (v.ktl && threadIdx.x == 0) {
    const unsigned long long p = *((volatile unsigned long long*)v.passes);
    if (p < (unsigned long long)kTimelinePasses) v.ktl[(p * kTimelineKernels + kid) * 2 + slot] = global_ns();
  }
}
__device__ __forceinline__ void tl_entry(const SysView& v, int kid) {
  if (blockIdx.x == 0 && blockIdx.y == 0) tl_mark(v, kid, 0);
}

// ---------------------------------------------------------------------------
// gradient gather + L-BFGS push / zeta (dynamics.py:470-478, solvers.py:83-103, 124-131)
// M = compile-time bound on the history window (the register footprint of the
// dot-product accumulators scales with it; the host picks the smallest that fits).
template <int M>
__global__ void __launch_bounds__(kVTB) k_grad(SysView v) {
  pdl_entry();
  constexpr int NG = 5 + 2 * M;
  tl_entry(v, 0);
  // instances in reverse launch order: the per-tet pass just wrote the last
  // instances' corner forces, which are the ones still resident in L2
  const int b = (int)(gridDim.y - 1 - blockIdx.y);
  const InstCtl* cc = v.ctl + b;
  if (cc->phase != PH_GRAD) return;
  __shared__ double red[kNG * 32];
  const int cur = cc->xs_cur, prv = cc->xs_prev, gcur = cc->gs_cur, gnew = gcur ^ 1;
  const int np = cc->npairs;
  const DevConfig& cfg = *v.cfg;
  const bool push = cc->have_prev && cfg.kind == 1 && cfg.m > 0;
  const int cand = cc->ring[np];
  double acc[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) acc[k] = 0.0;
  // one thread per (vertex, coordinate): 3x the parallelism of a vertex loop,
  // coalesced vector accesses, and the same per-coordinate summation order
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;
  if (ci < 3 * v.n) {
    const int i = ci / 3;
    const size_t oc = inst_off(v, b) + (size_t)ci;
    const double xc = v.X[vec_off(v, cur, b) + ci];
    double g = __dmul_rn(__ldg(v.w_in + i), __dsub_rn(xc, v.y[oc]));
    // corner forces are stored in gather order: this vertex's entries are the
    // contiguous run [v2e_ptr[i], v2e_ptr[i+1]) (element order = the
    // reference's np.add.at order)
    const double* fb = v.forces + (size_t)b * v.mt * 12 + (ci - 3 * i);
    const int e1 = __ldg(v.v2e_ptr + i + 1);
    int e = __ldg(v.v2e_ptr + i);
    if (e1 - e <= kGatherFast) {
      const int cnt = e1 - e;
      double f[kGatherFast];
#pragma unroll
      for (int q = 0; q < kGatherFast; ++q)
        if (q < cnt) f[q] = QN_GATHER_LD(fb + 3 * (size_t)(e + q));
#pragma unroll
      for (int q = 0; q < kGatherFast; ++q)
        if (q < cnt) g = __dadd_rn(g, f[q]);
    } else {
      for (; e + 8 <= e1; e += 8) {
        double f[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = QN_GATHER_LD(fb + 3 * (size_t)(e + q));
#pragma unroll
        for (int q = 0; q < 8; ++q) g = __dadd_rn(g, f[q]);
      }
      for (; e < e1; ++e) g = __dadd_rn(g, QN_GATHER_LD(fb + 3 * (size_t)e));
    }
    if (v.n_col) g = __dadd_rn(g, v.col_g[oc]);  // add_collision_gradient (dynamics.py:476)
    if (v.is_fixed[i]) g = 0.0;
    v.Gr[vec_off(v, gnew, b) + ci] = g;
    acc[0] = g * g;
    double s = 0.0, t = 0.0;
    if (push) {
      s = __dsub_rn(xc, v.X[vec_off(v, prv, b) + ci]);
      t = __dsub_rn(g, v.Gr[vec_off(v, gcur, b) + ci]);
      v.S[vec_off(v, cand, b) + ci] = s;
      v.T[vec_off(v, cand, b) + ci] = t;
      acc[1] = t * s;
      acc[2] = s * s;
      acc[3] = t * t;
      acc[4] = s * g;
    }
#pragma unroll
    for (int p = 0; p < M; ++p) {  // compile-time indices keep acc[] in registers
      if (p < np) {
        const double si = v.S[vec_off(v, cc->ring[p], b) + ci];
        acc[5 + M + p] = si * g;
        if (push) acc[5 + p] = si * t;
      }
    }
  }
  // reduce only the dot products in use: 0..4, 5..5+np, 5+M..5+M+np
  const unsigned long long used = ((1ull << (5 + np)) - 1ull) | (((1ull << np) - 1ull) << (5 + M));
  block_sum_masked<NG>(acc, red, used);
  // compact partial row: [0..5) scalars, [5, 5+np) <s_i,t_new>, [5+np, 5+2np) <s_i,g>
  const int nval = 5 + 2 * np;
  if (threadIdx.x == 0) {
    double* pv = v.part_v + ((size_t)b * v.nblk_v + blockIdx.x) * kNG;
#pragma unroll
    for (int k = 0; k < 5; ++k) pv[k] = acc[k];
#pragma unroll
    for (int p = 0; p < M; ++p) {
      if (p < np) {
        pv[5 + p] = acc[5 + p];
        pv[5 + np + p] = acc[5 + M + p];
      }
    }
  }
  if (!last_block(v.cnt, 0, b, v.n_inst, gridDim.x)) return;
  // ---- finalise: block-parallel partial sums, control block staged in shared
  //      memory, scalar logic on one thread, control block written back ----
  double* tot = red;
  sum_partials(v.part_v + (size_t)b * v.nblk_v * kNG, gridDim.x, kNG, nval, tot);
  __shared__ InstCtl sc;
  ctl_load(v.ctl + b, &sc);
  if (threadIdx.x == 0) grad_finalize(v, b, sc, tot, push, np, cand, gnew);
  ctl_store(v.ctl + b, &sc);
  tl_mark(v, 0, 1);
}

__device__ void grad_finalize(const SysView& v, int b, InstCtl& c, const double* tot, bool push, int np, int cand,
                              int gnew) {
  const DevConfig& cfg = *v.cfg;
  c.gs_cur = gnew;
  if (push) {
    const double rho = tot[1];
    const double guard = kCurvatureGuard * sqrt(tot[2]) * sqrt(tot[3]);
    for (int p = 0; p < np; ++p) c.sg[c.ring[p]] = tot[5 + np + p];
    if (rho > guard) {
      for (int p = 0; p < np; ++p) c.gram[c.ring[p]][cand] = tot[5 + p];
      c.rho[cand] = rho;
      c.tt[cand] = tot[3];
      c.sg[cand] = tot[4];
      if (np < cfg.m) {
        c.npairs = np + 1;
      } else {  // evict the oldest pair (solvers.py:96-97)
        const int old = c.ring[0];
        for (int p = 0; p < cfg.m; ++p) c.ring[p] = c.ring[p + 1];
        c.ring[cfg.m] = old;
      }
    }
  } else {
    for (int p = 0; p < np; ++p) c.sg[c.ring[p]] = tot[5 + np + p];
  }
  c.have_prev = 1;
  if (sqrt(tot[0]) <= cfg.grad_tol) {  // solvers.py:292-298
    record(v, b, c, c.g_x, 0, 0.0);
    if (cfg.kind != 2) c.xs_prev = c.xs_cur;  // chebyshev keeps x_prev_iter (solvers.py:347)
    c.phase = c.k >= cfg.iterations ? PH_DONE : PH_GRAD;  // forces still belong to x
    if (c.phase == PH_DONE) atomicSub(v.active, 1);
    return;
  }
  const int npn = c.npairs;
  for (int p = npn - 1; p >= 0; --p) {
    const int sp = c.ring[p];
    double q = -c.sg[sp];
    for (int j = p + 1; j < npn; ++j) q -= c.zeta[j] * c.gram[sp][c.ring[j]];
    c.zeta[p] = q / c.rho[sp];
  }
  if (cfg.kind == 2) {  // chebyshev weight of this iteration (solvers.py:154-161), k = c.k + 1
    const int k = c.k + 1;
    const double r2 = cfg.cheb_rho * cfg.cheb_rho;
    c.omega = k < cfg.cheb_S ? 1.0 : k == cfg.cheb_S ? 2.0 / (2.0 - r2) : 4.0 / (4.0 - r2 * c.omega);
    c.cheb_fb = 0;
  }
  c.xs_trial = free_slot(c.xs_cur, c.xs_prev);
  c.phase = PH_DIR;
}

// RHS / output mapping of the solves inside the frame
struct SolverIO {
  SysView v;
  __device__ bool active(int b) const { return v.ctl[b].phase == PH_DIR; }
  __device__ void rhs(int b, int row, double (&q)[3]) const {
    const InstCtl* c = v.ctl + b;
    const int vx = v.fact_vtx[row];
    const double* g = v.Gr + vec_off(v, c->gs_cur, b) + (size_t)vx * 3;
    q[0] = -g[0];
    q[1] = -g[1];
    q[2] = -g[2];
    for (int p = c->npairs - 1; p >= 0; --p) {  // q -= zeta t, newest first
      const double z = c->zeta[p];
      const double* t = v.T + vec_off(v, c->ring[p], b) + (size_t)vx * 3;
      q[0] = __dsub_rn(q[0], __dmul_rn(z, t[0]));
      q[1] = __dsub_rn(q[1], __dmul_rn(z, t[1]));
      q[2] = __dsub_rn(q[2], __dmul_rn(z, t[2]));
    }
  }
  __device__ double* dest(int b, int row) const { return v.R0 + inst_off(v, b) + (size_t)v.fact_vtx[row] * 3; }
  __device__ void store(int b, int row, const double (&x)[3]) const {
    double* r = v.R0 + inst_off(v, b) + (size_t)v.fact_vtx[row] * 3;
    r[0] = x[0];
    r[1] = x[1];
    r[2] = x[2];
  }
};

// lbfgs_init = "scaled_identity" (solvers.py:136-141): r = (rho / <t, t>) q of
// the newest pair (1 with an empty history) in place of A^-1 q, every row
// (fixed rows of q are zero), one thread per (vertex, coordinate)
__global__ void __launch_bounds__(kVTB) k_scaled(SysView v) {
  const int b = blockIdx.y;
  const InstCtl* c = v.ctl + b;
  if (c->phase != PH_DIR) return;
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= 3 * v.n) return;
  const int np = c->npairs;
  double q = -v.Gr[vec_off(v, c->gs_cur, b) + ci];
  for (int p = np - 1; p >= 0; --p)  // q -= zeta t, newest first
    q = __dsub_rn(q, __dmul_rn(c->zeta[p], v.T[vec_off(v, c->ring[p], b) + ci]));
  const double scale = np > 0 ? c->rho[c->ring[np - 1]] / c->tt[c->ring[np - 1]] : 1.0;
  v.R0[inst_off(v, b) + ci] = scale * q;
}

// lbfgs_init = "rest_pose_hessian": q on the free dofs (two-loop first half,
// reference rounding), then r = H_rest^-1 q as a dense product (the inverse
// is formed once from the Cholesky factor), warp per row; fixed rows of R0 = 0
__global__ void __launch_bounds__(kVertexThreads) k_rest_rhs(SysView v) {
  const InstCtl* c = v.ctl;
  if (c->phase != PH_DIR) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < 3 * v.n) v.R0[k] = 0.0;
  if (k >= v.nf3) return;
  const int dof = v.free3[k];
  double q = -v.Gr[vec_off(v, c->gs_cur, 0) + dof];
  for (int p = c->npairs - 1; p >= 0; --p)
    q = __dsub_rn(q, __dmul_rn(c->zeta[p], v.T[vec_off(v, c->ring[p], 0) + dof]));
  v.qbuf[k] = q;
}

__global__ void __launch_bounds__(256) k_rest_apply(SysView v) {
  if (v.ctl->phase != PH_DIR) return;
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * 8 + (threadIdx.x >> 5), nw = gridDim.x * 8;
  for (int r = w0; r < v.nf3; r += nw) {
    const double* row = v.hrest_inv + (size_t)r * v.nf3;
    double a = 0.0;
    for (int j = lane; j < v.nf3; j += 32) a = fma(__ldg(row + j), v.qbuf[j], a);
    a = warp_sum(a);
    if (lane == 0) v.R0[v.free3[r]] = a;
  }
}

// The persistent solve's right-hand side precomputed once per direction in
// factor order (qf), so a forward task loads its rows contiguously instead of
// forming q' = -g - sum zeta t row by row (the wide supernodes' row tasks all
// need the same nc rows).  Same rounding as SolverIO::rhs.
__global__ void __launch_bounds__(kVTB) k_solve_rhs(SysView v) {
  pdl_entry();
  const int b = blockIdx.y;
  const InstCtl* c = v.ctl + b;
  if (c->phase != PH_DIR) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (factor row, coordinate)
  if (i >= 3 * v.n_free) return;
  const int row = i / 3, k = i - 3 * row;
  const size_t o = (size_t)v.fact_vtx[row] * 3 + k;
  double q = -v.Gr[vec_off(v, c->gs_cur, b) + o];
  for (int p = c->npairs - 1; p >= 0; --p)  // q -= zeta t, newest first
    q = __dsub_rn(q, __dmul_rn(c->zeta[p], v.T[vec_off(v, c->ring[p], b) + o]));
  v.qf[(size_t)b * v.n_free * 3 + i] = q;
}

struct FactorRhsIO : SolverIO {
  __device__ void rhs(int b, int row, double (&q)[3]) const {
    const double* r = v.qf + ((size_t)b * v.n_free + row) * 3;
    q[0] = __ldcg(r);
    q[1] = __ldcg(r + 1);
    q[2] = __ldcg(r + 2);
  }
};

// stand-alone timing of the solve kernels (qn_system_time_kernel): every
// instance, right-hand side = the resident q_l, result into the R0 scratch
struct TimingIO {
  SysView v;
  __device__ bool active(int) const { return true; }
  __device__ void rhs(int b, int row, double (&q)[3]) const {
    const double* x = v.q_l + inst_off(v, b) + (size_t)v.fact_vtx[row] * 3;
    q[0] = x[0];
    q[1] = x[1];
    q[2] = x[2];
  }
  __device__ double* dest(int b, int row) const { return v.R0 + inst_off(v, b) + (size_t)v.fact_vtx[row] * 3; }
  __device__ void store(int b, int row, const double (&x)[3]) const {
    double* r = dest(b, row);
    r[0] = x[0];
    r[1] = x[1];
    r[2] = x[2];
  }
};

int launch_solve_timing(qn_system* S, cudaStream_t st) { return launch_solve(S->factor, TimingIO{S->v}, st); }

// <t_i, r0> and the eta recursion (solvers.py:147-150)
template <int M>
__global__ void __launch_bounds__(kVTB) k_eta(SysView v) {
  pdl_entry();
  tl_entry(v, 1);
  const int b = blockIdx.y;
  const InstCtl* cc = v.ctl + b;
  if (cc->phase != PH_DIR || cc->npairs == 0) return;
  __shared__ double red[kMaxM * 32];
  const int np = cc->npairs;
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; ++k) acc[k] = 0.0;
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;  // (vertex, coordinate)
  if (ci < 3 * v.n) {
    const double r = v.R0[inst_off(v, b) + ci];
#pragma unroll
    for (int p = 0; p < M; ++p)
      if (p < np) acc[p] = v.T[vec_off(v, cc->ring[p], b) + ci] * r;
  }
  block_sum_masked<M>(acc, red, (1ull << np) - 1ull);
  if (threadIdx.x == 0) {
    double* pv = v.part_v + ((size_t)b * v.nblk_v + blockIdx.x) * kNG;
    for (int k = 0; k < M; ++k) pv[k] = acc[k];
  }
  if (!last_block(v.cnt, 1, b, v.n_inst, gridDim.x)) return;
  double* tot = red;
  sum_partials(v.part_v + (size_t)b * v.nblk_v * kNG, gridDim.x, kNG, np, tot);
  __shared__ InstCtl sc;
  ctl_load(v.ctl + b, &sc);
  if (threadIdx.x == 0) eta_finalize(sc, tot, np);
  tl_mark(v, 1, 1);
  __syncthreads();
  // only coef[] changed
  if (threadIdx.x < np) v.ctl[b].coef[threadIdx.x] = sc.coef[threadIdx.x];
}

__device__ void eta_finalize(InstCtl& c, const double* tot, int np) {
  for (int p = 0; p < np; ++p) {
    const int sp = c.ring[p];
    double tr = tot[p];
    for (int j = 0; j < p; ++j) tr += c.coef[j] * c.gram[c.ring[j]][sp];
    const double eta = tr / c.rho[sp];
    c.coef[p] = c.zeta[p] - eta;
  }
}

// direction, trial point, inertia / slope partials
__global__ void __launch_bounds__(kVTB) k_vec(SysView v) {
  pdl_entry();
  tl_entry(v, 2);
  const int b = blockIdx.y;
  const InstCtl* cc = v.ctl + b;
  const int ph = cc->phase;
  if (ph == PH_GRAD || ph == PH_DONE) return;
  __shared__ double red[2 * 32];
  double acc[2] = {0.0, 0.0};
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;  // (vertex, coordinate)
  if (ci < 3 * v.n) {
    const size_t oc = inst_off(v, b) + (size_t)ci;
    const double x = v.X[vec_off(v, cc->xs_cur, b) + ci];
    double xt = x;
    if (ph == PH_DIR || ph == PH_ALPHA) {
      double d;
      if (ph == PH_DIR) {
        d = v.R0[oc];
        const int np = cc->npairs;
        for (int p = 0; p < np; ++p)  // r += s (zeta - eta), oldest first
          d = __dadd_rn(d, __dmul_rn(v.S[vec_off(v, cc->ring[p], b) + ci], cc->coef[p]));
        if (v.cfg->kind == 2 && !cc->cheb_fb) {
          // d = omega (x + q - x_prev_iter) + x_prev_iter - x (solvers.py:162-163), q = the pd_qn direction
          const int xp = cc->xs_prev < 0 ? cc->xs_cur : cc->xs_prev;
          const double xkm1 = v.X[vec_off(v, xp, b) + ci];
          const double xhat = __dadd_rn(x, d);
          d = __dsub_rn(__dadd_rn(__dmul_rn(cc->omega, __dsub_rn(xhat, xkm1)), xkm1), x);
        }
        double ds = d;  // step direction (differs from d only under test fault injection)
        const int fault = v.cfg->fault;
        if (fault && cc->k + 1 >= (fault >> 4)) {  // cc->k = iterations recorded so far
          if ((fault & 15) == 1) d = ds = -d;  // ascent
          else ds = -d;                        // steps that only increase g: stagnation
        }
        v.D[oc] = ds;
        acc[1] = v.Gr[vec_off(v, cc->gs_cur, b) + ci] * d;
        d = ds;
      } else {
        d = v.D[oc];
      }
      const double al = (ph == PH_DIR) ? (v.cfg->line_search ? __dmul_rn(v.cfg->alpha_init, v.cfg->shrink) : 1.0)
                                        : cc->alpha;
      xt = __dadd_rn(x, __dmul_rn(al, d));
      v.X[vec_off(v, cc->xs_trial, b) + ci] = xt;
    }
    const double e = xt - v.y[oc];
    acc[0] = __ldg(v.masses + ci / 3) * (e * e);
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    double* pv = v.part_v + ((size_t)b * v.nblk_v + blockIdx.x) * kNG + (kNG - 2);
    pv[0] = acc[0];
    pv[1] = acc[1];
  }
}

// one thread; e_el / inert / slope are the block-parallel sums of the partials
__device__ void finalize_trial(const SysView& v, int b, InstCtl& c, double e_el, double inert, double slope) {
  const DevConfig& cfg = *v.cfg;
  const double e_base = (0.5 / __dmul_rn(v.h, v.h)) * inert + e_el;  // dynamics.py:463-465
  const double g_new = v.n_col ? e_base + c.e_col : e_base;          // + collision_energy (:466)
  const int ph = c.phase;
  if (ph == PH_FIRST) {
    c.g0 = c.g_x = g_new;
    c.e_base = e_base;
    c.phase = PH_GRAD;
    return;
  }
  if (ph == PH_COPY) {
    c.phase = PH_GRAD;
    return;
  }
  bool accept = false;
  if (ph == PH_DIR) {
    if (cfg.kind == 2 && !c.cheb_fb && slope >= 0.0) {  // solvers.py:309-311: d = q, fallbacks += 1
      c.fallbacks += 1;
      c.cheb_fb = 1;  // the next pass re-forms the first trial from the pd_qn direction
      return;
    }
    c.slope = slope;
    c.trials = 1;
    c.alpha = __dmul_rn(cfg.alpha_init, cfg.shrink);
    if (!cfg.line_search) {
      accept = true;
    } else if (slope >= 0.0) {  // solvers.py:244-246 -> SolverError
      c.status |= 2;
      atomicOr(v.passes + 1, 2ull);
      c.phase = PH_DONE;
      atomicSub(v.active, 1);
      return;
    } else if (-slope <= 1e-12 * fmax(fabs(c.g_x), 1.0)) {  // solvers.py:319-326
      record(v, b, c, c.g_x, 0, 0.0);
      if (cfg.kind != 2) c.xs_prev = c.xs_cur;
      c.phase = c.k >= cfg.iterations ? PH_DONE : PH_COPY;
      c.xs_trial = c.xs_cur;
      if (c.phase == PH_DONE) atomicSub(v.active, 1);
      return;
    } else if (c.alpha < kAlphaFloor) {
      accept = false;  // handled as stagnation below
    }
  }
  if (cfg.line_search && !accept) {
    const double thr = __dadd_rn(c.g_x, __dmul_rn(__dmul_rn(cfg.gamma, c.alpha), c.slope));
    accept = c.alpha >= kAlphaFloor && g_new <= thr;  // Armijo (solvers.py:255)
  }
  if (accept) {
    c.xs_prev = c.xs_cur;
    c.xs_cur = c.xs_trial;
    c.g_x = g_new;
    c.e_base = e_base;
    record(v, b, c, g_new, c.trials, cfg.line_search ? c.alpha : 1.0);
    c.phase = c.k >= cfg.iterations ? PH_DONE : PH_GRAD;
  } else {
    c.alpha = __dmul_rn(c.alpha, cfg.shrink);
    if (c.alpha < kAlphaFloor) {  // StagnationError: pad the record (solvers.py:329-336)
      c.status |= 1;
      while (c.k < cfg.iterations) record(v, b, c, c.g_x, 0, 0.0);
      c.phase = PH_DONE;
    } else {
      c.trials += 1;
      c.phase = PH_ALPHA;
    }
  }
  if (c.phase == PH_DONE) atomicSub(v.active, 1);
}

// ---------------------------------------------------------------------------
// colliders (dynamics.py:199-285): signed distance and projection per kind

__device__ __forceinline__ double norm3(double a, double b, double c) { return sqrt((a * a + b * b) + c * c); }

// torus ring point of `local` (TorusCollider._ring, dynamics.py:244-255), including
// the reference's treatment of on-axis points (only the x component is replaced)
__device__ __forceinline__ void torus_ring(const qn_collider& C, const double* local, double* ring) {
  const double radial = sqrt(local[0] * local[0] + local[1] * local[1]);
  const double safe = fmax(radial, 1e-12);
  ring[0] = radial < 1e-12 ? C.r0 : C.r0 * local[0] / safe;
  ring[1] = C.r0 * local[1] / safe;
  ring[2] = 0.0;
}

__device__ double col_sdist(const qn_collider& C, const double* x) {
  if (C.kind == QN_COL_HALFSPACE)
    return (x[0] - C.p[0]) * C.n[0] + (x[1] - C.p[1]) * C.n[1] + (x[2] - C.p[2]) * C.n[2];
  if (C.kind == QN_COL_SPHERE) return norm3(x[0] - C.p[0], x[1] - C.p[1], x[2] - C.p[2]) - C.r0;
  double l[3] = {x[0] - C.p[0], x[1] - C.p[1], x[2] - C.p[2]}, ring[3];
  torus_ring(C, l, ring);
  return norm3(l[0] - ring[0], l[1] - ring[1], l[2] - ring[2]) - C.r1;
}

// surface point t and outward normal n of a penetrating vertex (project, :207-270)
__device__ void col_project(const qn_collider& C, const double* x, double* t, double* n) {
  if (C.kind == QN_COL_HALFSPACE) {
    const double sd = col_sdist(C, x);
    for (int a = 0; a < 3; ++a) {
      t[a] = x[a] - sd * C.n[a];
      n[a] = C.n[a];
    }
    return;
  }
  double q[3], base[3], rad;
  if (C.kind == QN_COL_SPHERE) {
    for (int a = 0; a < 3; ++a) {
      q[a] = x[a] - C.p[a];
      base[a] = C.p[a];
    }
    rad = C.r0;
  } else {
    double l[3] = {x[0] - C.p[0], x[1] - C.p[1], x[2] - C.p[2]}, ring[3];
    torus_ring(C, l, ring);
    for (int a = 0; a < 3; ++a) {
      q[a] = l[a] - ring[a];
      base[a] = C.p[a] + ring[a];
    }
    rad = C.r1;
  }
  const double dist = norm3(q[0], q[1], q[2]);
  const double safe = fmax(dist, 1e-12);
  for (int a = 0; a < 3; ++a) n[a] = q[a] / safe;
  if (dist < 1e-12) n[0] = n[1] = 0.0, n[2] = 1.0;
  for (int a = 0; a < 3; ++a) t[a] = base[a] + rad * n[a];
}

// which = 0 (before k_grad, PH_GRAD): rebuild the active set at the current
//   iterate (update_collisions, dynamics.py:486-516), its gradient terms
//   2 w_col depth n (:453-457) and g_x = objective(x) with the new set
//   (solvers.py:285-286);
// which = 1 (before k_tet, evaluation phases): collision energy at the trial
//   (PH_FIRST: the set is first built at x = y, solvers.py:280-281).
__global__ void __launch_bounds__(kVT) k_col(SysView v, int which) {
  const int b = blockIdx.y;
  InstCtl* cc = v.ctl + b;
  const int ph = cc->phase;
  bool rebuild;
  int xs;
  if (which == 0) {
    if (ph != PH_GRAD) return;
    rebuild = true;
    xs = cc->xs_cur;
  } else {
    if (ph != PH_FIRST && ph != PH_DIR && ph != PH_ALPHA) return;
    rebuild = ph == PH_FIRST;
    xs = cc->xs_trial;
  }
  __shared__ double red[32];
  double e[1] = {0.0};
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < v.n) {
    const size_t o = inst_off(v, b) + (size_t)i * 3;
    const double* xp = v.X + vec_off(v, xs, b) + (size_t)i * 3;
    const double x[3] = {xp[0], xp[1], xp[2]};
    const double w2 = 2.0 * v.w_col;
    double g[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < v.n_col; ++k) {
      const size_t ck = ((size_t)b * v.n + i) * v.n_col + k;
      const qn_collider& C = v.cols[k];
      double* t = v.col_t + 3 * ck;
      double* nr = v.col_n + 3 * ck;
      if (rebuild) {
        bool act = false;
        if (col_sdist(C, x) < 0.0) {
          double tt[3], nn[3];
          col_project(C, x, tt, nn);
          const double* ql = v.q_l + o;
          const double vn = ((x[0] - ql[0]) / v.h) * nn[0] + ((x[1] - ql[1]) / v.h) * nn[1] +
                            ((x[2] - ql[2]) / v.h) * nn[2];
          act = vn < 0.0 || col_sdist(C, ql) < 0.0;
          for (int a = 0; a < 3; ++a) {
            t[a] = tt[a];
            nr[a] = nn[a];
          }
        }
        v.col_act[ck] = act ? 1 : 0;
      }
      if (v.col_act[ck]) {
        const double depth = (x[0] - t[0]) * nr[0] + (x[1] - t[1]) * nr[1] + (x[2] - t[2]) * nr[2];
        e[0] = fma(depth, depth, e[0]);
        if (which == 0)
          for (int a = 0; a < 3; ++a) g[a] += (w2 * depth) * nr[a];
      }
    }
    if (which == 0)
      for (int a = 0; a < 3; ++a) v.col_g[o + a] = g[a];
  }
  block_sum<1>(e, red);
  if (threadIdx.x == 0) v.part_c[(size_t)b * v.nblk_c + blockIdx.x] = e[0];
  if (last_block(v.cnt_c, 0, b, v.n_inst, gridDim.x)) {
    __shared__ double tot[1];
    sum_partials(v.part_c + (size_t)b * v.nblk_c, gridDim.x, 1, 1, tot);
    if (threadIdx.x == 0) {
      const double ec = v.w_col * tot[0];  // collision_energy (dynamics.py:446-450)
      if (which == 0) {
        cc->g_x = cc->e_base + ec;  // objective(x) with the new set
      } else {
        cc->e_col = ec;
      }
    }
  }
}

int launch_col(qn_system* S, int which, cudaStream_t st) {
  if (!S->v.n_col) return QN_OK;
  k_col<<<dim3(S->v.nblk_c, S->v.n_inst), kVT, 0, st>>>(S->v, which);
  QN_CHECK_LAUNCH();
  return QN_OK;
}

// per-tet pass at the trial point: energy partials + corner forces
template <bool kSm, bool kAniso, bool kF32 = false>
__global__ void __launch_bounds__(kTT, kTetBlocksPerSm) k_tet(SysView v) {
  pdl_entry();
  tl_entry(v, 3);
  const int b = blockIdx.y;
  const InstCtl* cc = v.ctl + b;
  const int ph = cc->phase;
  const bool on = ph == PH_FIRST || ph == PH_DIR || ph == PH_ALPHA || ph == PH_COPY;
  if (on) {
    __shared__ double red[32];
    __shared__ qn_material smat[kMatSmem];
    __shared__ double fsm[kTT * kFStride];
    double e[1] = {0.0};
    if (v.mt > 0) {
      const qn_material* mats = stage_materials<kSm>(v, b, smat);
      e[0] = tet_thread<kAniso, kF32>(v, v.X + vec_off(v, cc->xs_trial, b), b, blockIdx.x * blockDim.x + threadIdx.x, mats, -1,
                        fsm);
      store_forces(v, b, fsm);
    }
    block_sum<1>(e, red);
    if (threadIdx.x == 0) v.part_t[(size_t)b * v.nblk_t + blockIdx.x] = e[0];
    if (last_block(v.cnt, 2, b, v.n_inst, gridDim.x)) {
      __shared__ double tot[3];
      sum_partials(v.part_t + (size_t)b * v.nblk_t, v.nblk_t, 1, 1, tot);
      sum_partials(v.part_v + (size_t)b * v.nblk_v * kNG + (kNG - 2), v.nblk_v, kNG, 2, tot + 1);
      __shared__ InstCtl sc;
      ctl_load(v.ctl + b, &sc);
      if (threadIdx.x == 0) finalize_trial(v, b, sc, tot[0], tot[1], tot[2]);
      ctl_store(v.ctl + b, &sc);
    }
  }
  // last block overall: loop condition of the frame graph
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned* gc = v.cnt + 4 * (size_t)v.n_inst;
    const unsigned total = gridDim.x * gridDim.y;
    const unsigned old = atomicAdd(gc, 1u);
    if (old == total - 1) {
      *gc = 0;
      __threadfence();
      int act = *((volatile int32_t*)v.active);
      tl_mark(v, 3, 1);
      *v.passes += 1;
      if (*v.passes > (unsigned long long)v.cfg->max_passes) act = 0;  // runaway guard (host reports it)
      if (v.cfg->use_graph) cudaGraphSetConditional(v.handle, act > 0 ? 1u : 0u);
    }
  }
}

// q_prev <- q_l, q_l <- x (next SimState, solvers.py:351)
__global__ void k_finish(SysView v) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && v.rec_g0) {  // record fields of the control block, next to the record arrays (one D2H)
    v.rec_g0[b] = v.ctl[b].g0;
    v.rec_status[b] = v.ctl[b].status;
    v.rec_fb[b] = v.ctl[b].fallbacks;
  }
  if (i >= v.n) return;
  const size_t o = inst_off(v, b) + (size_t)i * 3;
  const double* x = v.X + vec_off(v, v.ctl[b].xs_cur, b) + (size_t)i * 3;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    v.q_prev[o + a] = v.q_l[o + a];
    v.q_l[o + a] = x[a];
  }
}

// ---------------------------------------------------------------------------
// seam kernels (objective / gradient / element groups / SVD / material)

template <bool kSm, bool kAniso, bool kF32 = false>
__global__ void __launch_bounds__(kTT, kTetBlocksPerSm) k_tet_plain(SysView v, const double* x, int b, int mat_sel,
                                                                   double* part) {
  // b < 0: every instance (blockIdx.y), x and part strided per instance (timing)
  const int bb = b < 0 ? (int)blockIdx.y : b;
  if (b < 0) {
    x += inst_off(v, bb);
    part += (size_t)bb * v.nblk_t;
  }
  __shared__ double red[32];
  __shared__ qn_material smat[kMatSmem];
  __shared__ double fsm[kTT * kFStride];
  double e[1] = {0.0};
  if (v.mt > 0) {
    const qn_material* mats = stage_materials<kSm>(v, bb, smat);
    e[0] = tet_thread<kAniso, kF32>(v, x, bb, blockIdx.x * blockDim.x + threadIdx.x, mats, mat_sel, fsm);
    store_forces(v, bb, fsm);
  }
  block_sum<1>(e, red);
  if (threadIdx.x == 0) part[blockIdx.x] = e[0];
}

// out[i] = init[i] (+ inertia) + sum of corner forces, element order; fixed rows zeroed if asked
__global__ void k_gather_plain(SysView v, const double* x, const double* y, double* out, int b, int inertia,
                               int zero_fixed, double* part) {
  __shared__ double red[32];
  double e[1] = {0.0};
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < v.n) {
    double g[3];
    if (inertia) {
      const double w = __ldg(v.w_in + i);
      for (int a = 0; a < 3; ++a) g[a] = __dmul_rn(w, __dsub_rn(x[3 * i + a], y[3 * i + a]));
      const double d0 = x[3 * i] - y[3 * i], d1 = x[3 * i + 1] - y[3 * i + 1], d2 = x[3 * i + 2] - y[3 * i + 2];
      e[0] = v.masses[i] * (d0 * d0 + d1 * d1 + d2 * d2);
    } else {
      for (int a = 0; a < 3; ++a) g[a] = out[3 * i + a];
    }
    const double* fb = v.forces + (size_t)b * v.mt * 12;
    for (int k = v.v2e_ptr[i]; k < v.v2e_ptr[i + 1]; ++k) {
      const double* f = fb + (size_t)k * 3;
      for (int a = 0; a < 3; ++a) g[a] = __dadd_rn(g[a], f[a]);
    }
    if (zero_fixed && v.is_fixed[i]) g[0] = g[1] = g[2] = 0.0;
    for (int a = 0; a < 3; ++a) out[3 * i + a] = g[a];
  }
  block_sum<1>(e, red);
  if (threadIdx.x == 0 && part) part[blockIdx.x] = e[0];
}

__global__ void k_svd(int64_t m, const double* F, double* U, double* s, double* V) {
  const int64_t t_raw = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t t = t_raw < m ? t_raw : m - 1;  // all lanes run the SVD (warp votes inside)
  double f[3][3], u[3][3], sg[3], vv[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) f[r][c] = F[t * 9 + r * 3 + c];
  svd_rv3(f, u, sg, vv);
  if (t_raw >= m) return;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      U[t * 9 + r * 3 + c] = u[r][c];
      V[t * 9 + r * 3 + c] = vv[r][c];
    }
  for (int k = 0; k < 3; ++k) s[t * 3 + k] = sg[k];
}

__global__ void k_material(const qn_material* M, int64_t k, const double* sig, double* psi, double* tau) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const double s[3] = {sig[3 * t], sig[3 * t + 1], sig[3 * t + 2]};
  double tt[3];
  psi[t] = vl_eval(*M, s, tt);
  for (int a = 0; a < 3; ++a) tau[3 * t + a] = tt[a];
}

// ---------------------------------------------------------------------------
// PCG solve (configs[4] scale): r0 = A_free^-1 q' by Jacobi-preconditioned CG,
// the three coordinates as three lockstep CG runs with their own scalars.
// Per iteration two kernels: SpMV with the direction update fused into the
// neighbour loads (p_new = z + beta p_old, double-buffered p), then the
// x / r / z update; each ends in a fixed-order block-partial reduction whose
// last block computes alpha (resp. beta and convergence).  The global last
// block of the update kernel drives the inner WHILE node of the frame graph.

constexpr int kPT = 128;  // PCG rows per block
constexpr int kSellUnroll = 8;  // SELL row entries in flight per lane (c5 rows have <= 15)

__device__ __forceinline__ bool pcg_on(const SysView& v, int b) {
  return v.ctl[b].phase == PH_DIR && !(v.pctl[b].conv & 8);
}

// global "last block" of a PCG kernel: write the inner loop condition
__device__ __forceinline__ void pcg_global_tail(const SysView& v, int which) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned* gc = v.cnt_p + 4 * (size_t)v.n_inst + which;
    const unsigned total = gridDim.x * gridDim.y;
    const unsigned old = atomicAdd(gc, 1u);
    if (old == total - 1) {
      *gc = 0;
      __threadfence();
      const int act = *((volatile int32_t*)v.pcg_active);
      if (v.cfg->use_graph) cudaGraphSetConditional(v.pcg_handle, act > 0 ? 1u : 0u);
    }
  }
}

__global__ void __launch_bounds__(kPT) k_pcg_init(SysView v) {
  const int b = blockIdx.y;
  if (v.ctl[b].phase == PH_DIR) {
    __shared__ double red[6 * 32];
    double acc[6] = {0, 0, 0, 0, 0, 0};
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < v.n_free) {
      SolverIO io{v};
      double q[3];
      io.rhs(b, i, q);  // fact_vtx = free vertex ids in PCG mode
      const size_t o = ((size_t)b * v.n_free + i) * 3;
      const double di = v.dinv[(size_t)b * v.n_free + i];
      const bool amg = v.pcg == 2;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double z = q[c] * di;
        v.px[o + c] = 0.0;
        v.pr[o + c] = q[c];
        v.pp[o + c] = amg ? 0.0 : z;  // buffer 0 (read with beta = 0 by the first SpMV)
        acc[c] = amg ? 0.0 : q[c] * z;  // AMG: r.z comes from k_pcg_rz after the first V-cycle
        acc[3 + c] = q[c] * q[c];
      }
    }
    block_sum<6>(acc, red);
    if (threadIdx.x == 0) {
      double* pv = v.part_p + ((size_t)b * v.nblk_p + blockIdx.x) * 8;
      for (int k = 0; k < 6; ++k) pv[k] = acc[k];
    }
    if (last_block(v.cnt_p, 0, b, v.n_inst, gridDim.x)) {
      __shared__ double tot[6];
      sum_partials(v.part_p + (size_t)b * v.nblk_p * 8, gridDim.x, 8, 6, tot);
      if (threadIdx.x == 0) {
        PcgCtl& p = v.pctl[b];
        int conv = 0;
        for (int c = 0; c < 3; ++c) {
          p.rz[c] = tot[c];
          p.bb[c] = tot[3 + c];
          p.rr[c] = tot[3 + c];
          p.alpha[c] = p.beta[c] = 0.0;
          if (!(tot[3 + c] > 0.0)) conv |= 1 << c;  // zero right-hand side
        }
        p.iter = 0;
        if (conv == 7) conv |= 8;  // nothing to do
        p.conv = conv;
        if (!(conv & 8)) atomicAdd(v.pcg_active, 1);
      }
    }
  }
  pcg_global_tail(v, 0);
}

// q = A p with p = z + beta p_old fused into the neighbour loads (z = dinv r
// recomputed, so z is never stored); one warp per SELL slice, lane = row.
// Partial p.q per block -> the last block computes alpha.
template <bool kZf>
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_pcg_spmv(SysView v, int force) {
  const int b = blockIdx.y;
  if (!force && !pcg_on(v, b)) return;  // force: stand-alone timing between frames (qn_system_time_kernel)
  __shared__ double red[3 * 32];
  const PcgCtl& pc = v.pctl[b];
  const int pb = pc.iter & 1;
  const double be0 = pc.beta[0], be1 = pc.beta[1], be2 = pc.beta[2];
  const size_t vo = (size_t)b * v.n_free * 3;
  const double* __restrict__ pold = v.pp + (size_t)pb * v.n_inst * v.n_free * 3 + vo;
  double* __restrict__ pnew = v.pp + (size_t)(pb ^ 1) * v.n_inst * v.n_free * 3 + vo;
  // z = D^-1 r recomputed (Jacobi) or the stored V-cycle output (AMG: r <- z, dinv <- 1)
  const bool amg = v.pcg == 2;
  const double* __restrict__ r = amg ? v.pz + vo : v.pr + vo;
  const float4* __restrict__ zf = v.pzf;  // kZf: z = the V-cycle output as fp32 rows (one 128-bit gather)
  const double* __restrict__ dinv = v.dinv + (size_t)b * v.n_free;
  const double* __restrict__ av = v.sell_val + (size_t)b * v.sell_nnz;
  double* __restrict__ q = v.pq + vo;
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5), nw = gridDim.x * kSpmvWarps;
  double acc[3] = {0, 0, 0};
  for (int sl = w0; sl < v.nslice; sl += nw) {
    const int64_t e0 = v.sell_ptr[sl], e1 = v.sell_ptr[sl + 1];
    double q0 = 0.0, q1 = 0.0, q2 = 0.0;
    int64_t e = e0 + lane;
    for (; e + 32 * (kSellUnroll - 1) < e1; e += 32 * kSellUnroll) {  // kSellUnroll entries in flight
      int j[kSellUnroll];
      double a[kSellUnroll], d[kSellUnroll];
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) {
        j[u] = __ldcs(v.sell_col + e + 32 * u);
        a[u] = __ldcs(av + e + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) d[u] = amg ? 1.0 : __ldg(dinv + j[u]);
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) {
        const double* pj = pold + 3 * (size_t)j[u];
        if (kZf) {
          const float4 zj = zf[j[u]];
          q0 = fma(a[u], fma(be0, pj[0], (double)zj.x), q0);
          q1 = fma(a[u], fma(be1, pj[1], (double)zj.y), q1);
          q2 = fma(a[u], fma(be2, pj[2], (double)zj.z), q2);
        } else {
          const double* rj = r + 3 * (size_t)j[u];
          q0 = fma(a[u], fma(be0, pj[0], rj[0] * d[u]), q0);
          q1 = fma(a[u], fma(be1, pj[1], rj[1] * d[u]), q1);
          q2 = fma(a[u], fma(be2, pj[2], rj[2] * d[u]), q2);
        }
      }
    }
    for (; e < e1; e += 32) {
      const int j = __ldg(v.sell_col + e);
      const double a = __ldg(av + e), d = amg ? 1.0 : __ldg(dinv + j);
      const double* pj = pold + 3 * (size_t)j;
      if (kZf) {
        const float4 zj = zf[j];
        q0 = fma(a, fma(be0, pj[0], (double)zj.x), q0);
        q1 = fma(a, fma(be1, pj[1], (double)zj.y), q1);
        q2 = fma(a, fma(be2, pj[2], (double)zj.z), q2);
      } else {
        const double* rj = r + 3 * (size_t)j;
        q0 = fma(a, fma(be0, pj[0], rj[0] * d), q0);
        q1 = fma(a, fma(be1, pj[1], rj[1] * d), q1);
        q2 = fma(a, fma(be2, pj[2], rj[2] * d), q2);
      }
    }
    const int i = 32 * sl + lane;
    if (i < v.n_free) {
      const double d = amg ? 1.0 : dinv[i];
      double z0, z1, z2;
      if (kZf) {
        const float4 zi = zf[i];
        z0 = zi.x, z1 = zi.y, z2 = zi.z;
      } else {
        z0 = r[3 * i + 0] * d, z1 = r[3 * i + 1] * d, z2 = r[3 * i + 2] * d;
      }
      const double p0 = fma(be0, pold[3 * i + 0], z0);
      const double p1 = fma(be1, pold[3 * i + 1], z1);
      const double p2 = fma(be2, pold[3 * i + 2], z2);
      pnew[3 * i + 0] = p0;
      pnew[3 * i + 1] = p1;
      pnew[3 * i + 2] = p2;
      q[3 * i + 0] = q0;
      q[3 * i + 1] = q1;
      q[3 * i + 2] = q2;
      acc[0] = fma(p0, q0, acc[0]);
      acc[1] = fma(p1, q1, acc[1]);
      acc[2] = fma(p2, q2, acc[2]);
    }
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0) {
    double* pv = v.part_p + ((size_t)b * v.nblk_spmv + blockIdx.x) * 8;
    for (int k = 0; k < 3; ++k) pv[k] = acc[k];
  }
  if (last_block(v.cnt_p, 1, b, v.n_inst, gridDim.x)) {
    __shared__ double tot[3];
    sum_partials(v.part_p + (size_t)b * v.nblk_spmv * 8, gridDim.x, 8, 3, tot);
    if (threadIdx.x == 0) {
      PcgCtl& p = v.pctl[b];
      for (int c = 0; c < 3; ++c) p.alpha[c] = (p.conv >> c) & 1 ? 0.0 : p.rz[c] / tot[c];
    }
  }
}

// AMG-PCG SpMV in recurrence form (single systems with the fp32 z row, v.pzf): p = z + beta p_old
// gives A p = A z + beta (A p_old) = A z + beta q_old, so the kernel gathers ONLY z (one 128-bit
// load per matrix entry; k_pcg_spmv<true> gathers p_old with three more loads) and finishes each
// row with q = A z + beta q_old, p = z + beta p_old in place.  The rounding of q accumulates like
// that of the CG's other recurrences (~1e-16 relative per iteration against a 1e-10 tolerance).
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_pcg_spmv_rec(SysView v, int force) {
  if (!force && !pcg_on(v, 0)) return;
  __shared__ double red[3 * 32];
  const PcgCtl& pc = v.pctl[0];
  const int pb = pc.iter & 1;
  const double be0 = pc.beta[0], be1 = pc.beta[1], be2 = pc.beta[2];
  const bool first = pc.iter == 0;  // beta = 0: q_old is not defined yet
  const double* __restrict__ pold = v.pp + (size_t)pb * v.n_free * 3;
  double* __restrict__ pnew = v.pp + (size_t)(pb ^ 1) * v.n_free * 3;
  const float4* __restrict__ zf = v.pzf;
  const double* __restrict__ av = v.sell_val;
  double* __restrict__ q = v.pq;
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5), nw = gridDim.x * kSpmvWarps;
  double acc[3] = {0, 0, 0};
  for (int sl = w0; sl < v.nslice; sl += nw) {
    const int64_t e0 = v.sell_ptr[sl], e1 = v.sell_ptr[sl + 1];
    double q0 = 0.0, q1 = 0.0, q2 = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 32 * kSellUnroll) {  // masked batches (the mask is warp-uniform)
      int j[kSellUnroll];
      double a[kSellUnroll];
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) {
        const bool ok = e + 32 * u < e1;
        j[u] = ok ? __ldcs(v.sell_col + e + 32 * u) : 0;
        a[u] = ok ? __ldcs(av + e + 32 * u) : 0.0;
      }
      float4 z[kSellUnroll];
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) z[u] = zf[j[u]];
#pragma unroll
      for (int u = 0; u < kSellUnroll; ++u) {
        if (e + 32 * u < e1) {
          q0 = fma(a[u], (double)z[u].x, q0);
          q1 = fma(a[u], (double)z[u].y, q1);
          q2 = fma(a[u], (double)z[u].z, q2);
        }
      }
    }
    const int i = 32 * sl + lane;
    if (i < v.n_free) {
      const float4 zi = zf[i];
      double p0 = zi.x, p1 = zi.y, p2 = zi.z;
      if (!first) {
        p0 = fma(be0, pold[3 * i + 0], p0);
        p1 = fma(be1, pold[3 * i + 1], p1);
        p2 = fma(be2, pold[3 * i + 2], p2);
        q0 = fma(be0, q[3 * i + 0], q0);
        q1 = fma(be1, q[3 * i + 1], q1);
        q2 = fma(be2, q[3 * i + 2], q2);
      }
      pnew[3 * i + 0] = p0;
      pnew[3 * i + 1] = p1;
      pnew[3 * i + 2] = p2;
      q[3 * i + 0] = q0;
      q[3 * i + 1] = q1;
      q[3 * i + 2] = q2;
      acc[0] = fma(p0, q0, acc[0]);
      acc[1] = fma(p1, q1, acc[1]);
      acc[2] = fma(p2, q2, acc[2]);
    }
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0) {
    double* pv = v.part_p + (size_t)blockIdx.x * 8;
    for (int k = 0; k < 3; ++k) pv[k] = acc[k];
  }
  if (last_block(v.cnt_p, 1, 0, v.n_inst, gridDim.x)) {
    __shared__ double tot[3];
    sum_partials(v.part_p, gridDim.x, 8, 3, tot);
    if (threadIdx.x == 0) {
      PcgCtl& p = v.pctl[0];
      for (int c = 0; c < 3; ++c) p.alpha[c] = (p.conv >> c) & 1 ? 0.0 : p.rz[c] / tot[c];
    }
  }
}

// x += alpha p, r -= alpha q; partial r.z and r.r.  One thread per (row,
// coordinate) of the flattened (n_free x 3) vectors, 4 elements in flight.
__global__ void __launch_bounds__(kUpdThreads, kUpdBlocksPerSm) k_pcg_update(SysView v) {
  const int b = blockIdx.y;
  if (pcg_on(v, b)) {
    __shared__ double red[6 * 32];
    const PcgCtl& pc = v.pctl[b];
    const size_t vo = (size_t)b * v.n_free * 3;
    const double* __restrict__ pnew = v.pp + (size_t)((pc.iter & 1) ^ 1) * v.n_inst * v.n_free * 3 + vo;
    double* __restrict__ x = v.px + vo;
    double* __restrict__ r = v.pr + vo;
    const double* __restrict__ q = v.pq + vo;
    const double* __restrict__ dinv = v.dinv + (size_t)b * v.n_free;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = (int)(t % 3);
    const double al = pc.alpha[c];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, n3 = 3 * (int64_t)v.n_free;
    double rz = 0.0, rr = 0.0;
    int64_t e = t;
    for (; e + 3 * stride < n3; e += 4 * stride) {
      double xv[4], pv[4], rv[4], qv[4], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t f = e + u * stride;
        xv[u] = x[f];
        pv[u] = pnew[f];
        rv[u] = r[f];
        qv[u] = q[f];
        dv[u] = __ldg(dinv + f / 3);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t f = e + u * stride;
        x[f] = fma(al, pv[u], xv[u]);
        const double rn = fma(-al, qv[u], rv[u]);
        r[f] = rn;
        const double z = rn * dv[u];
        rz = fma(rn, z, rz);
        rr = fma(rn, rn, rr);
      }
    }
    for (; e < n3; e += stride) {
      x[e] = fma(al, pnew[e], x[e]);
      const double rn = fma(-al, q[e], r[e]);
      r[e] = rn;
      const double z = rn * __ldg(dinv + e / 3);
      rz = fma(rn, z, rz);
      rr = fma(rn, rn, rr);
    }
    double acc[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      acc[k] = k == c ? rz : 0.0;
      acc[3 + k] = k == c ? rr : 0.0;
    }
    block_sum<6>(acc, red);
    if (threadIdx.x == 0) {
      double* pp = v.part_p + ((size_t)b * v.nblk_upd + blockIdx.x) * 8;
      for (int k = 0; k < 6; ++k) pp[k] = acc[k];
    }
    if (last_block(v.cnt_p, 2, b, v.n_inst, gridDim.x)) {
      __shared__ double tot[6];
      sum_partials(v.part_p + (size_t)b * v.nblk_upd * 8, gridDim.x, 8, 6, tot);
      if (threadIdx.x == 0) {
        PcgCtl& p = v.pctl[b];
        const double tol2 = v.pcg_tol * v.pcg_tol;
        int conv = p.conv;
        for (int k = 0; k < 3; ++k) {
          if ((conv >> k) & 1) continue;
          if (v.pcg != 2) {  // AMG: beta and r.z come from k_pcg_rz after the V-cycle
            p.beta[k] = tot[k] / p.rz[k];
            p.rz[k] = tot[k];
          }
          p.rr[k] = tot[3 + k];
          if (tot[3 + k] <= tol2 * p.bb[k]) conv |= 1 << k;
        }
        p.iter += 1;
        p.total += 1;
        if ((conv & 7) == 7 || p.iter >= v.pcg_maxit) {
          if ((conv & 7) != 7) {  // stopped at pcg_maxit short of pcg_tol: reported by the host
            v.ctl[b].status |= 4;
            atomicOr(v.passes + 1, 4ull);
          }
          conv |= 8;
          atomicSub(v.pcg_active, 1);
        }
        p.conv = conv;
      }
    }
  }
  pcg_global_tail(v, 1);
}

// ---- AMG V(1,1) cycle (pcg == 2, one instance): every kernel is one warp
// per 32-row SELL slice, grid-stride, 3 right-hand sides; all no-ops once the
// CG has converged.  Level l: x = w D^-1 b (written by the producer of b: the
// pre-smoothing kernel on level 0, the restriction below), r = b - A x,
// b_{l+1} = R r, ..., x += P t_{l+1}, t = x + w D^-1 (b - A x).
// The cycle's own vectors are fp32 rows of 16 bytes (x, y, z, 0): these kernels
// are bound by the L1 wavefronts of the scattered column gathers (ncu: l1tex
// 76-92 % of peak with three 8-byte loads per matrix entry), so a gathered
// column is one 128-bit load.  Sums run in fp64.

__device__ __forceinline__ float4 f4(double a, double b, double c) {
  return make_float4((float)a, (float)b, (float)c, 0.0f);
}

// One lane's batch of a CSR row: 4 entries K apart, masked at the row end (col -1).
struct CsrBatch {
  int j[4];
  float a[4];
};
__device__ __forceinline__ void csr_batch_load(const int32_t* __restrict__ col, const float* __restrict__ val, int64_t e,
                                               int64_t e1, int K, CsrBatch& B) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {  // streamed once per cycle: evict-first, keep L2 for the vectors
    const int64_t ee = e + (int64_t)K * u;
    const bool ok = ee < e1;
    B.j[u] = ok ? __ldcs(col + ee) : -1;
    B.a[u] = ok ? __ldcs(val + ee) : 0.0f;
  }
}

// Row products y_i = sum_j a_ij X[j] (3 columns) of a V-cycle operator, for
// every row, handed to `epi(i, acc)`.  Two layouts (chosen per operator at
// upload from its mean row length, qn_api.cu sell_upload):
//  * S.kl == 0: SELL-32, one warp per 32-row slice, lane = row (short rows:
//    the fine-level operators of configs[4] have ~13 entries per row);
//  * S.kl = K in {4, 8, 16, 32}: CSR, K lanes per row, 32/K rows per warp;
//    the lanes of a row stride its entries (coalesced), a K-lane butterfly
//    sums them (long rows: Galerkin coarse operators, restriction).
// kCg: the vector was written earlier in the SAME launch by other CTAs (k_amg_tail): read it through
// L2 (ld.global.cg), never through the non-coherent L1 / read-only path
template <bool kCg>
__device__ __forceinline__ float4 ldv(const float4* p) {
  // (intrinsics, not a plain dereference: the compiler split `*p` into 8-byte loads because w is unused;
  // the vectors gathered by the per-level kernels are read-only for the duration of the launch)
  return kCg ? __ldcg(p) : __ldg(p);
}

template <bool kCg, class EPI>
__device__ __forceinline__ void op_rows(const SellDevF S, const float4* X, EPI epi) {  // S by value: the level
  // structs live in global memory, a reference would reload the operator's pointers for every matrix entry
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5), nw = gridDim.x * kSpmvWarps;
  if (S.kl == 0) {
    // every batch is kSellUnroll masked entries (the mask is warp-uniform: a slice is padded to one
    // length), so a 15-entry slice is two round trips instead of one batch plus seven single loads;
    // the next slice's bounds are fetched while this one runs
    int sl = w0;
    int64_t n0 = 0, n1 = 0;
    if (sl < S.nslice) {
      n0 = S.ptr[sl];
      n1 = S.ptr[sl + 1];
    }
    for (; sl < S.nslice; sl += nw) {
      const int64_t e1 = n1;
      int64_t e = n0 + lane;
      if (sl + nw < S.nslice) {
        n0 = S.ptr[sl + nw];
        n1 = S.ptr[sl + nw + 1];
      }
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (; e < e1; e += 32 * kSellUnroll) {
        int j[kSellUnroll];
        float a[kSellUnroll];
#pragma unroll
        for (int u = 0; u < kSellUnroll; ++u) {
          const bool ok = e + 32 * u < e1;
          j[u] = ok ? __ldcs(S.col + e + 32 * u) : -1;
          a[u] = ok ? __ldcs(S.val + e + 32 * u) : 0.0f;
        }
        float4 x[kSellUnroll];
#pragma unroll
        for (int u = 0; u < kSellUnroll; ++u) x[u] = ldv<kCg>(X + (j[u] < 0 ? 0 : j[u]));
        // a batch's products are summed in fp32 (the operands are fp32; the cycle is a preconditioner),
        // the batch sums are added in fp64: 3 float->double conversions per batch instead of 4 per entry
        float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
#pragma unroll
        for (int u = 0; u < kSellUnroll; ++u) {
          if (j[u] >= 0) {
            s0 = fmaf(a[u], x[u].x, s0);
            s1 = fmaf(a[u], x[u].y, s1);
            s2 = fmaf(a[u], x[u].z, s2);
          }
        }
        a0 += (double)s0;
        a1 += (double)s1;
        a2 += (double)s2;
      }
      const int i = 32 * sl + lane;
      if (i < S.nrows) {
        const double acc[3] = {a0, a1, a2};
        epi(i, acc);
      }
    }
    return;
  }
  // CSR, K lanes per row: software pipeline over masked 4-entry batches.  While a batch's column
  // values are gathered, the next batch (of this row or, at its end, of the warp's next rows) is
  // already in flight, and the row bounds are fetched two rows ahead.  Per lane the entries are
  // summed in the order of a plain strided loop.
  const int K = S.kl, g = lane / K, q = lane % K, rpw = 32 / K, step = nw * rpw;
  int r0 = w0 * rpw;
  if (r0 >= S.nrows) return;
  auto bounds = [&](int r, int64_t& b0, int64_t& b1) {
    b0 = b1 = 0;
    if (r + g < S.nrows) {
      b0 = S.ptr[r + g];
      b1 = S.ptr[r + g + 1];
    }
  };
  int64_t e0, e1, n0, n1;
  bounds(r0, e0, e1);
  bounds(r0 + step, n0, n1);
  CsrBatch cur, nxt;
  csr_batch_load(S.col, S.val, e0 + q, e1, K, cur);
  for (; r0 < S.nrows; r0 += step) {  // warp-uniform loop
    const int i = r0 + g;
    int64_t m0, m1;
    bounds(r0 + 2 * step, m0, m1);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int64_t e = e0 + q;
    for (;;) {
      const int64_t en = e + 4 * (int64_t)K;
      const bool more = __any_sync(0xffffffffu, en - q < e1);
      if (more)
        csr_batch_load(S.col, S.val, en, e1, K, nxt);
      else
        csr_batch_load(S.col, S.val, n0 + q, n1, K, nxt);
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = ldv<kCg>(X + (cur.j[u] < 0 ? 0 : cur.j[u]));
      float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (cur.j[u] >= 0) {
          s0 = fmaf(cur.a[u], x[u].x, s0);
          s1 = fmaf(cur.a[u], x[u].y, s1);
          s2 = fmaf(cur.a[u], x[u].z, s2);
        }
      }
      a0 += (double)s0;
      a1 += (double)s1;
      a2 += (double)s2;
      cur = nxt;
      if (!more) break;
      e = en;
    }
    for (int o = K >> 1; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (q == 0 && i < S.nrows) {
      const double acc[3] = {a0, a1, a2};
      epi(i, acc);
    }
    e0 = n0;
    e1 = n1;
    n0 = m0;
    n1 = m1;
  }
}

__device__ __forceinline__ bool amg_on(const SysView& v) { return pcg_on(v, 0); }

// level 0 pre-smoothing from zero: x = w D^-1 b (b = the fp64 CG residual)
__global__ void __launch_bounds__(kUpdThreads, kUpdBlocksPerSm) k_amg_presmooth(SysView v) {
  if (!amg_on(v)) return;
  const AmgDevLevel& L = v.alev[0];
  const double w = L.omega;
  const double* __restrict__ b = L.b;
  const double* __restrict__ dinv = L.dinv;
  float4* __restrict__ xf = L.xf;
  const int n = L.n;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double wd = w * dinv[i];
    const double* bi = b + 3 * (size_t)i;
    xf[i] = f4(wd * bi[0], wd * bi[1], wd * bi[2]);
  }
}

// r = b - A x
template <bool kCg>
__device__ __forceinline__ void amg_residual(const SysView& v, int l) {
  const AmgDevLevel& L = v.alev[l];
  const double* __restrict__ b = L.b;  // the level's fields in registers (the struct is in global memory)
  const float4* bf = L.bf;
  float4* rf = L.rf;
  op_rows<kCg>(L.A, L.xf, [&](int i, const double* a) {
    double bi[3];
    if (l == 0) {
      const double* bp = b + 3 * (size_t)i;
      bi[0] = bp[0], bi[1] = bp[1], bi[2] = bp[2];
    } else {
      const float4 bq = ldv<kCg>(bf + i);
      bi[0] = bq.x, bi[1] = bq.y, bi[2] = bq.z;
    }
    rf[i] = f4(bi[0] - a[0], bi[1] - a[1], bi[2] - a[2]);
  });
}
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_amg_residual(SysView v, int l) {
  if (amg_on(v)) amg_residual<false>(v, l);
}

// b_{l+1} = R_l r_l and the coarse level's pre-smoothed x = w D^-1 b
template <bool kCg>
__device__ __forceinline__ void amg_restrict(const SysView& v, int l) {
  const AmgDevLevel& L = v.alev[l];
  const AmgDevLevel& C = v.alev[l + 1];
  float4* cbf = C.bf;
  float4* cxf = C.xf;
  const double* __restrict__ cdinv = C.dinv;
  const double cw = C.omega;
  op_rows<kCg>(L.R, L.rf, [&](int i, const double* a) {
    cbf[i] = f4(a[0], a[1], a[2]);
    const double wd = cw * cdinv[i];
    cxf[i] = f4(wd * a[0], wd * a[1], wd * a[2]);
  });
}
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_amg_restrict(SysView v, int l) {
  if (amg_on(v)) amg_restrict<false>(v, l);
}

// coarsest level: t = A_c^-1 b (dense inverse, warp per row, b staged in shared memory)
constexpr int kCoarseUnroll = 16;
template <bool kCg>
__device__ __forceinline__ void amg_coarse(const SysView& v, double* sb) {
  const AmgDevLevel& L = v.alev[v.amg_levels - 1];
  const int nc = v.ncoarse;
  const bool single = v.amg_levels == 1;  // one-level hierarchy: the coarsest level is the CG's own (fp64 b, t)
  for (int q = threadIdx.x; q < nc; q += blockDim.x) {
    if (single) {
      sb[3 * q + 0] = L.b[3 * q + 0];
      sb[3 * q + 1] = L.b[3 * q + 1];
      sb[3 * q + 2] = L.b[3 * q + 2];
    } else {
      const float4 bq = ldv<kCg>(L.bf + q);
      sb[3 * q + 0] = bq.x;
      sb[3 * q + 1] = bq.y;
      sb[3 * q + 2] = bq.z;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5), nw = gridDim.x * kSpmvWarps;
  for (int k = w0; k < nc; k += nw) {
    const float* row = v.cinv + (size_t)k * nc;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int c = lane;
    for (; c + 32 * (kCoarseUnroll - 1) < nc; c += 32 * kCoarseUnroll) {  // kCoarseUnroll loads in flight per lane
      float m[kCoarseUnroll];
#pragma unroll
      for (int u = 0; u < kCoarseUnroll; ++u) m[u] = __ldg(row + c + 32 * u);
#pragma unroll
      for (int u = 0; u < kCoarseUnroll; ++u) {
        const int cc = c + 32 * u;
        a0 = fma((double)m[u], sb[3 * cc + 0], a0);
        a1 = fma((double)m[u], sb[3 * cc + 1], a1);
        a2 = fma((double)m[u], sb[3 * cc + 2], a2);
      }
    }
    if (c < nc) {  // the row's tail as one masked batch (same per-lane order as a one-by-one loop)
      float m[kCoarseUnroll];
#pragma unroll
      for (int u = 0; u < kCoarseUnroll; ++u) m[u] = c + 32 * u < nc ? __ldg(row + c + 32 * u) : 0.0f;
#pragma unroll
      for (int u = 0; u < kCoarseUnroll; ++u) {
        const int cc = c + 32 * u;
        if (cc < nc) {
          a0 = fma((double)m[u], sb[3 * cc + 0], a0);
          a1 = fma((double)m[u], sb[3 * cc + 1], a1);
          a2 = fma((double)m[u], sb[3 * cc + 2], a2);
        }
      }
    }
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) {
      if (single) {
        L.t[3 * k + 0] = a0;
        L.t[3 * k + 1] = a1;
        L.t[3 * k + 2] = a2;
      } else {
        L.tf[k] = f4(a0, a1, a2);
      }
    }
  }
}
__global__ void __launch_bounds__(kSpmvThreads) k_amg_coarse(SysView v) {
  extern __shared__ double sb[];
  if (amg_on(v)) amg_coarse<false>(v, sb);
}

// x_l += P_l t_{l+1}
template <bool kCg>
__device__ __forceinline__ void amg_prolong(const SysView& v, int l) {
  const AmgDevLevel& L = v.alev[l];
  const AmgDevLevel& C = v.alev[l + 1];
  float4* xf = L.xf;
  op_rows<kCg>(L.P, C.tf, [&](int i, const double* a) {
    const float4 xi = kCg ? __ldcg(xf + i) : xf[i];  // read-modify-write: not the read-only path
    xf[i] = f4((double)xi.x + a[0], (double)xi.y + a[1], (double)xi.z + a[2]);
  });
}
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_amg_prolong(SysView v, int l) {
  if (amg_on(v)) amg_prolong<false>(v, l);
}

// t = x + w D^-1 (b - A x)  (post-smoothing; level 0 writes z in fp64)
template <bool kCg>
__device__ __forceinline__ void amg_smooth(const SysView& v, int l) {
  const AmgDevLevel& L = v.alev[l];
  const double w = L.omega;
  const double* __restrict__ dinv = L.dinv;
  const float4* xf = L.xf;
  const double* __restrict__ b = L.b;
  double* __restrict__ t = L.t;
  const float4* bf = L.bf;
  float4* tf = L.tf;
  op_rows<kCg>(L.A, xf, [&](int i, const double* a) {
    const double wd = w * dinv[i];
    const float4 xi = ldv<kCg>(xf + i);
    if (l == 0) {
      const double* bi = b + 3 * (size_t)i;
      double* ti = t + 3 * (size_t)i;
      ti[0] = fma(wd, bi[0] - a[0], (double)xi.x);
      ti[1] = fma(wd, bi[1] - a[1], (double)xi.y);
      ti[2] = fma(wd, bi[2] - a[2], (double)xi.z);
    } else {
      const float4 bq = ldv<kCg>(bf + i);
      tf[i] = f4(fma(wd, (double)bq.x - a[0], (double)xi.x), fma(wd, (double)bq.y - a[1], (double)xi.y),
                   fma(wd, (double)bq.z - a[2], (double)xi.z));
    }
  });
}
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_amg_smooth(SysView v, int l) {
  if (amg_on(v)) amg_smooth<false>(v, l);
}

// The small levels of the hierarchy (levels l0 .. coarsest, a few thousand rows each) in ONE
// launch: their kernels do microseconds of work but pay a launch boundary each (13 graph nodes
// per V-cycle on configs[4]).  The CTAs of this kernel are all resident (grid sized from the
// occupancy query, prepare_kernels) and separate the phases with a grid-wide barrier: arrivals
// on amg_bar[0], which only grows; amg_bar[1] is the count at kernel entry, advanced by the last
// arrival of the last barrier.  A barrier that does not complete (a CTA not resident) gives up
// after ~1 s and reports through the frame's error word instead of hanging.
__device__ __forceinline__ bool amg_grid_barrier(const SysView& v, unsigned base, unsigned k, bool last) {
  __syncthreads();
  __shared__ int ok;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned target = k * gridDim.x;
    const unsigned arrived = atomicAdd(v.amg_bar, 1u) + 1u - base;
    ok = 1;
    if (arrived == target) {
      if (last) {
        atomicExch(v.amg_bar + 1, base + target);
        __threadfence();
      }
    } else {
      unsigned spins = 0;
      while (*((volatile unsigned*)v.amg_bar) - base < target) {
        if (++spins > (1u << 22)) {
          __nanosleep(200);
          if (spins > (1u << 22) + 5000000u) {
            ok = 0;
            atomicOr(v.passes + 1, 8ull);
            break;
          }
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
  return ok != 0;
}

__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_amg_tail(SysView v, int l0) {
  extern __shared__ double sb[];
  if (!amg_on(v)) return;  // uniform over the grid: no CTA enters the barriers
  const unsigned base = *((volatile unsigned*)(v.amg_bar + 1));
  const int nl = v.amg_levels;
  const unsigned nbar = 4u * (unsigned)(nl - 1 - l0);
  unsigned k = 0;
  for (int l = l0; l + 1 < nl; ++l) {
    amg_residual<true>(v, l);
    ++k;
    if (!amg_grid_barrier(v, base, k, false)) return;
    amg_restrict<true>(v, l);
    ++k;
    if (!amg_grid_barrier(v, base, k, false)) return;
  }
  amg_coarse<true>(v, sb);
  for (int l = nl - 2; l >= l0; --l) {
    ++k;
    if (!amg_grid_barrier(v, base, k, false)) return;
    amg_prolong<true>(v, l);
    ++k;
    if (!amg_grid_barrier(v, base, k, k == nbar)) return;
    amg_smooth<true>(v, l);
  }
}

// Level-0 post-smoothing of a single system: z = x + w D^-1 (b - A x) rounded to fp32 rows (v.pzf:
// the CG reads z only through it, so p, q and r.z all see the same z), with the r.z partial sums
// of k_pcg_rz in the epilogue (b is the CG residual): the last block forms beta and r.z.
__global__ void __launch_bounds__(kSpmvThreads, kSpmvBlocksPerSm) k_amg_smooth_rz(SysView v) {
  if (!amg_on(v)) return;
  __shared__ double red[3 * 32];
  const AmgDevLevel& L = v.alev[0];
  double acc[3] = {0.0, 0.0, 0.0};
  const double w = L.omega;
  const double* __restrict__ dinv = L.dinv;
  const float4* __restrict__ xf = L.xf;
  const double* __restrict__ b = L.b;
  float4* __restrict__ zf = v.pzf;
  op_rows<false>(L.A, xf, [&](int i, const double* a) {
    const double wd = w * dinv[i];
    const float4 xi = __ldg(xf + i);
    const double* bi = b + 3 * (size_t)i;
    const double b0 = bi[0], b1 = bi[1], b2 = bi[2];
    const float4 z = f4(fma(wd, b0 - a[0], (double)xi.x), fma(wd, b1 - a[1], (double)xi.y),
                        fma(wd, b2 - a[2], (double)xi.z));
    zf[i] = z;
    acc[0] = fma(b0, (double)z.x, acc[0]);
    acc[1] = fma(b1, (double)z.y, acc[1]);
    acc[2] = fma(b2, (double)z.z, acc[2]);
  });
  block_sum<3>(acc, red);
  if (threadIdx.x == 0) {
    double* pp = v.part_p + (size_t)blockIdx.x * 8;
    for (int k = 0; k < 3; ++k) pp[k] = acc[k];
  }
  if (last_block(v.cnt_p, 3, 0, v.n_inst, gridDim.x)) {
    __shared__ double tot[3];
    sum_partials(v.part_p, gridDim.x, 8, 3, tot);
    if (threadIdx.x == 0) {
      PcgCtl& p = v.pctl[0];
      const bool init = p.iter == 0;  // the V-cycle after k_pcg_init: beta stays 0
      for (int k = 0; k < 3; ++k) {
        if ((p.conv >> k) & 1) continue;
        p.beta[k] = init ? 0.0 : tot[k] / p.rz[k];
        p.rz[k] = tot[k];
      }
    }
  }
}

// r.z after a V-cycle: init -> rz (beta stays 0); else beta = rz_new / rz
__global__ void __launch_bounds__(kUpdThreads, kUpdBlocksPerSm) k_pcg_rz(SysView v, int init) {
  if (!amg_on(v)) return;
  __shared__ double red[3 * 32];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(t % 3);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, n3 = 3 * (int64_t)v.n_free;
  double rz = 0.0;
  for (int64_t e = t; e < n3; e += stride) rz = fma(v.pr[e], v.pz[e], rz);
  double acc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) acc[k] = k == c ? rz : 0.0;
  block_sum<3>(acc, red);
  if (threadIdx.x == 0) {
    double* pp = v.part_p + (size_t)blockIdx.x * 8;
    for (int k = 0; k < 3; ++k) pp[k] = acc[k];
  }
  if (last_block(v.cnt_p, 3, 0, v.n_inst, gridDim.x)) {
    __shared__ double tot[3];
    sum_partials(v.part_p, gridDim.x, 8, 3, tot);
    if (threadIdx.x == 0) {
      PcgCtl& p = v.pctl[0];
      for (int k = 0; k < 3; ++k) {
        if ((p.conv >> k) & 1) continue;
        p.beta[k] = init ? 0.0 : tot[k] / p.rz[k];
        p.rz[k] = tot[k];
      }
    }
  }
}

// stand-alone timing of the CG's SpMV (qn_system_time_kernel "spmv"): the CG's own kernel (q = A p
// with p = z + beta p_old formed in the neighbour loads, p and q written, p.q partials), forced on
// between frames; k_pcg_init resets everything it touches
int launch_spmv_timing(qn_system* S, cudaStream_t st) {
  const SysView& v = S->v;
  if (v.pcg == 2 && v.pzf)
    if (S->pcg_rec)
      k_pcg_spmv_rec<<<v.nblk_spmv, kSpmvThreads, 0, st>>>(v, 1);
    else
      k_pcg_spmv<true><<<dim3(v.nblk_spmv, v.n_inst), kSpmvThreads, 0, st>>>(v, 1);
  else
    k_pcg_spmv<false><<<dim3(v.nblk_spmv, v.n_inst), kSpmvThreads, 0, st>>>(v, 1);
  QN_CHECK_LAUNCH();
  return QN_OK;
}

// Several systems (e.g. the slabs held by one process) stage coarse levels of
// different sizes: the kernel's dynamic shared-memory limit only ever grows.
// Called before any graph capture (prepare_kernels) and before direct launches.
static int ensure_coarse_smem(int nc) {
  static std::mutex mu;
  static int smem_set = 0;
  const int need = (int)(3 * sizeof(double) * nc);
  std::lock_guard<std::mutex> lock(mu);
  if (need > smem_set) {
    QN_CUDA(cudaFuncSetAttribute(k_amg_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, need));
    smem_set = need;
  }
  return QN_OK;
}

int launch_vcycle(qn_system* S, cudaStream_t st) {
  const SysView& v = S->v;
  const int nl = (int)S->h_alev.size();
  const int lt = S->amg_tail_level > 0 ? S->amg_tail_level : nl;  // levels lt .. coarsest run in k_amg_tail
  k_amg_presmooth<<<S->v.nblk_upd, kUpdThreads, 0, st>>>(v);
  QN_CHECK_LAUNCH();
  for (int l = 0; l + 1 < nl && l < lt; ++l) {
    const auto& L = S->h_alev[l];
    k_amg_residual<<<L.A.nblk, kSpmvThreads, 0, st>>>(v, l);
    QN_CHECK_LAUNCH();
    k_amg_restrict<<<L.R.nblk, kSpmvThreads, 0, st>>>(v, l);
    QN_CHECK_LAUNCH();
  }
  const int nc = v.ncoarse;
  if (lt < nl) {
    k_amg_tail<<<S->amg_tail_grid, kSpmvThreads, (size_t)3 * nc * sizeof(double), st>>>(v, lt);
  } else {
    if (int rc = ensure_coarse_smem(nc)) return rc;
    k_amg_coarse<<<std::max(1, std::min(2 * kSMs, div_up(nc, kSpmvWarps))), kSpmvThreads,
                   (size_t)3 * nc * sizeof(double), st>>>(v);
  }
  QN_CHECK_LAUNCH();
  for (int l = std::min(nl - 2, lt - 1); l >= 0; --l) {
    const auto& L = S->h_alev[l];
    k_amg_prolong<<<L.P.nblk, kSpmvThreads, 0, st>>>(v, l);
    QN_CHECK_LAUNCH();
    if (l == 0 && v.pzf)
      k_amg_smooth_rz<<<L.A.nblk, kSpmvThreads, 0, st>>>(v);
    else
      k_amg_smooth<<<L.A.nblk, kSpmvThreads, 0, st>>>(v, l);
    QN_CHECK_LAUNCH();
  }
  return QN_OK;
}

// The tail kernel's grid: every CTA resident (its phases meet at grid-wide barriers).  Levels with at
// most QN_AMG_TAIL_ROWS rows below the finest join the tail.  Experiment knob, off by default (0):
// measured neutral on configs[4] (V-cycle 1.104 ms with levels 3-5 in the tail vs 1.107 ms with
// their 13 separate graph nodes: inside the frame graph the small levels' launch boundaries cost
// almost nothing).
int prepare_amg_tail(qn_system* S) {
  S->amg_tail_level = 0;
  const int nl = (int)S->h_alev.size();
  if (S->v.pcg != 2 || nl < 3) return QN_OK;
  int64_t max_rows = 0;
  if (const char* e = std::getenv("QN_AMG_TAIL_ROWS")) max_rows = std::atoll(e);
  int lt = nl;
  for (int l = nl - 2; l >= 1 && S->h_alev[l].n <= max_rows; --l) lt = l;
  if (lt > nl - 2) return QN_OK;
  const size_t smem = (size_t)3 * S->v.ncoarse * sizeof(double);
  {  // several systems may stage coarse levels of different sizes: the limit only grows
    static std::mutex mu;
    static size_t smem_set = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (smem > smem_set) {
      QN_CUDA(cudaFuncSetAttribute(k_amg_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      smem_set = smem;
    }
  }
  int per = 0, dev = 0, sms = 0;
  QN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_amg_tail, kSpmvThreads, smem));
  QN_CUDA(cudaGetDevice(&dev));
  QN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per < 1) return QN_OK;
  S->amg_tail_grid = std::min(per, kSpmvBlocksPerSm) * sms;
  S->amg_tail_level = lt;
  return QN_OK;
}

int launch_pcg_rz(qn_system* S, int init, cudaStream_t st) {
  if (S->v.pzf) return QN_OK;  // fused into the V-cycle's last kernel (k_amg_smooth_rz)
  k_pcg_rz<<<S->v.nblk_upd, kUpdThreads, 0, st>>>(S->v, init);
  QN_CHECK_LAUNCH();
  return QN_OK;
}

__global__ void __launch_bounds__(kPT) k_pcg_store(SysView v) {
  const int b = blockIdx.y;
  if (v.ctl[b].phase != PH_DIR) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.n_free) return;
  const double* x = v.px + ((size_t)b * v.n_free + i) * 3;
  double* r = v.R0 + inst_off(v, b) + (size_t)v.fact_vtx[i] * 3;
  r[0] = x[0];
  r[1] = x[1];
  r[2] = x[2];
}

// ---------------------------------------------------------------------------
// host: body launch / graph

// body pass = pre (gradient, then the direct solve or the PCG set-up)
//           [+ PCG iterations] + post (eta, direction / trial, tet pass)
int launch_body_pre(qn_system* S, cudaStream_t st) {
  const SysView& v = S->v;
  const dim3 gv(v.nblk_v, v.n_inst);
  if (int rc = launch_col(S, 0, st)) return rc;
  if (S->h_cfg.m <= 5) {  // default window: smaller register footprint
    launch_k(k_grad<5>, gv, dim3(v.vt), 0, st, S->pdl, v);
  } else {
    launch_k(k_grad<kMaxM>, gv, dim3(v.vt), 0, st, S->pdl, v);
  }
  QN_CHECK_LAUNCH();
  if (v.pcg) {
    k_pcg_init<<<dim3(v.nblk_p, v.n_inst), kPT, 0, st>>>(v);
    QN_CHECK_LAUNCH();
    if (v.pcg == 2) {  // z0 = B r0, rz0
      int rc = launch_vcycle(S, st);
      return rc ? rc : launch_pcg_rz(S, 1, st);
    }
    return QN_OK;
  }
  if (S->h_cfg.lbfgs_init == 1) {
    k_scaled<<<gv, v.vt, 0, st>>>(v);
    QN_CHECK_LAUNCH();
    return QN_OK;
  }
  if (S->h_cfg.lbfgs_init == 2) {
    k_rest_rhs<<<div_up(std::max<int64_t>(3 * (int64_t)v.n, v.nf3), kVT), kVT, 0, st>>>(v);
    QN_CHECK_LAUNCH();
    k_rest_apply<<<std::max(1, std::min(4 * kSMs, div_up(v.nf3, 8))), 256, 0, st>>>(v);
    QN_CHECK_LAUNCH();
    return QN_OK;
  }
  // batched (one CTA per instance: every row's rhs is formed exactly once) and
  // latency-bound factors (few tasks per CTA, c2: the extra kernel node costs
  // more than the redundant row loads) form the rhs inside the solve
  if (S->factor->batch_smem > 0 || !S->factor->many_tasks) {
    SolverIO io{v};
    return launch_solve(S->factor, io, st);
  }
  launch_k(k_solve_rhs, dim3(div_up(3 * (int64_t)v.n_free, kVTB), v.n_inst), dim3(kVTB), 0, st, S->pdl, v);
  QN_CHECK_LAUNCH();
  FactorRhsIO io{{v}};
  return launch_solve(S->factor, io, st);
}

int launch_pcg_iter(qn_system* S, cudaStream_t st) {
  const SysView& v = S->v;
  if (v.pcg == 2 && v.pzf)
    if (S->pcg_rec)
      k_pcg_spmv_rec<<<v.nblk_spmv, kSpmvThreads, 0, st>>>(v, 0);
    else
      k_pcg_spmv<true><<<dim3(v.nblk_spmv, v.n_inst), kSpmvThreads, 0, st>>>(v, 0);
  else
    k_pcg_spmv<false><<<dim3(v.nblk_spmv, v.n_inst), kSpmvThreads, 0, st>>>(v, 0);
  QN_CHECK_LAUNCH();
  k_pcg_update<<<dim3(v.nblk_upd, v.n_inst), kUpdThreads, 0, st>>>(v);
  QN_CHECK_LAUNCH();
  if (v.pcg == 2) {  // z = B r, beta = r.z / r.z_old
    int rc = launch_vcycle(S, st);
    return rc ? rc : launch_pcg_rz(S, 0, st);
  }
  return QN_OK;
}

int launch_body_post(qn_system* S, cudaStream_t st) {
  const SysView& v = S->v;
  const dim3 gv(v.nblk_v, v.n_inst), gt(v.nblk_t, v.n_inst);
  const bool small_m = S->h_cfg.m <= 5;
  if (v.pcg) {
    k_pcg_store<<<dim3(v.nblk_p, v.n_inst), kPT, 0, st>>>(v);
    QN_CHECK_LAUNCH();
  }
  if (small_m) {
    launch_k(k_eta<5>, gv, dim3(v.vt), 0, st, S->pdl, v);
  } else {
    launch_k(k_eta<kMaxM>, gv, dim3(v.vt), 0, st, S->pdl, v);
  }
  QN_CHECK_LAUNCH();
  launch_k(k_vec, gv, dim3(v.vt), 0, st, S->pdl, v);
  QN_CHECK_LAUNCH();
  if (int rc = launch_col(S, 1, st)) return rc;
  if (v.n_mat <= kMatSmem) {
    if (v.f32) {
      launch_k(k_tet<true, false, true>, gt, dim3(kTT), 0, st, S->pdl, v);
    } else if (v.aniso) {
      launch_k(k_tet<true, true>, gt, dim3(kTT), 0, st, S->pdl, v);
    } else {
      launch_k(k_tet<true, false>, gt, dim3(kTT), 0, st, S->pdl, v);
    }
  } else if (v.f32) {
    launch_k(k_tet<false, false, true>, gt, dim3(kTT), 0, st, S->pdl, v);
  } else if (v.aniso) {
    launch_k(k_tet<false, true>, gt, dim3(kTT), 0, st, S->pdl, v);
  } else {
    launch_k(k_tet<false, false>, gt, dim3(kTT), 0, st, S->pdl, v);
  }
  QN_CHECK_LAUNCH();
  return QN_OK;
}

// host-driven body (no graph): PCG iterations loop with a host read per iteration
int launch_body(qn_system* S, cudaStream_t st) {
  int rc = launch_body_pre(S, st);
  if (rc) return rc;
  if (S->v.pcg) {
    for (int it = 0; it < S->v.pcg_maxit; ++it) {
      int32_t act = 0;
      QN_CUDA(cudaMemcpyAsync(&act, S->v.pcg_active, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      QN_CUDA(cudaStreamSynchronize(st));
      if (act <= 0) break;
      if ((rc = launch_pcg_iter(S, st))) return rc;
    }
  }
  return launch_body_post(S, st);
}

int launch_tet_plain(qn_system* S, const double* x, int b, int mat_sel, double* part, cudaStream_t st) {
  const SysView& v = S->v;
  const dim3 g(v.nblk_t, b < 0 ? v.n_inst : 1);
  if (v.n_mat <= kMatSmem) {
    if (v.f32) {
      k_tet_plain<true, false, true><<<g, kTT, 0, st>>>(v, x, b, mat_sel, part);
    } else if (v.aniso) {
      k_tet_plain<true, true><<<g, kTT, 0, st>>>(v, x, b, mat_sel, part);
    } else {
      k_tet_plain<true, false><<<g, kTT, 0, st>>>(v, x, b, mat_sel, part);
    }
  } else if (v.f32) {
    k_tet_plain<false, false, true><<<g, kTT, 0, st>>>(v, x, b, mat_sel, part);
  } else if (v.aniso) {
    k_tet_plain<false, true><<<g, kTT, 0, st>>>(v, x, b, mat_sel, part);
  } else {
    k_tet_plain<false, false><<<g, kTT, 0, st>>>(v, x, b, mat_sel, part);
  }
  QN_CHECK_LAUNCH();
  return QN_OK;
}

int launch_init(qn_system* S, cudaStream_t st) {
  const dim3 gv(S->v.nblk_v, S->v.n_inst);
  k_init<<<gv, S->v.vt, 0, st>>>(S->v);
  QN_CHECK_LAUNCH();
  return QN_OK;
}

int launch_finish(qn_system* S, cudaStream_t st) {
  const dim3 gv(S->v.nblk_v, S->v.n_inst);
  k_finish<<<gv, S->v.vt, 0, st>>>(S->v);
  QN_CHECK_LAUNCH();
  return QN_OK;
}

int prepare_kernels(qn_system* S) {
  if (S->v.pcg == 2) {
    if (int rc = ensure_coarse_smem(S->v.ncoarse)) return rc;
    if (int rc = prepare_amg_tail(S)) return rc;
  }
  if (!S->factor) return QN_OK;
  int rc = prepare_solve_kernels<SolverIO>(S->factor);
  if (!rc) rc = prepare_solve_kernels<FactorRhsIO>(S->factor);
  return rc ? rc : prepare_solve_kernels<TimingIO>(S->factor);
}

// kernel nodes of a (sub)graph, for launch accounting only: any query error
// is cleared so it cannot surface at the next launch check
static int64_t kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  int64_t k = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) == cudaSuccess && n > 0) {
    std::vector<cudaGraphNode_t> nodes(n);
    if (cudaGraphGetNodes(g, nodes.data(), &n) == cudaSuccess)
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
      }
  }
  (void)cudaGetLastError();
  return k;
}

int build_graph(qn_system* S) {
  CaptureScope capture_scope;  // launches while capturing are nodes, not executions
  cudaStream_t st = S->stream;
  if (S->exec) {
    cudaGraphExecDestroy(S->exec);
    S->exec = nullptr;
  }
  if (S->graph) {
    cudaGraphDestroy(S->graph);
    S->graph = nullptr;
  }
  cudaGraph_t g;
  QN_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  QN_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  S->v.handle = h;
  // init
  QN_CUDA(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int rc = launch_init(S, st);
  cudaGraph_t tmp;
  QN_CUDA(cudaStreamEndCapture(st, &tmp));
  if (rc) return rc;
  size_t nn = 0;
  QN_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
  QN_REQUIRE(nn == 1, QN_ERR_CUDA, "graph: unexpected init capture");
  cudaGraphNode_t init_node;
  QN_CUDA(cudaGraphGetNodes(g, &init_node, &nn));
  // WHILE(active) { body }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond;
  QN_CUDA(cudaGraphAddNode(&cond, g, &init_node, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (!S->v.pcg) {
    // kBodyUnroll passes per WHILE iteration: the loop edge (~6 us) is paid
    // once per kBodyUnroll passes; a pass after every instance is done is a
    // no-op in every kernel (phase checks), so the extra pass at the end of
    // a frame only costs its launches
    QN_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (int u = 0; u < kBodyUnroll && rc == QN_OK; ++u) {
      rc = launch_body_pre(S, st);
      if (rc == QN_OK) rc = launch_body_post(S, st);
    }
    QN_CUDA(cudaStreamEndCapture(st, &body));
    if (rc) return rc;
    S->kernels_per_pass = kernel_nodes(body) / kBodyUnroll;
    S->kernels_per_cg = 0;
  } else {
    // pre -> WHILE(pcg active){ spmv, update } -> post, all inside the body
    cudaGraphConditionalHandle hp;
    QN_CUDA(cudaGraphConditionalHandleCreate(&hp, body, 0, 0));
    S->v.pcg_handle = hp;
    QN_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    rc = launch_body_pre(S, st);
    cudaGraph_t tmpb;
    QN_CUDA(cudaStreamEndCapture(st, &tmpb));
    if (rc) return rc;
    // leaf of the captured chain
    size_t nb = 0;
    QN_CUDA(cudaGraphGetNodes(body, nullptr, &nb));
    std::vector<cudaGraphNode_t> nodes(nb);
    QN_CUDA(cudaGraphGetNodes(body, nodes.data(), &nb));
    cudaGraphNode_t leaf = nullptr;
    for (cudaGraphNode_t nd : nodes) {
      size_t ndep = 0;
      QN_CUDA(cudaGraphNodeGetDependentNodes(nd, nullptr, &ndep));
      if (ndep == 0) leaf = nd;
    }
    QN_REQUIRE(leaf != nullptr, QN_ERR_CUDA, "graph: no leaf in the PCG pre-segment");
    cudaGraphNodeParams ci = {};
    ci.type = cudaGraphNodeTypeConditional;
    ci.conditional.handle = hp;
    ci.conditional.type = cudaGraphCondTypeWhile;
    ci.conditional.size = 1;
    cudaGraphNode_t pcond;
    QN_CUDA(cudaGraphAddNode(&pcond, body, &leaf, 1, &ci));
    cudaGraph_t ibody = ci.conditional.phGraph_out[0];
    QN_CUDA(cudaStreamBeginCaptureToGraph(st, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    rc = launch_pcg_iter(S, st);
    QN_CUDA(cudaStreamEndCapture(st, &ibody));
    if (rc) return rc;
    QN_CUDA(cudaStreamBeginCaptureToGraph(st, body, &pcond, nullptr, 1, cudaStreamCaptureModeThreadLocal));
    rc = launch_body_post(S, st);
    QN_CUDA(cudaStreamEndCapture(st, &tmpb));
    if (rc) return rc;
    S->kernels_per_pass = kernel_nodes(body);
    S->kernels_per_cg = kernel_nodes(ibody);
  }
  // finish
  QN_CUDA(cudaStreamBeginCaptureToGraph(st, g, &cond, nullptr, 1, cudaStreamCaptureModeThreadLocal));
  rc = launch_finish(S, st);
  QN_CUDA(cudaStreamEndCapture(st, &g));
  if (rc) return rc;
  QN_CUDA(cudaGraphInstantiate(&S->exec, g, 0));
  S->graph = g;
  return QN_OK;
}

}  // namespace qn

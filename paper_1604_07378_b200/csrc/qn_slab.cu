// Slab-decomposed frame for one mesh split across ranks (configs[4],
// SURVEY.md §8e): element-slab partition along x with a one-cell ghost layer,
// a one-plane halo exchange per CG iteration and per direction, and global
// sums of every dot product / energy.  The per-rank arithmetic is the same
// as the single-system frame (solvers.py:260-352): gradient gather in the
// reference's element order, L-BFGS two-loop in Gram form, CG on A_free to
// ||r|| <= tol ||b|| per coordinate, Armijo backtracking.
//
// Layout of rank r with own cells [c0, c1):
//   local cells  [c0 - 1 (r > 0), c1)      local tets: ghost layer first (global order)
//   local planes [c0 - 1 (r > 0), c1]      local vertex ids = global ids - first plane
//   owned planes [c0, c1) (+ plane nx on the last rank): a contiguous local range
// Every owned vertex sees all its incident tets locally, so its gradient is
// the single-system gradient bit for bit (same element order).  Ghost planes
// carry copies of the neighbours' owned values (positions, directions,
// search vectors); vector updates run over every local vertex, dot products
// and energies over owned vertices / tets only.
//
// Global sums are all-gathers of each rank's fixed-order partial sums
// (`send`, kSlabSend doubles) into `gath` [ranks][kSlabSend]; every consumer
// adds the ranks in index order, so every rank computes identical scalars
// (and the in-process emulation of several ranks on one device is bitwise
// the multi-GPU result).  The collectives themselves (NCCL all-gather and
// send/recv on torch tensors wrapping these buffers) are issued by the host
// between the stages below (paper_1604_07378_b200/slab.py), stream-ordered.
#include <algorithm>
#include <cstring>
#include <vector>

#include "qn_kernels.cuh"

extern "C" void sell_build(int64_t nrows, int64_t ncols, const int64_t* ptr, const int32_t* col,
                           const double* val, int64_t ni, int64_t nnz, std::vector<int64_t>& sptr,
                           std::vector<int32_t>& scol, std::vector<double>& sval);  // qn_api.cu

namespace qn {

int launch_vcycle(qn_system* S, cudaStream_t st);

constexpr int kSlabMaxM = 8;          // history window bound of the slab frame
constexpr int kSlabSend = 32;         // doubles per rank in one all-gather
constexpr int kSlabVT = 256;          // vertex-kernel block
constexpr int kSlabRing = kSlabMaxM + 1;
constexpr int kSlabGradVals = 4 + 2 * kSlabMaxM + 1;  // gg, st, ss, tt, <s_j,t>, <s_j,g>, <s_new,g>
constexpr int kSlabSellUnroll = 8;

struct SlabPcg {
  double rz[3], bb[3], alpha[3];
  double rzc[3];                   // <r_c, A_c^-1 r_c> of the coarse correction (two-level preconditioner)
  int32_t conv, iter, total, pad;  // conv: bit c = column c converged, bit 3 = all done
};

struct SlabArgs {  // per-stage scalars passed by value
  int32_t xs, xs_to, have_prev, new_slot, nring, first;
  int32_t ring[kSlabRing];  // slot ids, oldest -> newest
  double coef[kSlabRing];   // zeta (PCG set-up) or zeta - eta (direction), by ring position
  double alpha;
};

struct SlabView {
  SysView v;  // the slab-local system: tets, Dm^-1, vols, materials, gather map, masses, forces, AMG levels
  int32_t n, mt, tet_own_lo, own_lo, own_hi, nf, G, amg;
  int32_t nblk_all, nblk_own, nblk_t, nblk_f, nblk_spmv, pcg_maxit, nblk_max, nblk_flat;
  double pcg_tol;
  const uint8_t* pinned;  // [n]
  const int32_t* f2v;     // [nf] owned free row -> local vertex
  const int32_t* v2f;     // [n] local vertex -> owned free row or -1
  double* q_l;            // [n][3]
  double* q_prev;
  double* y;
  double* X;              // [2][n][3] current / trial positions
  double* g;
  double* xp;             // previous iterate and gradient (L-BFGS push)
  double* gp;
  double* d;
  double* r0;             // A_free^-1 q in vertex layout (ghost planes exchanged)
  double* S;              // [kSlabRing][n][3]
  double* T;
  SellDev A;              // owned free rows x local non-pinned vertices (column = local vertex id)
  const double* dinv;     // [nf] Jacobi
  double* px;             // [nf][3]
  double* pr;
  double* pz;
  double* pq;
  double* pv;             // [n][3] search direction in vertex layout (halo-exchanged)
  double* part;           // [8][maxblk][kSlabSend]
  unsigned* cnt;          // [8]
  double* send;           // [kSlabSend]
  const double* gath;     // [G][kSlabSend]
  SlabPcg* pc;
  // two-level additive preconditioner: z += P_c A_c^-1 P_c^T r with P_c the
  // trilinear hat functions of a coarse grid of the bar (separable, applied
  // dimension by dimension; every rank holds A_c^-1)
  int32_t nc, gx, gy, gz;     // coarse nodes; fine grid cells per dimension
  int32_t cx, cy, cz, npl;    // coarse nodes per dimension; owned x-planes of this rank
  int32_t i_lo, v0;           // first owned x-plane (global), global id of local vertex 0
  const int32_t* hI[3];       // per dimension and fine index: first coarse node of its cell
  const double* hw[3];        // per dimension and fine index: weights (node I, node I+1)
  const int32_t* hpos[3];     // per dimension: fine index of each coarse node
  const double* cinv;         // [nc][nc]
  double* t0;                 // [npl][gy+1][cz][3] restricted along z
  double* t1;                 // [npl][cy][cz][3] restricted along z and y
  double* csend;              // [nc][3] this rank's P_c^T r
  const double* cgath;        // [G][nc][3]
  double* ec;                 // [nc][3] A_c^-1 (sum over ranks of P_c^T r)
};

__device__ __forceinline__ double* part_of(const SlabView& s, int which) {
  return s.part + (size_t)which * s.nblk_max * kSlabSend;
}

// sum over ranks (index order) of gathered value k
__device__ __forceinline__ double gsum(const SlabView& s, int k) {
  double a = 0.0;
  for (int r = 0; r < s.G; ++r) a += s.gath[r * kSlabSend + k];
  return a;
}

// block partials of K values -> the last block adds them in block order into send[off..off+K)
template <int K>
__device__ __forceinline__ void finish_sum(const SlabView& s, double (&acc)[K], int which, int off, int nval = K) {
  __shared__ double red[K * 32];
  block_sum<K>(acc, red);
  double* part = part_of(s, which);
  if (threadIdx.x == 0)
    for (int k = 0; k < K; ++k) part[(size_t)blockIdx.x * kSlabSend + k] = acc[k];
  if (last_block(s.cnt, which, 0, 1, gridDim.x)) {
    __shared__ double tot[K];
    sum_partials(part, gridDim.x, kSlabSend, nval, tot);
    if (threadIdx.x < nval) s.send[off + threadIdx.x] = tot[threadIdx.x];
  }
}

// ---- frame init: y = 2 q_l - q_prev + h^2 g, pinned rows = q_l; x = y (dynamics.py:437-443)
__global__ void __launch_bounds__(kSlabVT) k_slab_init(SlabView s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const size_t o = (size_t)i * 3;
  double y[3];
  if (s.pinned[i]) {
    for (int a = 0; a < 3; ++a) y[a] = s.q_l[o + a];
  } else {
    const double hh = __dmul_rn(s.v.h, s.v.h);
    for (int a = 0; a < 3; ++a)
      y[a] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, s.q_l[o + a]), s.q_prev[o + a]), __dmul_rn(hh, s.v.grav[a]));
  }
  for (int a = 0; a < 3; ++a) {
    s.y[o + a] = y[a];
    s.X[o + a] = y[a];
  }
}

// ---- objective at X[xs] (dynamics.py:460-467): per-tet pass over every local
// tet (corner forces for the gradient), energy of the owned tets -> send[0]
template <bool kSm>
__global__ void __launch_bounds__(kTT, kTetBlocksPerSm) k_slab_tet(SlabView s, int xs) {
  __shared__ qn_material smat[kMatSmem];
  __shared__ double fsm[kTT * kFStride];
  double e[1] = {0.0};
  const SysView& v = s.v;
  if (v.mt > 0) {
    const qn_material* mats = stage_materials<kSm>(v, 0, smat);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const double et = tet_thread(v, s.X + (size_t)xs * s.n * 3, 0, t, mats, -1, fsm);
    e[0] = t >= s.tet_own_lo ? et : 0.0;
    store_forces(v, 0, fsm);
  }
  finish_sum<1>(s, e, 0, 0);
}

// inertia sum_v m_v |x_v - y_v|^2 over owned vertices -> send[1]
__global__ void __launch_bounds__(kSlabVT) k_slab_inertia(SlabView s, int xs) {
  const int i = s.own_lo + blockIdx.x * blockDim.x + threadIdx.x;
  double e[1] = {0.0};
  if (i < s.own_hi) {
    const double* x = s.X + (size_t)xs * s.n * 3 + (size_t)i * 3;
    const double* y = s.y + (size_t)i * 3;
    const double d0 = x[0] - y[0], d1 = x[1] - y[1], d2 = x[2] - y[2];
    e[0] = s.v.masses[i] * (d0 * d0 + d1 * d1 + d2 * d2);
  }
  finish_sum<1>(s, e, 1, 1);
}

// ---- gradient at X[xs] (dynamics.py:470-478) for every local vertex
// (inertia, then corner forces in element order, pinned rows zeroed), the
// L-BFGS pair s = x - x_prev, t = g - g_prev into ring slot new_slot
// (solvers.py:289-291), and the owned dot products:
//   send[0] <g,g>  [1] <s,t>  [2] <s,s>  [3] <t,t>
//   send[4 + j] <s_ring[j], t>   send[4 + M + j] <s_ring[j], g>   send[4 + 2M] <s, g>
__global__ void __launch_bounds__(kSlabVT) k_slab_grad(SlabView s, SlabArgs a) {
  constexpr int K = kSlabGradVals;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.n) {
    const SysView& v = s.v;
    const size_t o = (size_t)i * 3;
    const double* x = s.X + (size_t)a.xs * s.n * 3 + o;
    double g[3];
    const double w = __ldg(v.w_in + i);
    for (int c = 0; c < 3; ++c) g[c] = __dmul_rn(w, __dsub_rn(x[c], s.y[o + c]));
    for (int k = v.v2e_ptr[i]; k < v.v2e_ptr[i + 1]; ++k) {
      const double* f = v.forces + (size_t)k * 3;  // gather order
      for (int c = 0; c < 3; ++c) g[c] = __dadd_rn(g[c], f[c]);
    }
    if (s.pinned[i]) g[0] = g[1] = g[2] = 0.0;
    double sn[3] = {0, 0, 0}, tn[3] = {0, 0, 0};
    if (a.have_prev) {
      double* Sn = s.S + (size_t)a.new_slot * s.n * 3 + o;
      double* Tn = s.T + (size_t)a.new_slot * s.n * 3 + o;
      for (int c = 0; c < 3; ++c) {
        sn[c] = x[c] - s.xp[o + c];
        tn[c] = g[c] - s.gp[o + c];
        Sn[c] = sn[c];
        Tn[c] = tn[c];
      }
    }
    for (int c = 0; c < 3; ++c) {
      s.g[o + c] = g[c];
      s.xp[o + c] = x[c];
      s.gp[o + c] = g[c];
    }
    if (i >= s.own_lo && i < s.own_hi) {
      acc[0] = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
      if (a.have_prev) {
        acc[1] = sn[0] * tn[0] + sn[1] * tn[1] + sn[2] * tn[2];
        acc[2] = sn[0] * sn[0] + sn[1] * sn[1] + sn[2] * sn[2];
        acc[3] = tn[0] * tn[0] + tn[1] * tn[1] + tn[2] * tn[2];
        acc[4 + 2 * kSlabMaxM] = sn[0] * g[0] + sn[1] * g[1] + sn[2] * g[2];
      }
      for (int j = 0; j < a.nring; ++j) {
        const double* Sj = s.S + (size_t)a.ring[j] * s.n * 3 + o;
        const double s0 = Sj[0], s1 = Sj[1], s2 = Sj[2];
        acc[4 + j] = s0 * tn[0] + s1 * tn[1] + s2 * tn[2];
        acc[4 + kSlabMaxM + j] = s0 * g[0] + s1 * g[1] + s2 * g[2];
      }
    }
  }
  finish_sum<K>(s, acc, 2, 0);
}

// ---- direction set-up (solvers.py:124-134): q = -g - sum_{newest..oldest} zeta_j t_j
// on the owned free rows, CG start x = 0, r = b = q.  Jacobi: z = D^-1 r.
//   send[0..2] <b,b> per column, send[3..5] <r,z> (Jacobi only)
__global__ void __launch_bounds__(kSlabVT) k_slab_pcg_setup(SlabView s, SlabArgs a) {
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < s.nf) {
    const int i = s.f2v[f];
    const size_t o = (size_t)i * 3, fo = (size_t)f * 3;
    double q[3];
    for (int c = 0; c < 3; ++c) q[c] = -s.g[o + c];
    for (int j = a.nring - 1; j >= 0; --j) {
      const double* Tj = s.T + (size_t)a.ring[j] * s.n * 3 + o;
      for (int c = 0; c < 3; ++c) q[c] = __dsub_rn(q[c], __dmul_rn(a.coef[j], Tj[c]));
    }
    const double di = s.amg ? 0.0 : s.dinv[f];
    for (int c = 0; c < 3; ++c) {
      s.px[fo + c] = 0.0;
      s.pr[fo + c] = q[c];
      acc[c] = q[c] * q[c];
      if (!s.amg) {
        const double z = q[c] * di;
        s.pz[fo + c] = z;
        acc[3 + c] = q[c] * z;
      }
    }
  }
  finish_sum<6>(s, acc, 3, 0);
}

// The CG vector kernels run over the flattened (row, coordinate) elements
// e = 3 f + c of the owned free rows, grid-stride with a stride that is a
// multiple of 3 (kSlabFT), so a thread keeps its coordinate c; the vertex-
// layout search vector is addressed through f2v.
constexpr int kSlabFT = 384;
constexpr int kSlabFU = 4;  // elements in flight per thread

// <r, z> after a V-cycle -> send[3..5]
__global__ void __launch_bounds__(kSlabFT) k_slab_rz(SlabView s) {
  if (s.pc->conv & 8) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(t % 3);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, n3 = 3 * (int64_t)s.nf;
  double rz = 0.0;
  for (int64_t e = t; e < n3; e += stride) rz = fma(s.pr[e], s.pz[e], rz);
  double acc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) acc[k] = k == c ? rz : 0.0;
  finish_sum<3>(s, acc, 4, 3);
}

// ---- CG direction p = z + beta p (first: p = z) from the gathered sums:
// first: gath = [bb, rz]; later: gath = [rr, rz_new].  Columns whose
// residual reached tol ||b|| freeze (the single-system rule).  The last
// block commits the scalars.
__global__ void __launch_bounds__(kSlabFT) k_slab_pcg_p(SlabView s, int first) {
  const SlabPcg pc = *s.pc;
  if (pc.conv & 8) return;
  double rz[3], beta[3], bb[3];
  int conv = pc.conv;
  const double tol2 = s.pcg_tol * s.pcg_tol;
  for (int c = 0; c < 3; ++c) {
    // <r, z> = sum_ranks <r, B_slab r> (+ <r_c, A_c^-1 r_c>: the coarse term, known to every rank)
    const double a0 = gsum(s, c), a1 = s.nc > 0 ? gsum(s, 3 + c) + pc.rzc[c] : gsum(s, 3 + c);
    rz[c] = a1;
    if (first) {
      bb[c] = a0;
      beta[c] = 0.0;
      if (!(a0 > 0.0)) conv |= 1 << c;  // zero right-hand side
    } else {
      bb[c] = pc.bb[c];
      beta[c] = (conv >> c) & 1 ? 0.0 : a1 / pc.rz[c];
      if (!((conv >> c) & 1) && a0 <= tol2 * pc.bb[c]) conv |= 1 << c;
    }
  }
  const bool done = (conv & 7) == 7 || (!first && pc.iter >= s.pcg_maxit);
  if (!done) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = (int)(t % 3);
    const double be = beta[c];
    const bool frozen = (conv >> c) & 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, n3 = 3 * (int64_t)s.nf;
    if (!frozen) {
      int64_t e = t;
      for (; e + (kSlabFU - 1) * stride < n3; e += kSlabFU * stride) {
        double z[kSlabFU], pv[kSlabFU];
        int64_t o[kSlabFU];
#pragma unroll
        for (int u = 0; u < kSlabFU; ++u) {
          const int64_t f = e + u * stride;
          o[u] = 3 * (int64_t)__ldg(s.f2v + f / 3) + c;
          z[u] = s.pz[f];
          pv[u] = first ? 0.0 : s.pv[o[u]];
        }
#pragma unroll
        for (int u = 0; u < kSlabFU; ++u) s.pv[o[u]] = first ? z[u] : fma(be, pv[u], z[u]);
      }
      for (; e < n3; e += stride) {
        const int64_t o = 3 * (int64_t)__ldg(s.f2v + e / 3) + c;
        s.pv[o] = first ? s.pz[e] : fma(be, s.pv[o], s.pz[e]);
      }
    }
  }
  if (last_block(s.cnt, 5, 0, 1, gridDim.x) && threadIdx.x == 0) {
    SlabPcg& p = *s.pc;
    for (int c = 0; c < 3; ++c) {
      if (first) p.bb[c] = bb[c];
      if (!((pc.conv >> c) & 1)) p.rz[c] = rz[c];
    }
    if (first) p.iter = 0;
    p.conv = conv | (done ? 8 : 0);
  }
}

// ---- q = A p over the owned free rows (p in vertex layout incl. ghost planes);
// send[0..2] <p, q>.  One warp per 32-row SELL slice, lane = row.
__global__ void __launch_bounds__(kSpmvThreads) k_slab_spmv(SlabView s) {
  if (s.pc->conv & 8) return;
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5), nw = gridDim.x * kSpmvWarps;
  double acc[3] = {0, 0, 0};
  const double* __restrict__ P = s.pv;
  for (int sl = w0; sl < s.A.nslice; sl += nw) {
    const int64_t e0 = s.A.ptr[sl], e1 = s.A.ptr[sl + 1];
    double q0 = 0.0, q1 = 0.0, q2 = 0.0;
    int64_t e = e0 + lane;
    for (; e + 32 * (kSlabSellUnroll - 1) < e1; e += 32 * kSlabSellUnroll) {
      int j[kSlabSellUnroll];
      double av[kSlabSellUnroll];
#pragma unroll
      for (int u = 0; u < kSlabSellUnroll; ++u) {
        j[u] = __ldcs(s.A.col + e + 32 * u);
        av[u] = __ldcs(s.A.val + e + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < kSlabSellUnroll; ++u) {
        const double* pj = P + 3 * (size_t)j[u];
        q0 = fma(av[u], pj[0], q0);
        q1 = fma(av[u], pj[1], q1);
        q2 = fma(av[u], pj[2], q2);
      }
    }
    for (; e < e1; e += 32) {
      const int j = __ldcs(s.A.col + e);
      const double av = __ldcs(s.A.val + e);
      const double* pj = P + 3 * (size_t)j;
      q0 = fma(av, pj[0], q0);
      q1 = fma(av, pj[1], q1);
      q2 = fma(av, pj[2], q2);
    }
    const int f = 32 * sl + lane;
    if (f < s.nf) {
      const double* pi = P + 3 * (size_t)s.f2v[f];
      s.pq[3 * (size_t)f + 0] = q0;
      s.pq[3 * (size_t)f + 1] = q1;
      s.pq[3 * (size_t)f + 2] = q2;
      acc[0] = fma(pi[0], q0, acc[0]);
      acc[1] = fma(pi[1], q1, acc[1]);
      acc[2] = fma(pi[2], q2, acc[2]);
    }
  }
  finish_sum<3>(s, acc, 6, 0);
}

// ---- x += alpha p, r -= alpha q with alpha = rz / <p, q> (gathered);
// send[0..2] <r, r>; Jacobi: z = D^-1 r, send[3..5] <r, z>
__global__ void __launch_bounds__(kSlabFT) k_slab_pcg_update(SlabView s) {
  const SlabPcg pc = *s.pc;
  if (pc.conv & 8) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(t % 3);
  const double al = (pc.conv >> c) & 1 ? 0.0 : pc.rz[c] / gsum(s, c);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, n3 = 3 * (int64_t)s.nf;
  const bool jac = !s.amg;
  double rr = 0.0, rz = 0.0;
  int64_t e = t;
  for (; e + (kSlabFU - 1) * stride < n3; e += kSlabFU * stride) {
    double xv[kSlabFU], pv[kSlabFU], rv[kSlabFU], qv[kSlabFU], dv[kSlabFU];
#pragma unroll
    for (int u = 0; u < kSlabFU; ++u) {
      const int64_t f = e + u * stride;
      xv[u] = s.px[f];
      pv[u] = s.pv[3 * (int64_t)__ldg(s.f2v + f / 3) + c];
      rv[u] = s.pr[f];
      qv[u] = s.pq[f];
      dv[u] = jac ? __ldg(s.dinv + f / 3) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kSlabFU; ++u) {
      const int64_t f = e + u * stride;
      s.px[f] = fma(al, pv[u], xv[u]);
      const double rn = fma(-al, qv[u], rv[u]);
      s.pr[f] = rn;
      rr = fma(rn, rn, rr);
      if (jac) {
        const double z = rn * dv[u];
        s.pz[f] = z;
        rz = fma(rn, z, rz);
      }
    }
  }
  for (; e < n3; e += stride) {
    s.px[e] = fma(al, s.pv[3 * (int64_t)__ldg(s.f2v + e / 3) + c], s.px[e]);
    const double rn = fma(-al, s.pq[e], s.pr[e]);
    s.pr[e] = rn;
    rr = fma(rn, rn, rr);
    if (jac) {
      const double z = rn * __ldg(s.dinv + e / 3);
      s.pz[e] = z;
      rz = fma(rn, z, rz);
    }
  }
  double acc[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    acc[k] = k == c ? rr : 0.0;
    acc[3 + k] = k == c ? rz : 0.0;
  }
  finish_sum<6>(s, acc, 7, 0);
}

// ---- coarse correction (additive two-level Schwarz with the slabs' local
// preconditioners): r_c = sum_ranks P_c^T r, e_c = A_c^-1 r_c, z += P_c e_c.
// P_c^T r of this rank is applied separably: along z, then y, then x; each
// output sums its hat support in a fixed order (deterministic).

// weight of coarse node I (dimension d) at fine index i
__device__ __forceinline__ double hat_w(const SlabView& s, int d, int i, int I) {
  const int I0 = s.hI[d][i];
  return I0 == I ? s.hw[d][2 * i] : (I0 + 1 == I ? s.hw[d][2 * i + 1] : 0.0);
}
__device__ __forceinline__ void hat_range(const SlabView& s, int d, int I, int nmax, int& lo, int& hi) {
  const int nI = d == 0 ? s.cx : d == 1 ? s.cy : s.cz;
  lo = I > 0 ? s.hpos[d][I - 1] : 0;
  hi = I + 1 < nI ? s.hpos[d][I + 1] : nmax;  // inclusive
}

// t0[pl][j][K][c] = sum_k w_z(k, K) r(i_lo + pl, j, k, c)   (r = 0 on pinned / non-owned vertices)
__global__ void __launch_bounds__(kSlabVT) k_slab_coarse_z(SlabView s) {
  if (s.pc->conv & 8) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)s.npl * (s.gy + 1) * s.cz * 3;
  if (t >= total) return;
  const int c = (int)(t % 3);
  const int K = (int)((t / 3) % s.cz);
  const int j = (int)((t / (3 * s.cz)) % (s.gy + 1));
  const int pl = (int)(t / (3 * (int64_t)s.cz * (s.gy + 1)));
  const int plane = (s.gy + 1) * (s.gz + 1);
  const int64_t base = (int64_t)(s.i_lo + pl) * plane + (int64_t)j * (s.gz + 1) - s.v0;  // local id of (i, j, 0)
  int lo, hi;
  hat_range(s, 2, K, s.gz, lo, hi);
  double a = 0.0;
  for (int k = lo; k <= hi; ++k) {
    const int f = s.v2f[base + k];
    if (f >= 0) a = fma(hat_w(s, 2, k, K), s.pr[3 * (size_t)f + c], a);
  }
  s.t0[t] = a;
}

// t1[pl][J][K][c] = sum_j w_y(j, J) t0[pl][j][K][c]
__global__ void __launch_bounds__(kSlabVT) k_slab_coarse_y(SlabView s) {
  if (s.pc->conv & 8) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)s.npl * s.cy * s.cz * 3;
  if (t >= total) return;
  const int c = (int)(t % 3);
  const int K = (int)((t / 3) % s.cz);
  const int J = (int)((t / (3 * s.cz)) % s.cy);
  const int pl = (int)(t / (3 * (int64_t)s.cz * s.cy));
  int lo, hi;
  hat_range(s, 1, J, s.gy, lo, hi);
  double a = 0.0;
  for (int j = lo; j <= hi; ++j)
    a = fma(hat_w(s, 1, j, J), s.t0[(((int64_t)pl * (s.gy + 1) + j) * s.cz + K) * 3 + c], a);
  s.t1[t] = a;
}

// csend[I][J][K][c] = sum_{owned planes i} w_x(i, I) t1[i - i_lo][J][K][c]
__global__ void __launch_bounds__(kSlabVT) k_slab_coarse_x(SlabView s) {
  if (s.pc->conv & 8) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * s.nc) return;
  const int c = t % 3;
  const int K = (t / 3) % s.cz;
  const int J = (t / (3 * s.cz)) % s.cy;
  const int I = t / (3 * s.cz * s.cy);
  int lo, hi;
  hat_range(s, 0, I, s.gx, lo, hi);
  lo = max(lo, s.i_lo);
  hi = min(hi, s.i_lo + s.npl - 1);
  double a = 0.0;
  for (int i = lo; i <= hi; ++i)
    a = fma(hat_w(s, 0, i, I), s.t1[(((int64_t)(i - s.i_lo) * s.cy + J) * s.cz + K) * 3 + c], a);
  s.csend[t] = a;
}

// the ranks' restricted residuals summed in rank order into shared memory,
// then the dense coarse inverse, warp per coarse row
// <r_c, e_c> per column (one block, fixed order): the coarse part of <r, z>,
// identical on every rank (r_c is the rank-order sum of the gathered shares)
__global__ void __launch_bounds__(kSpmvThreads) k_slab_coarse_dot(SlabView s) {
  if (s.pc->conv & 8) return;
  __shared__ double red[kSpmvThreads / 32][3];
  const int n3 = 3 * s.nc;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int k = threadIdx.x; k < s.nc; k += blockDim.x)
    for (int c = 0; c < 3; ++c) {
      double rc = 0.0;
      for (int r = 0; r < s.G; ++r) rc += s.cgath[(size_t)r * n3 + 3 * k + c];
      acc[c] = fma(rc, s.ec[3 * (size_t)k + c], acc[c]);
    }
  for (int c = 0; c < 3; ++c) acc[c] = warp_sum(acc[c]);
  if ((threadIdx.x & 31) == 0)
    for (int c = 0; c < 3; ++c) red[threadIdx.x >> 5][c] = acc[c];
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < kSpmvThreads / 32; ++w) t += red[w][threadIdx.x];
    s.pc->rzc[threadIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kSpmvThreads) k_slab_coarse_solve(SlabView s) {
  if (s.pc->conv & 8) return;
  extern __shared__ double rcs[];
  const int n3 = 3 * s.nc;
  for (int q = threadIdx.x; q < n3; q += blockDim.x) {
    double a = 0.0;
    for (int r = 0; r < s.G; ++r) a += s.cgath[(size_t)r * n3 + q];
    rcs[q] = a;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5), nw = gridDim.x * kSpmvWarps;
  for (int k = w0; k < s.nc; k += nw) {
    const double* row = s.cinv + (size_t)k * s.nc;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int c = lane; c < s.nc; c += 32) {
      const double m = __ldg(row + c);
      a0 = fma(m, rcs[3 * c + 0], a0);
      a1 = fma(m, rcs[3 * c + 1], a1);
      a2 = fma(m, rcs[3 * c + 2], a2);
    }
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) {
      s.ec[3 * (size_t)k + 0] = a0;
      s.ec[3 * (size_t)k + 1] = a1;
      s.ec[3 * (size_t)k + 2] = a2;
    }
  }
}

// z += P_c e_c on the owned free rows: 8 trilinear terms per (row, coordinate)
__global__ void __launch_bounds__(kSlabFT) k_slab_coarse_p(SlabView s) {
  if (s.pc->conv & 8) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(t % 3);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, n3 = 3 * (int64_t)s.nf;
  const int plane = (s.gy + 1) * (s.gz + 1);
  for (int64_t e = t; e < n3; e += stride) {
    const int64_t gid = (int64_t)__ldg(s.f2v + e / 3) + s.v0;
    const int i = (int)(gid / plane), rem = (int)(gid % plane);
    const int j = rem / (s.gz + 1), k = rem % (s.gz + 1);
    const int Ix = s.hI[0][i], Iy = s.hI[1][j], Iz = s.hI[2][k];
    const double wx[2] = {s.hw[0][2 * i], s.hw[0][2 * i + 1]};
    const double wy[2] = {s.hw[1][2 * j], s.hw[1][2 * j + 1]};
    const double wz[2] = {s.hw[2][2 * k], s.hw[2][2 * k + 1]};
    double a = 0.0;
#pragma unroll
    for (int dx = 0; dx < 2; ++dx)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dz = 0; dz < 2; ++dz) {
          const double w = wx[dx] * wy[dy] * wz[dz];
          if (w != 0.0) a = fma(w, s.ec[(((size_t)(Ix + dx) * s.cy + (Iy + dy)) * s.cz + (Iz + dz)) * 3 + c], a);
        }
    s.pz[e] += a;
  }
}

__global__ void k_slab_pcg_count(SlabView s) {
  if (s.pc->conv & 8) return;
  s.pc->iter += 1;
  s.pc->total += 1;
}

// ---- r0 in vertex layout: CG solution on owned free rows, 0 elsewhere
// (fixed rows of the direction are zero, solvers.py:133-134); ghost planes
// are then overwritten by the halo exchange
__global__ void __launch_bounds__(kSlabVT) k_slab_store(SlabView s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const int f = s.v2f[i];
  for (int c = 0; c < 3; ++c) s.r0[(size_t)i * 3 + c] = f >= 0 ? s.px[(size_t)f * 3 + c] : 0.0;
}

// ---- second loop (solvers.py:136-141): send[j] = <t_ring[j], r0> over owned vertices
__global__ void __launch_bounds__(kSlabVT) k_slab_eta(SlabView s, SlabArgs a) {
  double acc[kSlabMaxM];
#pragma unroll
  for (int k = 0; k < kSlabMaxM; ++k) acc[k] = 0.0;
  const int i = s.own_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.own_hi) {
    const size_t o = (size_t)i * 3;
    const double r0 = s.r0[o], r1 = s.r0[o + 1], r2 = s.r0[o + 2];
    for (int j = 0; j < a.nring; ++j) {
      const double* Tj = s.T + (size_t)a.ring[j] * s.n * 3 + o;
      acc[j] = Tj[0] * r0 + Tj[1] * r1 + Tj[2] * r2;
    }
  }
  finish_sum<kSlabMaxM>(s, acc, 2, 0);
}

// ---- d = r0 + sum_{oldest..newest} s_j (zeta_j - eta_j) over every local
// vertex (reference rounding: mul, then add); send[0] = <g, d> over owned
__global__ void __launch_bounds__(kSlabVT) k_slab_dir(SlabView s, SlabArgs a) {
  double acc[1] = {0.0};
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.n) {
    const size_t o = (size_t)i * 3;
    double d[3];
    for (int c = 0; c < 3; ++c) d[c] = s.r0[o + c];
    for (int j = 0; j < a.nring; ++j) {
      const double* Sj = s.S + (size_t)a.ring[j] * s.n * 3 + o;
      for (int c = 0; c < 3; ++c) d[c] = __dadd_rn(d[c], __dmul_rn(Sj[c], a.coef[j]));
    }
    for (int c = 0; c < 3; ++c) s.d[o + c] = d[c];
    if (i >= s.own_lo && i < s.own_hi) acc[0] = s.g[o] * d[0] + s.g[o + 1] * d[1] + s.g[o + 2] * d[2];
  }
  finish_sum<1>(s, acc, 3, 0);
}

// ---- trial X[to] = X[from] + alpha d (solvers.py:252)
__global__ void __launch_bounds__(kSlabVT) k_slab_trial(SlabView s, int from, int to, double alpha) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3 * s.n) return;
  s.X[(size_t)to * s.n * 3 + e] = __dadd_rn(s.X[(size_t)from * s.n * 3 + e], __dmul_rn(alpha, s.d[e]));
}

// ---- q_prev <- q_l, q_l <- x (solvers.py:351)
__global__ void __launch_bounds__(kSlabVT) k_slab_finish(SlabView s, int xs) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3 * s.n) return;
  s.q_prev[e] = s.q_l[e];
  s.q_l[e] = s.X[(size_t)xs * s.n * 3 + e];
}

}  // namespace qn

struct qn_slab {
  qn_system* local = nullptr;
  qn::SlabView s{};
  std::vector<void*> allocs;
  int nblk_max = 1;
};

namespace {

template <class T>
int slab_alloc(qn_slab* S, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    qn::set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return QN_ERR_ALLOC;
  }
  S->allocs.push_back((void*)*p);
  e = cudaMemset(*p, 0, count * sizeof(T));
  if (e != cudaSuccess) {
    qn::set_error(std::string("cudaMemset: ") + cudaGetErrorString(e));
    return QN_ERR_CUDA;
  }
  return QN_OK;
}

template <class T>
int slab_upload(qn_slab* S, T** p, const T* h, size_t count) {
  int rc = slab_alloc(S, p, count);
  if (rc) return rc;
  if (count) QN_CUDA(cudaMemcpy(*p, h, count * sizeof(T), cudaMemcpyHostToDevice));
  return QN_OK;
}

void slab_free(qn_slab* S) {
  for (void* p : S->allocs) cudaFree(p);
  delete S;
}

int args_from(const double* v, int32_t nv, qn::SlabArgs* a) {
  std::memset(a, 0, sizeof(*a));
  // layout: [xs, xs_to, have_prev, new_slot, nring, first, alpha, ring[kSlabRing], coef[kSlabRing]]
  QN_REQUIRE(nv >= 7, QN_ERR_ARG, "slab stage: args");
  a->xs = (int32_t)v[0];
  a->xs_to = (int32_t)v[1];
  a->have_prev = (int32_t)v[2];
  a->new_slot = (int32_t)v[3];
  a->nring = (int32_t)v[4];
  a->first = (int32_t)v[5];
  a->alpha = v[6];
  QN_REQUIRE(a->nring >= 0 && a->nring <= qn::kSlabMaxM, QN_ERR_ARG, "slab stage: ring length");
  QN_REQUIRE(nv >= 7 + 2 * qn::kSlabRing || a->nring == 0, QN_ERR_ARG, "slab stage: ring args");
  if (nv >= 7 + 2 * qn::kSlabRing) {
    for (int j = 0; j < qn::kSlabRing; ++j) {
      a->ring[j] = (int32_t)v[7 + j];
      a->coef[j] = v[7 + qn::kSlabRing + j];
    }
  }
  for (int j = 0; j < a->nring; ++j)
    QN_REQUIRE(a->ring[j] >= 0 && a->ring[j] < qn::kSlabRing, QN_ERR_ARG, "slab stage: ring slot");
  QN_REQUIRE(a->new_slot >= 0 && a->new_slot < qn::kSlabRing, QN_ERR_ARG, "slab stage: new slot");
  QN_REQUIRE((a->xs == 0 || a->xs == 1) && (a->xs_to == 0 || a->xs_to == 1), QN_ERR_ARG, "slab stage: x slot");
  return QN_OK;
}

}  // namespace

extern "C" {

int qn_slab_create(const qn_slab_desc* d, qn_slab** out) {
  using namespace qn;
  QN_REQUIRE(d && out && d->local, QN_ERR_ARG, "slab_create: null");
  qn_system* L = d->local;
  QN_REQUIRE(L->n_inst == 1, QN_ERR_UNSUPPORTED, "slab_create: one instance per slab");
  QN_REQUIRE(L->v.pcg == 1 || L->v.pcg == 2, QN_ERR_ARG, "slab_create: the local system must be built in pcg/amg mode");
  QN_REQUIRE(d->n_ranks >= 1 && d->own_lo >= 0 && d->own_lo < d->own_hi && d->own_hi <= L->n, QN_ERR_ARG,
             "slab_create: owned range");
  QN_REQUIRE(d->tet_own_lo >= 0 && d->tet_own_lo <= L->mt, QN_ERR_ARG, "slab_create: tet_own_lo");
  QN_REQUIRE(d->pcg_tol > 0 && d->pcg_maxit > 0, QN_ERR_ARG, "slab_create: pcg_tol / pcg_maxit");
  const int64_t n = L->n, nf = L->n_free;
  QN_REQUIRE(d->a_indptr && d->a_indptr[0] == 0 && d->a_nnz == d->a_indptr[nf], QN_ERR_ARG, "slab_create: A rows");
  for (int64_t p = 0; p < d->a_nnz; ++p)
    QN_REQUIRE(d->a_indices[p] >= 0 && d->a_indices[p] < n, QN_ERR_ARG, "slab_create: A column out of range");
  qn_slab* S = new qn_slab();
  auto fail = [&](int rc) {
    slab_free(S);
    return rc;
  };
  S->local = L;
  SlabView& s = S->s;
  s.v = L->v;
  s.n = (int32_t)n;
  s.mt = (int32_t)L->mt;
  s.tet_own_lo = (int32_t)d->tet_own_lo;
  s.own_lo = (int32_t)d->own_lo;
  s.own_hi = (int32_t)d->own_hi;
  s.nf = (int32_t)nf;
  s.G = d->n_ranks;
  s.amg = L->v.pcg == 2 ? 1 : 0;
  s.pcg_tol = d->pcg_tol;
  s.pcg_maxit = d->pcg_maxit;
  int dev = 0, nsm = kSMs;
  QN_CUDA(cudaGetDevice(&dev));
  QN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  s.nblk_all = std::max(1, div_up(std::max<int64_t>(n, nf), kSlabVT));
  s.nblk_own = std::max(1, div_up(d->own_hi - d->own_lo, kSlabVT));
  s.nblk_t = std::max(1, div_up(L->mt, kTT));
  s.nblk_f = std::max(1, div_up(nf, kSlabVT));
  const int64_t nsl = (nf + 31) / 32;
  s.nblk_spmv = (int32_t)std::max<int64_t>(1, std::min<int64_t>(div_up(nsl, kSpmvWarps), (int64_t)nsm * 3));
  s.nblk_flat = (int32_t)std::max<int64_t>(1, std::min<int64_t>(div_up(3 * nf, 384), (int64_t)nsm * 4));
  S->nblk_max = std::max(std::max(std::max(s.nblk_all, s.nblk_t), s.nblk_spmv), s.nblk_flat);
  s.nblk_max = S->nblk_max;

  // free rows of the local system (= owned free vertices, increasing): read its fact_vtx map
  std::vector<int32_t> f2v((size_t)std::max<int64_t>(nf, 1)), v2f((size_t)n, -1);
  QN_CUDA(cudaMemcpy(f2v.data(), L->v.fact_vtx, nf * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int64_t f = 0; f < nf; ++f) {
    QN_REQUIRE(f2v[f] >= d->own_lo && f2v[f] < d->own_hi, QN_ERR_ARG, "slab_create: local free vertex not owned");
    v2f[f2v[f]] = (int32_t)f;
  }
  std::vector<uint8_t> pin(d->pinned, d->pinned + n);
  std::vector<double> dinv((size_t)std::max<int64_t>(nf, 1), 0.0);
  for (int64_t f = 0; f < nf; ++f)
    for (int64_t p = d->a_indptr[f]; p < d->a_indptr[f + 1]; ++p)
      if (d->a_indices[p] == f2v[f]) dinv[f] = 1.0 / d->a_values[p];
  for (int64_t f = 0; f < nf; ++f)
    if (!(dinv[f] > 0.0)) {
      set_error("slab_create: matrix is not positive definite (non-positive diagonal)");
      return fail(QN_ERR_NOT_SPD);
    }
  std::vector<int64_t> sptr;
  std::vector<int32_t> scol;
  std::vector<double> sval;
  sell_build(nf, n, d->a_indptr, d->a_indices, d->a_values, 1, d->a_nnz, sptr, scol, sval);
  int rc;
  int32_t *df2v, *dv2f, *dcol;
  uint8_t* dpin;
  int64_t* dptr;
  double *dval, *ddinv;
  if ((rc = slab_upload(S, &df2v, f2v.data(), f2v.size())) || (rc = slab_upload(S, &dv2f, v2f.data(), v2f.size())) ||
      (rc = slab_upload(S, &dpin, pin.data(), pin.size())) || (rc = slab_upload(S, &dptr, sptr.data(), sptr.size())) ||
      (rc = slab_upload(S, &dcol, scol.data(), scol.size())) ||
      (rc = slab_upload(S, &dval, sval.data(), sval.size())) ||
      (rc = slab_upload(S, &ddinv, dinv.data(), dinv.size())))
    return fail(rc);
  s.f2v = df2v;
  s.v2f = dv2f;
  s.pinned = dpin;
  s.A = SellDev{dptr, dcol, dval, (int32_t)nsl, (int32_t)nf};
  s.dinv = ddinv;
  const size_t v3 = (size_t)n * 3, f3 = (size_t)std::max<int64_t>(nf, 1) * 3;
  double* gath;
  if ((rc = slab_alloc(S, &s.q_l, v3)) || (rc = slab_alloc(S, &s.q_prev, v3)) || (rc = slab_alloc(S, &s.y, v3)) ||
      (rc = slab_alloc(S, &s.X, 2 * v3)) || (rc = slab_alloc(S, &s.g, v3)) || (rc = slab_alloc(S, &s.xp, v3)) ||
      (rc = slab_alloc(S, &s.gp, v3)) || (rc = slab_alloc(S, &s.d, v3)) || (rc = slab_alloc(S, &s.r0, v3)) ||
      (rc = slab_alloc(S, &s.S, kSlabRing * v3)) || (rc = slab_alloc(S, &s.T, kSlabRing * v3)) ||
      (rc = slab_alloc(S, &s.px, f3)) || (rc = slab_alloc(S, &s.pq, f3)) || (rc = slab_alloc(S, &s.pv, v3)) ||
      (rc = slab_alloc(S, &s.part, (size_t)8 * S->nblk_max * kSlabSend)) || (rc = slab_alloc(S, &s.cnt, 8)) ||
      (rc = slab_alloc(S, &s.send, kSlabSend)) || (rc = slab_alloc(S, &gath, (size_t)s.G * kSlabSend)) ||
      (rc = slab_alloc(S, &s.pc, 1)))
    return fail(rc);
  s.gath = gath;
  if (s.amg) {  // the local V-cycle reads the residual from v.pr and writes z to v.pz
    s.pr = L->v.pr;
    s.pz = L->v.pz;
    L->v.pzf = nullptr;  // the slab CG adds its coarse share to the fp64 z: the V-cycle writes v.pz
    // its kernels run while the local system's instance is "in a direction
    // phase with an unconverged CG" (the local frame itself is never run)
    int32_t ph = PH_DIR;
    QN_CUDA(cudaMemcpy(&L->v.ctl[0].phase, &ph, sizeof(ph), cudaMemcpyHostToDevice));
    int32_t conv = 0;
    QN_CUDA(cudaMemcpy(&L->v.pctl[0].conv, &conv, sizeof(conv), cudaMemcpyHostToDevice));
  } else if ((rc = slab_alloc(S, &s.pr, f3)) || (rc = slab_alloc(S, &s.pz, f3))) {
    return fail(rc);
  }
  *out = S;
  return QN_OK;
}

int qn_slab_destroy(qn_slab* S) {
  if (S) slab_free(S);
  return QN_OK;
}

int qn_slab_buffer(qn_slab* S, int32_t which, void** ptr, int64_t* count) {
  QN_REQUIRE(S && ptr && count, QN_ERR_ARG, "slab_buffer: null");
  const qn::SlabView& s = S->s;
  const int64_t v3 = (int64_t)s.n * 3;
  switch (which) {
    case QN_SLAB_SEND: *ptr = s.send; *count = qn::kSlabSend; break;
    case QN_SLAB_GATHER: *ptr = (void*)s.gath; *count = (int64_t)s.G * qn::kSlabSend; break;
    case QN_SLAB_P: *ptr = s.pv; *count = v3; break;
    case QN_SLAB_R0: *ptr = s.r0; *count = v3; break;
    case QN_SLAB_QL: *ptr = s.q_l; *count = v3; break;
    case QN_SLAB_QPREV: *ptr = s.q_prev; *count = v3; break;
    case QN_SLAB_Y: *ptr = s.y; *count = v3; break;
    case QN_SLAB_X: *ptr = s.X; *count = 2 * v3; break;
    case QN_SLAB_G: *ptr = s.g; *count = v3; break;
    case QN_SLAB_CSEND: *ptr = s.csend; *count = 3 * (int64_t)s.nc; break;
    case QN_SLAB_CGATHER: *ptr = (void*)s.cgath; *count = 3 * (int64_t)s.nc * s.G; break;
    default: qn::set_error("slab_buffer: unknown buffer"); return QN_ERR_ARG;
  }
  return QN_OK;
}

int qn_slab_stage(qn_slab* S, int32_t stage, const double* args, int32_t nargs, void* stream) {
  using namespace qn;
  QN_REQUIRE(S, QN_ERR_ARG, "slab_stage: null");
  const SlabView& s = S->s;
  cudaStream_t st = (cudaStream_t)stream;
  SlabArgs a;
  int rc = args_from(args, nargs, &a);
  if (rc) return rc;
  const int gv = std::max(1, div_up(3 * (int64_t)s.n, kSlabVT));
  switch (stage) {
    case QN_SLAB_INIT:
      k_slab_init<<<s.nblk_all, kSlabVT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_EVAL:
      if (s.v.n_mat <= kMatSmem) {
        k_slab_tet<true><<<s.nblk_t, kTT, 0, st>>>(s, a.xs);
      } else {
        k_slab_tet<false><<<s.nblk_t, kTT, 0, st>>>(s, a.xs);
      }
      QN_CHECK_LAUNCH();
      k_slab_inertia<<<s.nblk_own, kSlabVT, 0, st>>>(s, a.xs);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_GRAD:
      k_slab_grad<<<s.nblk_all, kSlabVT, 0, st>>>(s, a);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_PCG_SETUP:
      QN_CUDA(cudaMemsetAsync(s.pc, 0, sizeof(SlabPcg), st));
      k_slab_pcg_setup<<<s.nblk_all, kSlabVT, 0, st>>>(s, a);
      QN_CHECK_LAUNCH();
      if (s.amg && (rc = launch_vcycle(S->local, st))) return rc;
      break;
    case QN_SLAB_PCG_P:
      k_slab_pcg_p<<<s.nblk_flat, kSlabFT, 0, st>>>(s, a.first);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_PCG_SPMV:
      k_slab_spmv<<<s.nblk_spmv, kSpmvThreads, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_PCG_UPDATE:
      k_slab_pcg_update<<<s.nblk_flat, kSlabFT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      k_slab_pcg_count<<<1, 1, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      if (s.amg && (rc = launch_vcycle(S->local, st))) return rc;
      break;
    case QN_SLAB_PCG_RZ:
      k_slab_rz<<<s.nblk_flat, kSlabFT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_COARSE_R:
      QN_REQUIRE(s.nc > 0, QN_ERR_ARG, "slab_stage: no coarse level set");
      k_slab_coarse_z<<<std::max(1, div_up((int64_t)s.npl * (s.gy + 1) * s.cz * 3, kSlabVT)), kSlabVT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      k_slab_coarse_y<<<std::max(1, div_up((int64_t)s.npl * s.cy * s.cz * 3, kSlabVT)), kSlabVT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      k_slab_coarse_x<<<std::max(1, div_up(3 * (int64_t)s.nc, kSlabVT)), kSlabVT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_COARSE_APPLY:
      QN_REQUIRE(s.nc > 0, QN_ERR_ARG, "slab_stage: no coarse level set");
      k_slab_coarse_solve<<<std::max(1, std::min(2 * kSMs, div_up(s.nc, kSpmvWarps))), kSpmvThreads,
                            (size_t)3 * s.nc * sizeof(double), st>>>(s);
      QN_CHECK_LAUNCH();
      k_slab_coarse_p<<<s.nblk_flat, kSlabFT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      k_slab_coarse_dot<<<1, kSpmvThreads, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_STORE:
      k_slab_store<<<s.nblk_all, kSlabVT, 0, st>>>(s);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_ETA:
      k_slab_eta<<<s.nblk_own, kSlabVT, 0, st>>>(s, a);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_DIR:
      k_slab_dir<<<s.nblk_all, kSlabVT, 0, st>>>(s, a);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_TRIAL:
      k_slab_trial<<<gv, kSlabVT, 0, st>>>(s, a.xs, a.xs_to, a.alpha);
      QN_CHECK_LAUNCH();
      break;
    case QN_SLAB_FINISH:
      k_slab_finish<<<gv, kSlabVT, 0, st>>>(s, a.xs);
      QN_CHECK_LAUNCH();
      break;
    default:
      set_error("slab_stage: unknown stage");
      return QN_ERR_ARG;
  }
  return QN_OK;
}

int qn_slab_set_coarse(qn_slab* S, const int32_t* grid, const int32_t* coarse_dims, int64_t v0, int64_t i_lo,
                       int64_t n_planes, const int32_t* hat_first, const double* hat_w, const int32_t* node_pos,
                       const double* cinv) {
  using namespace qn;
  QN_REQUIRE(S && grid && coarse_dims && hat_first && hat_w && node_pos && cinv, QN_ERR_ARG, "slab_set_coarse: null");
  SlabView& s = S->s;
  QN_REQUIRE(s.nc == 0, QN_ERR_ARG, "slab_set_coarse: already set");
  const int64_t nc = (int64_t)coarse_dims[0] * coarse_dims[1] * coarse_dims[2];
  QN_REQUIRE(nc > 0 && 3 * nc * (int64_t)sizeof(double) <= 200 * 1024, QN_ERR_ARG, "slab_set_coarse: coarse size");
  const int64_t plane = (int64_t)(grid[1] + 1) * (grid[2] + 1);
  QN_REQUIRE(n_planes >= 1 && i_lo >= 0 && i_lo + n_planes <= grid[0] + 1 && i_lo * plane >= v0 &&
                 (i_lo + n_planes) * plane - v0 <= s.n,
             QN_ERR_ARG, "slab_set_coarse: owned planes outside the slab");
  int rc;
  int64_t off_h = 0, off_p = 0;
  for (int d = 0; d < 3; ++d) {
    const int nf = grid[d] + 1;
    int32_t* dI;
    double* dw;
    int32_t* dp;
    for (int i = 0; i < nf; ++i)
      QN_REQUIRE(hat_first[off_h + i] >= 0 && hat_first[off_h + i] + 1 < coarse_dims[d], QN_ERR_ARG,
                 "slab_set_coarse: hat table");
    if ((rc = slab_upload(S, &dI, hat_first + off_h, (size_t)nf)) ||
        (rc = slab_upload(S, &dw, hat_w + 2 * off_h, (size_t)2 * nf)) ||
        (rc = slab_upload(S, &dp, node_pos + off_p, (size_t)coarse_dims[d])))
      return rc;
    s.hI[d] = dI;
    s.hw[d] = dw;
    s.hpos[d] = dp;
    off_h += nf;
    off_p += coarse_dims[d];
  }
  double *dci, *dgath;
  if ((rc = slab_upload(S, &dci, cinv, (size_t)(nc * nc))) || (rc = slab_alloc(S, &s.csend, (size_t)nc * 3)) ||
      (rc = slab_alloc(S, &dgath, (size_t)nc * 3 * s.G)) || (rc = slab_alloc(S, &s.ec, (size_t)nc * 3)) ||
      (rc = slab_alloc(S, &s.t0, (size_t)n_planes * (grid[1] + 1) * coarse_dims[2] * 3)) ||
      (rc = slab_alloc(S, &s.t1, (size_t)n_planes * coarse_dims[1] * coarse_dims[2] * 3)))
    return rc;
  QN_CUDA(cudaFuncSetAttribute(k_slab_coarse_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(3 * nc * sizeof(double))));
  s.cinv = dci;
  s.cgath = dgath;
  s.gx = grid[0];
  s.gy = grid[1];
  s.gz = grid[2];
  s.cx = coarse_dims[0];
  s.cy = coarse_dims[1];
  s.cz = coarse_dims[2];
  s.npl = (int32_t)n_planes;
  s.i_lo = (int32_t)i_lo;
  s.v0 = (int32_t)v0;
  s.nc = (int32_t)nc;
  return QN_OK;
}

int qn_slab_pcg_status(qn_slab* S, int32_t* conv, int32_t* iters, void* stream) {
  QN_REQUIRE(S && conv && iters, QN_ERR_ARG, "slab_pcg_status: null");
  qn::SlabPcg pc;
  cudaStream_t st = (cudaStream_t)stream;
  QN_CUDA(cudaMemcpyAsync(&pc, S->s.pc, sizeof(pc), cudaMemcpyDeviceToHost, st));
  QN_CUDA(cudaStreamSynchronize(st));
  *conv = pc.conv;
  *iters = pc.total;
  return QN_OK;
}

}  // extern "C"

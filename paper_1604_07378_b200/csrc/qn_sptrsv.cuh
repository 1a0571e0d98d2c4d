// Device supernodal triangular solves with 3 right-hand sides (x, y, z of the
// (n_free, 3) RHS — A is the same scalar matrix for all three coordinates,
// dynamics.py:413 / solvers.py:134), replacing scipy cho_solve (linalg.py:40).
//
// Scheduling: one CTA per (supernode, batch instance) work item.  CTAs take
// tickets from a global counter in topological order (postorder for L y = b,
// reverse for L^T x = y) and wait on the int flags of their dependencies
// (children / parent), so there are no level barriers and no inter-kernel
// launches per tree level.  A ticket is only taken by a running CTA, and a
// dependency always has a smaller ticket, so the wait cannot deadlock.
// All arithmetic is in fixed order (no float atomics): results are
// bitwise reproducible run to run.
#pragma once

#include "qn_common.cuh"
#include "qn_factor.h"

namespace qn {

struct FactorView {
  int32_t n, nsup, nbatch;
  int64_t nvals, nupd;
  const int32_t* sup_col;
  const int64_t* sup_row_ptr;
  const int32_t* sup_rows;
  const int64_t* sup_val_ptr;
  const int64_t* sup_upd_ptr;
  const int32_t* parent;
  const int32_t* child_ptr;
  const int32_t* child_idx;
  const int64_t* rel_ptr;
  const int32_t* rel;
  const double* vals;
  double* y;
  double* x;
  double* u;
  unsigned* flags;  // [2][nbatch][nsup]
  unsigned* sched;  // ticket_f, done_f, epoch_f, ticket_b, done_b, epoch_b
};

inline FactorView factor_view(const qn_factor* f) {
  FactorView v;
  v.n = (int32_t)f->n;
  v.nsup = f->nsup;
  v.nbatch = (int32_t)f->nbatch;
  v.nvals = f->nvals;
  v.nupd = f->nupd;
  v.sup_col = f->d_sup_col;
  v.sup_row_ptr = f->d_sup_row_ptr;
  v.sup_rows = f->d_sup_rows;
  v.sup_val_ptr = f->d_sup_val_ptr;
  v.sup_upd_ptr = f->d_sup_upd_ptr;
  v.parent = f->d_parent;
  v.child_ptr = f->d_child_ptr;
  v.child_idx = f->d_child_idx;
  v.rel_ptr = f->d_rel_ptr;
  v.rel = f->d_rel;
  v.vals = f->d_vals;
  v.y = f->d_y;
  v.x = f->d_x;
  v.u = f->d_u;
  v.flags = f->d_flags;
  v.sched = f->d_sched;
  return v;
}

constexpr int kSolveThreads = 256;

__device__ __forceinline__ void wait_flag(const unsigned* p, unsigned epoch) {
  while (ld_acquire(p) != epoch) __nanosleep(32);
}

// Take a ticket; returns (item, epoch) through shared memory.
__device__ __forceinline__ void take_ticket(unsigned* sched, int* s_item, unsigned* s_epoch) {
  if (threadIdx.x == 0) {
    *s_item = (int)atomicAdd(&sched[0], 1u);
    *s_epoch = *((volatile unsigned*)&sched[2]);
  }
  __syncthreads();
}

__device__ __forceinline__ void finish_item(unsigned* sched, unsigned total, unsigned epoch) {
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&sched[1], 1u);
    if (d == total - 1) {  // last CTA of this launch: reset for the next one
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
      atomicExch(&sched[2], epoch + 1);
    }
  }
}

// IO: struct with
//   __device__ bool active(int b) const;
//   __device__ void rhs(int b, int row, double (&v)[3]) const;   // factor row
//   __device__ void store(int b, int row, const double (&v)[3]) const;
template <class IO>
__global__ void __launch_bounds__(kSolveThreads) sptrsv_forward(FactorView F, IO io) {
  extern __shared__ double sm[];  // acc[max_rows*3] | y[max_nc*3] (aliases tail)
  __shared__ int s_item;
  __shared__ unsigned s_epoch;
  unsigned* sched = F.sched;
  take_ticket(sched, &s_item, &s_epoch);
  const int item = s_item;
  const unsigned epoch = s_epoch;
  const int s = item / F.nbatch, b = item % F.nbatch;
  const unsigned total = (unsigned)F.nsup * (unsigned)F.nbatch;
  if (io.active(b)) {
    const int c0 = F.sup_col[s], nc = F.sup_col[s + 1] - c0;
    const int64_t r0 = F.sup_row_ptr[s];
    const int nr = (int)(F.sup_row_ptr[s + 1] - r0), mb = nr - nc;
    double* acc = sm;            // nr x 3
    double* ys = sm + 3 * nr;    // nc x 3
    const int ch0 = F.child_ptr[s], ch1 = F.child_ptr[s + 1];
    if (threadIdx.x == 0)
      for (int q = ch0; q < ch1; ++q) wait_flag(&F.flags[(size_t)b * F.nsup + F.child_idx[q]], epoch);
    for (int i = threadIdx.x; i < 3 * nr; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    // extend-add children's update vectors in child order (deterministic)
    for (int q = ch0; q < ch1; ++q) {
      const int c = F.child_idx[q];
      const int64_t rp = F.rel_ptr[c];
      const int mc = (int)(F.rel_ptr[c + 1] - rp);
      const double* uc = F.u + ((size_t)b * F.nupd + F.sup_upd_ptr[c]) * 3;
      for (int i = threadIdx.x; i < mc; i += blockDim.x) {
        const int p = F.rel[rp + i];
        acc[3 * p + 0] += __ldcg(uc + 3 * i + 0);
        acc[3 * p + 1] += __ldcg(uc + 3 * i + 1);
        acc[3 * p + 2] += __ldcg(uc + 3 * i + 2);
      }
      __syncthreads();
    }
    // top rows: f = b - sum(children contributions)
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      double v[3];
      io.rhs(b, c0 + i, v);
      acc[3 * i + 0] = v[0] - acc[3 * i + 0];
      acc[3 * i + 1] = v[1] - acc[3 * i + 1];
      acc[3 * i + 2] = v[2] - acc[3 * i + 2];
    }
    __syncthreads();
    const double* Xv = F.vals + (size_t)b * F.nvals + F.sup_val_ptr[s];
    // y = inv(L11) f_top  (lower triangular, column-major: coalesced over rows)
    double* yg = F.y + ((size_t)b * F.n + c0) * 3;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int k = 0; k <= i; ++k) {
        const double l = __ldg(Xv + i + (size_t)k * nc);
        a0 = fma(l, acc[3 * k + 0], a0);
        a1 = fma(l, acc[3 * k + 1], a1);
        a2 = fma(l, acc[3 * k + 2], a2);
      }
      ys[3 * i + 0] = a0;
      ys[3 * i + 1] = a1;
      ys[3 * i + 2] = a2;
      yg[3 * i + 0] = a0;
      yg[3 * i + 1] = a1;
      yg[3 * i + 2] = a2;
    }
    __syncthreads();
    // u_s = (children contributions to rows below) + L21 y
    if (mb > 0 && F.parent[s] >= 0) {
      const double* Lb = Xv + (size_t)nc * nc;
      double* us = F.u + ((size_t)b * F.nupd + F.sup_upd_ptr[s]) * 3;
      for (int r = threadIdx.x; r < mb; r += blockDim.x) {
        double a0 = acc[3 * (nc + r) + 0], a1 = acc[3 * (nc + r) + 1], a2 = acc[3 * (nc + r) + 2];
        for (int k = 0; k < nc; ++k) {
          const double l = __ldg(Lb + r + (size_t)k * mb);
          a0 = fma(l, ys[3 * k + 0], a0);
          a1 = fma(l, ys[3 * k + 1], a1);
          a2 = fma(l, ys[3 * k + 2], a2);
        }
        __stcg(us + 3 * r + 0, a0);
        __stcg(us + 3 * r + 1, a1);
        __stcg(us + 3 * r + 2, a2);
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(&F.flags[(size_t)b * F.nsup + s], epoch);
  }
  finish_item(sched, total, epoch);
}

template <class IO>
__global__ void __launch_bounds__(kSolveThreads) sptrsv_backward(FactorView F, IO io) {
  extern __shared__ double sm[];  // xb[max_rows*3] | t[max_nc*3]
  __shared__ int s_item;
  __shared__ unsigned s_epoch;
  unsigned* sched = F.sched + 3;
  take_ticket(sched, &s_item, &s_epoch);
  const int item = s_item;
  const unsigned epoch = s_epoch;
  const int s = F.nsup - 1 - item / F.nbatch, b = item % F.nbatch;
  const unsigned total = (unsigned)F.nsup * (unsigned)F.nbatch;
  unsigned* flags = F.flags + (size_t)F.nbatch * F.nsup;
  if (io.active(b)) {
    const int c0 = F.sup_col[s], nc = F.sup_col[s + 1] - c0;
    const int64_t r0 = F.sup_row_ptr[s];
    const int nr = (int)(F.sup_row_ptr[s + 1] - r0), mb = nr - nc;
    double* xb = sm;            // mb x 3
    double* t = sm + 3 * nr;    // nc x 3
    const int p = F.parent[s];
    if (threadIdx.x == 0 && p >= 0) wait_flag(&flags[(size_t)b * F.nsup + p], epoch);
    __syncthreads();
    const double* xg = F.x + (size_t)b * F.n * 3;
    for (int r = threadIdx.x; r < mb; r += blockDim.x) {
      const int row = F.sup_rows[r0 + nc + r];
      xb[3 * r + 0] = __ldcg(xg + 3 * row + 0);
      xb[3 * r + 1] = __ldcg(xg + 3 * row + 1);
      xb[3 * r + 2] = __ldcg(xg + 3 * row + 2);
    }
    __syncthreads();
    const double* Xv = F.vals + (size_t)b * F.nvals + F.sup_val_ptr[s];
    const double* Lb = Xv + (size_t)nc * nc;
    const double* yg = F.y + ((size_t)b * F.n + c0) * 3;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // t_k = y_k - L21[:,k] . xb   (warp per column; column is contiguous)
    for (int k = warp; k < nc; k += nw) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      const double* col = Lb + (size_t)k * mb;
      for (int r = lane; r < mb; r += 32) {
        const double l = __ldg(col + r);
        a0 = fma(l, xb[3 * r + 0], a0);
        a1 = fma(l, xb[3 * r + 1], a1);
        a2 = fma(l, xb[3 * r + 2], a2);
      }
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      if (lane == 0) {
        t[3 * k + 0] = __ldcg(yg + 3 * k + 0) - a0;
        t[3 * k + 1] = __ldcg(yg + 3 * k + 1) - a1;
        t[3 * k + 2] = __ldcg(yg + 3 * k + 2) - a2;
      }
    }
    __syncthreads();
    // x_k = sum_{i >= k} inv(L11)[i,k] t_i   (warp per column)
    double* xo = F.x + ((size_t)b * F.n + c0) * 3;
    for (int k = warp; k < nc; k += nw) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      const double* col = Xv + (size_t)k * nc;
      for (int i = k + lane; i < nc; i += 32) {
        const double l = __ldg(col + i);
        a0 = fma(l, t[3 * i + 0], a0);
        a1 = fma(l, t[3 * i + 1], a1);
        a2 = fma(l, t[3 * i + 2], a2);
      }
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      if (lane == 0) {
        xo[3 * k + 0] = a0;
        xo[3 * k + 1] = a1;
        xo[3 * k + 2] = a2;
        const double v[3] = {a0, a1, a2};
        io.store(b, c0 + k, v);
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(&flags[(size_t)b * F.nsup + s], epoch);
  }
  finish_item(sched, total, epoch);
}

// Plain solve: B (n,3) -> X (n,3) in the original row order, one instance.
struct PlainIO {
  const double* B;
  double* X;
  const int32_t* perm;  // factor row -> original row
  int batch;
  __device__ bool active(int b) const { return b == batch; }
  __device__ void rhs(int, int row, double (&v)[3]) const {
    const int o = perm[row];
    v[0] = B[3 * o + 0];
    v[1] = B[3 * o + 1];
    v[2] = B[3 * o + 2];
  }
  __device__ void store(int, int row, const double (&v)[3]) const {
    const int o = perm[row];
    X[3 * o + 0] = v[0];
    X[3 * o + 1] = v[1];
    X[3 * o + 2] = v[2];
  }
};

template <class IO>
int launch_solve(qn_factor* f, const IO& io, cudaStream_t stream) {
  const FactorView v = factor_view(f);
  const int grid = f->nsup * (int)f->nbatch;
  sptrsv_forward<IO><<<grid, kSolveThreads, f->smem_bytes, stream>>>(v, io);
  QN_CHECK_LAUNCH();
  sptrsv_backward<IO><<<grid, kSolveThreads, f->smem_bytes, stream>>>(v, io);
  QN_CHECK_LAUNCH();
  return QN_OK;
}

template <class IO>
int prepare_solve_kernels(int smem_bytes) {
  QN_CUDA(cudaFuncSetAttribute(sptrsv_forward<IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  QN_CUDA(cudaFuncSetAttribute(sptrsv_backward<IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  return QN_OK;
}

}  // namespace qn

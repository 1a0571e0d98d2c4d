// Device supernodal triangular solves with 3 right-hand sides (x, y, z of the
// (n_free, 3) RHS — A is the same scalar matrix for all three coordinates,
// dynamics.py:413 / solvers.py:134), replacing scipy cho_solve (linalg.py:40).
//
// Per supernode s (columns J_s, front rows R_s, nc = |J_s|, nr = |R_s|) the host
// stores Z_s = [inv(L_ss); L_Bs inv(L_ss)] (nr x nc, column-major), so
//   forward  (L y = b):   f = b_J - sum(children updates);  v = Z_s f;
//                         y_J = v[0:nc],  u_s = (children updates below) + v[nc:nr]
//   backward (L^T x = y): x_J = Z_s^T [y_J; -x_below]
// Both are dense mat-vecs whose rows (forward) / columns (backward) are
// independent, so a supernode is split into many small tasks (32-row blocks /
// 8-column blocks) that run on different SMs — the top separators no longer
// serialise on one SM.
//
// Scheduling: one CTA per (task, batch instance).  CTAs take tickets from a
// global counter in topological order (postorder forward, reverse backward)
// and spin on integer flags of the supernodes they depend on (all children /
// the parent).  A ticket is only taken by a running CTA and dependencies have
// smaller tickets, so the wait cannot deadlock.  All arithmetic is in fixed
// order (no float atomics): results are bitwise reproducible run to run.
#pragma once

#include "qn_common.cuh"
#include "qn_factor.h"

namespace qn {

struct FactorView {
  int32_t n, nsup, nbatch, nftask, nbtask;
  int64_t nvals, nupd;
  const int32_t* sup_col;
  const int64_t* sup_row_ptr;
  const int32_t* sup_rows;
  const int64_t* sup_val_ptr;
  const int64_t* sup_upd_ptr;
  const int32_t* parent;
  const int32_t* child_ptr;
  const int32_t* child_idx;
  const int64_t* cptr;
  const int32_t* cidx;
  const int4* ftask;
  const int4* btask;
  const int32_t* fcount;
  const int32_t* bcount;
  const double* vals;
  double* y;
  double* x;
  double* u;
  unsigned long long* done;  // [2][nbatch][nsup]
  unsigned* flags;           // [2][nbatch][nsup]
  unsigned* sched;           // ticket_f, done_f, epoch_f, ticket_b, done_b, epoch_b
};

inline FactorView factor_view(const qn_factor* f) {
  FactorView v;
  v.n = (int32_t)f->n;
  v.nsup = f->nsup;
  v.nbatch = (int32_t)f->nbatch;
  v.nftask = (int32_t)f->ftask.size();
  v.nbtask = (int32_t)f->btask.size();
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
  v.cptr = f->d_cptr;
  v.cidx = f->d_cidx;
  v.ftask = f->d_ftask;
  v.btask = f->d_btask;
  v.fcount = f->d_fcount;
  v.bcount = f->d_bcount;
  v.vals = f->d_vals;
  v.y = f->d_y;
  v.x = f->d_x;
  v.u = f->d_u;
  v.done = f->d_done;
  v.flags = f->d_flags;
  v.sched = f->d_sched;
  return v;
}

constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;

// Spin on a dependency flag.  A wait longer than 2 s means a scheduling bug:
// record it in sched[6] (checked by the host after the frame) and give up
// instead of hanging the device.
__device__ __forceinline__ void wait_flag(const unsigned* p, unsigned epoch, unsigned* sched) {
  if (ld_acquire(p) == epoch) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire(p) != epoch) {
    __nanosleep(20);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) {
      atomicOr(&sched[6], 1u);
      return;
    }
  }
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

// task completion: the last task of supernode s resets the per-launch counter
// (no other task of s touches it again in this launch) and publishes the flag.
// Instances skipped by a launch never touch their counters, so they stay 0.
__device__ __forceinline__ void complete_task(unsigned long long* done, unsigned* flag, int ntasks, unsigned epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long old = atomicAdd(done, 1ull);
    if (old + 1 == (unsigned long long)ntasks) {
      *done = 0ull;
      st_release(flag, epoch);
    }
  }
}

// IO: struct with
//   __device__ bool active(int b) const;
//   __device__ void rhs(int b, int row, double (&v)[3]) const;   // factor row
//   __device__ void store(int b, int row, const double (&v)[3]) const;
template <class IO>
__global__ void __launch_bounds__(kSolveThreads) sptrsv_forward(FactorView F, IO io) {
  extern __shared__ double sm[];  // f[nc*3] | part[8][32][3]
  __shared__ int s_item;
  __shared__ unsigned s_epoch;
  unsigned* sched = F.sched;
  take_ticket(sched, &s_item, &s_epoch);
  const int item = s_item;
  const unsigned epoch = s_epoch;
  const int4 task = F.ftask[item / F.nbatch];
  const int b = item % F.nbatch;
  const int s = task.x, lo = task.y, hi = task.z;
  const unsigned total = (unsigned)F.nftask * (unsigned)F.nbatch;
  if (io.active(b)) {
    const int c0 = F.sup_col[s], nc = F.sup_col[s + 1] - c0;
    const int64_t R0 = F.sup_row_ptr[s];
    const int nr = (int)(F.sup_row_ptr[s + 1] - R0);
    double* f = sm;
    double* part = sm + 3 * nc;
    const double* ub = F.u + (size_t)b * F.nupd * 3;
    if (threadIdx.x == 0)
      for (int q = F.child_ptr[s]; q < F.child_ptr[s + 1]; ++q)
        wait_flag(&F.flags[(size_t)b * F.nsup + F.child_idx[q]], epoch, F.sched);
    __syncthreads();
    // f = b_J - sum of children's updates landing on J (children in order)
    for (int p = threadIdx.x; p < nc; p += blockDim.x) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int64_t q = F.cptr[R0 + p]; q < F.cptr[R0 + p + 1]; ++q) {
        const double* uc = ub + 3 * (size_t)F.cidx[q];
        a0 += __ldcg(uc);
        a1 += __ldcg(uc + 1);
        a2 += __ldcg(uc + 2);
      }
      double v[3];
      io.rhs(b, c0 + p, v);
      f[3 * p + 0] = v[0] - a0;
      f[3 * p + 1] = v[1] - a1;
      f[3 * p + 2] = v[2] - a2;
    }
    __syncthreads();
    // rows [lo, hi) of v = Z f: lane = row, warp = slice of k (coalesced over rows)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kmax = hi <= nc ? hi : nc;  // rows inside the triangle need k <= row only
    const int per = (kmax + kSolveWarps - 1) / kSolveWarps;
    const int kb = warp * per, ke = min(kmax, kb + per);
    const int r = lo + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (r < hi) {
      const double* Z = F.vals + (size_t)b * F.nvals + F.sup_val_ptr[s] + r;
      int k = kb;
      for (; k + 16 <= ke; k += 16) {
        double l[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) l[q] = __ldg(Z + (int64_t)(k + q) * nr);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          a0 = fma(l[q], f[3 * (k + q) + 0], a0);
          a1 = fma(l[q], f[3 * (k + q) + 1], a1);
          a2 = fma(l[q], f[3 * (k + q) + 2], a2);
        }
      }
      for (; k < ke; ++k) {
        const double l = __ldg(Z + (int64_t)k * nr);
        a0 = fma(l, f[3 * k + 0], a0);
        a1 = fma(l, f[3 * k + 1], a1);
        a2 = fma(l, f[3 * k + 2], a2);
      }
    }
    part[(warp * 32 + lane) * 3 + 0] = a0;
    part[(warp * 32 + lane) * 3 + 1] = a1;
    part[(warp * 32 + lane) * 3 + 2] = a2;
    __syncthreads();
    if (threadIdx.x < 32 && r < hi) {
      double v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
      for (int w = 0; w < kSolveWarps; ++w) {
        v0 += part[(w * 32 + lane) * 3 + 0];
        v1 += part[(w * 32 + lane) * 3 + 1];
        v2 += part[(w * 32 + lane) * 3 + 2];
      }
      if (r < nc) {
        double* yg = F.y + ((size_t)b * F.n + c0 + r) * 3;
        yg[0] = v0;
        yg[1] = v1;
        yg[2] = v2;
      } else {
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
        for (int64_t q = F.cptr[R0 + r]; q < F.cptr[R0 + r + 1]; ++q) {
          const double* uc = ub + 3 * (size_t)F.cidx[q];
          e0 += __ldcg(uc);
          e1 += __ldcg(uc + 1);
          e2 += __ldcg(uc + 2);
        }
        double* us = F.u + ((size_t)b * F.nupd + F.sup_upd_ptr[s] + (r - nc)) * 3;
        __stcg(us + 0, e0 + v0);
        __stcg(us + 1, e1 + v1);
        __stcg(us + 2, e2 + v2);
      }
    }
    complete_task(&F.done[(size_t)b * F.nsup + s], &F.flags[(size_t)b * F.nsup + s], F.fcount[s], epoch);
  }
  finish_item(sched, total, epoch);
}

template <class IO>
__global__ void __launch_bounds__(kSolveThreads) sptrsv_backward(FactorView F, IO io) {
  extern __shared__ double sm[];  // w[nr*3] = [y_J; -x_below]
  __shared__ int s_item;
  __shared__ unsigned s_epoch;
  unsigned* sched = F.sched + 3;
  take_ticket(sched, &s_item, &s_epoch);
  const int item = s_item;
  const unsigned epoch = s_epoch;
  const int4 task = F.btask[item / F.nbatch];
  const int b = item % F.nbatch;
  const int s = task.x, k0 = task.y, k1 = task.z;
  const unsigned total = (unsigned)F.nbtask * (unsigned)F.nbatch;
  const size_t off2 = (size_t)F.nbatch * F.nsup;
  if (io.active(b)) {
    const int c0 = F.sup_col[s], nc = F.sup_col[s + 1] - c0;
    const int64_t R0 = F.sup_row_ptr[s];
    const int nr = (int)(F.sup_row_ptr[s + 1] - R0);
    double* w = sm;
    const int p = F.parent[s];
    if (threadIdx.x == 0 && p >= 0) wait_flag(&F.flags[off2 + (size_t)b * F.nsup + p], epoch, F.sched);
    __syncthreads();
    const double* xg = F.x + (size_t)b * F.n * 3;
    const double* yg = F.y + ((size_t)b * F.n + c0) * 3;
    for (int q = threadIdx.x; q < nr; q += blockDim.x) {
      if (q < nc) {
        w[3 * q + 0] = __ldcg(yg + 3 * q + 0);
        w[3 * q + 1] = __ldcg(yg + 3 * q + 1);
        w[3 * q + 2] = __ldcg(yg + 3 * q + 2);
      } else {
        const int row = F.sup_rows[R0 + q];
        w[3 * q + 0] = -__ldcg(xg + 3 * row + 0);
        w[3 * q + 1] = -__ldcg(xg + 3 * row + 1);
        w[3 * q + 2] = -__ldcg(xg + 3 * row + 2);
      }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = k0 + warp;
    if (k < k1) {
      const double* col = F.vals + (size_t)b * F.nvals + F.sup_val_ptr[s] + (int64_t)k * nr;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      int r = k + lane;
      for (; r + 224 < nr; r += 256) {
        double l[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) l[q] = __ldg(col + r + 32 * q);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = r + 32 * q;
          a0 = fma(l[q], w[3 * rr + 0], a0);
          a1 = fma(l[q], w[3 * rr + 1], a1);
          a2 = fma(l[q], w[3 * rr + 2], a2);
        }
      }
      for (; r < nr; r += 32) {
        const double l = __ldg(col + r);
        a0 = fma(l, w[3 * r + 0], a0);
        a1 = fma(l, w[3 * r + 1], a1);
        a2 = fma(l, w[3 * r + 2], a2);
      }
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      if (lane == 0) {
        double* xo = F.x + ((size_t)b * F.n + c0 + k) * 3;
        xo[0] = a0;
        xo[1] = a1;
        xo[2] = a2;
        const double v[3] = {a0, a1, a2};
        io.store(b, c0 + k, v);
      }
    }
    complete_task(&F.done[off2 + (size_t)b * F.nsup + s], &F.flags[off2 + (size_t)b * F.nsup + s], F.bcount[s],
                  epoch);
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
  sptrsv_forward<IO><<<(int)f->ftask.size() * (int)f->nbatch, kSolveThreads, f->smem_bytes, stream>>>(v, io);
  QN_CHECK_LAUNCH();
  sptrsv_backward<IO><<<(int)f->btask.size() * (int)f->nbatch, kSolveThreads, f->smem_bytes, stream>>>(v, io);
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

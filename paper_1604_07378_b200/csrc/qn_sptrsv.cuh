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
// independent, so a supernode is split into tasks (row blocks / column blocks
// of <= kTaskEntries entries of Z) that run on different SMs.
//
// Scheduling: persistent CTAs loop over tickets taken from a global counter in
// level order (forward: height above the leaves; backward: depth below the
// root).  Each task publishes its own epoch flag; a dependent task polls the
// flags of all tasks of its children (forward) / parent (backward) with one
// lane per flag.  Before polling, a CTA stages everything that does not
// depend on them — its Z tile (cp.async into shared memory), the RHS or y,
// and the index lists — so the critical path per tree level is only
// flag -> one round of dependent gathers -> shared-memory FMAs -> flag.
// A ticket is only taken by a running CTA and dependencies have smaller
// tickets, so the waits cannot deadlock.  All arithmetic is in fixed order
// (no float atomics): results are bitwise reproducible run to run.
#pragma once

#include <type_traits>

#include "qn_common.cuh"
#include "qn_factor.h"

namespace qn {

struct FactorView {
  int32_t n, nsup, nbatch, nftask, nbtask, bwd_entries, fwd_entries, batch_max_nc, batch_zmax, nhlev, ndlev;
  int64_t nvals, nupd;
  const int32_t* sup_col;
  const int64_t* sup_row_ptr;
  const int32_t* sup_rows;
  const int64_t* sup_val_ptr;
  const int64_t* sup_upd_ptr;
  const int32_t* parent;
  const int64_t* cptr;
  const int32_t* cidx;
  const int4* ftask;
  const int4* btask;
  const int32_t* bfirst;    // first backward task of each supernode
  const int32_t* bcount;
  const int32_t* fdep_ptr;  // forward: task ids of all children's tasks
  const int32_t* fdep_idx;
  const qn_fdesc* fdesc;     // forward task descriptors
  const qn_bdesc* bdesc;     // backward task descriptors
  const int32_t* fblob;      // forward tasks' relative extend-add lists
  const int32_t* hlev_ptr;   // batched: supernodes by height (forward levels)
  const int32_t* hlev_sup;
  const int32_t* dlev_ptr;   // batched: supernodes by depth (backward levels)
  const int32_t* dlev_sup;
  const double* vals;
  const double* ftile;       // task-tiled Z copies (persistent kernels): forward / backward
  const double* btile;
  int64_t ftile_n, btile_n;
  double* y;
  double* x;
  double* u;
  unsigned* flags;           // [nbatch][nftask + nbtask] epoch of completion per task
  unsigned* sched;           // [ticket, exited, epoch] forward, then backward; [6] watchdog
  unsigned long long* trace; // diagnostics: kTraceSlots timestamps per forward then backward item, or null
  int32_t ktop;              // dense top (0 = none)
  int32_t lookahead;         // ticket pipe prefetches the next task (many tasks per CTA)
  int32_t fuse_top;          // dense-top tiles run as tasks of the persistent fused kernel
  unsigned* stage_cnt;       // [forward tasks done, top blocks done] (fuse_top)
  int32_t tiled;             // tasks stage Z from the task-tiled copies (TMA) instead of vals (cp.async)
  int32_t opts;              // experiment knob (QN_SOLVE_OPTS): bit 0 = no forward lane groups, bit 1 = ticket lookahead,
                             // bit 2 = dense-top tiles inside the fused persistent kernel, bit 3 = next-tile prefetch, bit 4 = no L2 evict-first hint on the streamed tiles,
                             // bit 5 = shallow lookahead, bit 6 = no lookahead in the backward kernel, bit 7 = no in-task ticket
  const double* stile;       // S^-1 as lower-triangle kTopTile^2 tiles, tile (I,J) at I(I+1)/2 + J
  double* tpart;             // [nbatch][nt][nt][kTopTile][3] partial products
  unsigned* tcnt;            // [nbatch][nt] arrivals per row block
  int32_t tnt;
  const int32_t* tcols;
  const int32_t* tg_ptr;
  const int32_t* tg_idx;
  unsigned long long* ktl;   // diagnostics timeline (qn_system_timeline) or null
  const unsigned long long* passes;
};

inline FactorView factor_view(const qn_factor* f) {
  FactorView v;
  v.n = (int32_t)f->n;
  v.nsup = f->nsup;
  v.nbatch = (int32_t)f->nbatch;
  v.nftask = (int32_t)f->ftask.size();
  v.nbtask = (int32_t)f->btask.size();
  v.bwd_entries = (int32_t)f->bwd_entries;
  v.fwd_entries = (int32_t)f->fwd_entries;
  v.batch_max_nc = f->batch_max_nc;
  v.batch_zmax = f->batch_zmax;
  v.nhlev = (int32_t)f->hlev_ptr.size() - 1;
  v.ndlev = (int32_t)f->dlev_ptr.size() - 1;
  v.hlev_ptr = f->d_hlev_ptr;
  v.hlev_sup = f->d_hlev_sup;
  v.dlev_ptr = f->d_dlev_ptr;
  v.dlev_sup = f->d_dlev_sup;
  v.nvals = f->nvals;
  v.nupd = f->nupd;
  v.sup_col = f->d_sup_col;
  v.sup_row_ptr = f->d_sup_row_ptr;
  v.sup_rows = f->d_sup_rows;
  v.sup_val_ptr = f->d_sup_val_ptr;
  v.sup_upd_ptr = f->d_sup_upd_ptr;
  v.parent = f->d_parent;
  v.cptr = f->d_cptr;
  v.cidx = f->d_cidx;
  v.ftask = f->d_ftask;
  v.btask = f->d_btask;
  v.bfirst = f->d_bfirst;
  v.bcount = f->d_bcount;
  v.fdep_ptr = f->d_fdep_ptr;
  v.fdep_idx = f->d_fdep_idx;
  v.fdesc = f->d_fdesc;
  v.bdesc = f->d_bdesc;
  v.fblob = f->d_fblob;
  v.vals = f->d_vals;
  v.ftile = f->d_ftile;
  v.btile = f->d_btile;
  v.ftile_n = f->ftile_n;
  v.btile_n = f->btile_n;
  v.y = f->d_y;
  v.x = f->d_x;
  v.u = f->d_u;
  v.flags = f->d_flags;
  v.sched = f->d_sched;
  v.trace = f->d_trace;
  v.ktop = f->ktop;
  v.opts = f->solve_opts;
  v.lookahead = f->lookahead;
  // measured slower on c3 (264 vs 249 us per solve: 296 persistent CTAs run the 1891
  // tiles' latency chains ~6 deep, the stand-alone top kernel keeps 6 tiles per SM in flight);
  // kept as an option (QN_SOLVE_OPTS bit 2)
  v.fuse_top = (f->fused && f->ktop > 0 && (f->solve_opts & 4)) ? 1 : 0;
  v.stage_cnt = f->d_stage_cnt;
  v.tiled = f->d_ftile != nullptr;
  v.stile = f->d_stile;
  v.tpart = f->d_tpart;
  v.tcnt = f->d_tcnt;
  v.tnt = f->tnt;
  v.tcols = f->d_tcols;
  v.tg_ptr = f->d_tg_ptr;
  v.tg_idx = f->d_tg_idx;
  v.ktl = f->d_ktl;
  v.passes = f->d_passes;
  return v;
}

constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int kStageIdx = 2048;  // int32 index slots staged in shared memory per task
constexpr int kTraceSlots = 9;   // globaltimer ticket, staged, ready; clock64 ready, data staged, computed, published,
                                 // (forward) own mat-vec done, past the mat-vec barrier
constexpr int kBwdCols = (int)kBwdTaskCols;  // max columns of a backward task
constexpr int kIssueThread = 32;  // warp 1 issues tile copies / takes tickets; warp 0 polls and publishes meanwhile

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void trace_mark(unsigned long long* trace, size_t slot) {
  if (trace && threadIdx.x == 0) trace[slot] = gtime();
}
// frame timeline (kid 4 = forward, 5 = backward), per body pass
__device__ __forceinline__ void solve_tl(const FactorView& F, int kid, int slot) {
  if (F.ktl) {
    const unsigned long long p = *((volatile const unsigned long long*)F.passes);
    if (p < (unsigned long long)kTimelinePasses) F.ktl[(p * kTimelineKernels + kid) * 2 + slot] = gtime();
  }
}
// latest stamp over several CTAs (kid 6 = dense top: the last finalised row block)
__device__ __forceinline__ void solve_tl_max(const FactorView& F, int kid, int slot) {
  if (F.ktl) {
    const unsigned long long p = *((volatile const unsigned long long*)F.passes);
    if (p < (unsigned long long)kTimelinePasses) atomicMax(F.ktl + (p * kTimelineKernels + kid) * 2 + slot, gtime());
  }
}

// SM cycle counter (phases inside one task run on one SM)
__device__ __forceinline__ void trace_clock(unsigned long long* trace, size_t slot) {
  if (trace && threadIdx.x == 0) trace[slot] = (unsigned long long)clock64();
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
// TMA bulk staging of a contiguous tile: thread 0 arms the CTA's mbarrier with
// the byte count and issues one cp.async.bulk; every thread later waits on the
// barrier's phase (parity flips once per task).
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
  if (threadIdx.x == 0) {
    const unsigned m = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n\tfence.mbarrier_init.release.cluster;" ::"r"(m)
                 : "memory");
  }
  __syncthreads();
}
// `stream`: the source is read once per sweep (Z tiles of a factor larger than
// L2, S^-1 tiles): the copy carries an L2 evict-first policy so the streamed
// matrix does not push the small reused data (update vectors, y / x, lists,
// descriptors, flags, right-hand sides) out of L2 — their dependent loads sit
// on every task's critical path.
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, unsigned bytes, uint64_t* mbar,
                                           bool stream = false) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst), m = (unsigned)__cvta_generic_to_shared(mbar);
  if (stream) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "fence.proxy.async.shared::cta;\n\t"
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%2], [%3], %1, [%0], %4;" ::"r"(m),
        "r"(bytes), "r"(d), "l"(src), "l"(pol)
        : "memory");
    return;
  }
  asm volatile(
      "fence.proxy.async.shared::cta;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %1, [%0];" ::"r"(m),
      "r"(bytes), "r"(d), "l"(src)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, unsigned parity) {
  const unsigned m = (unsigned)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(m),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Warp 0 polls n flags (lane-parallel) until all equal `epoch`; then a CTA
// barrier.  A wait longer than 2 s means a scheduling bug: it is recorded in
// sched[6] (checked by the host) instead of hanging the device.
__device__ __forceinline__ void poll_flags_warp0(const unsigned* flags, const int32_t* ids, int n, unsigned epoch,
                                                 unsigned* sched) {
  const unsigned long long t0 = gtime();
  for (int q = threadIdx.x; q < n; q += 32) {
    const unsigned* p = flags + ids[q];
    while (ld_acquire(p) != epoch) {
      __nanosleep(8);
      if (gtime() - t0 > 2000000000ull) {
        atomicOr(&sched[6], 1u);
        break;
      }
    }
  }
  __syncwarp();
}
__device__ __forceinline__ void wait_flags(const unsigned* flags, const int32_t* ids, int n, unsigned epoch,
                                           unsigned* sched) {
  if (threadIdx.x < 32) poll_flags_warp0(flags, ids, n, epoch, sched);
  __syncthreads();
}
// Warp 0 polls a completion counter until it reaches `target`; then a CTA barrier.
__device__ __forceinline__ void wait_count(const unsigned* cnt, unsigned target, unsigned* sched) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = gtime();
    while (ld_acquire(cnt) < target) {
      __nanosleep(32);
      if (gtime() - t0 > 2000000000ull) {
        atomicOr(&sched[6], 1u);
        break;
      }
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void wait_flag_range(const unsigned* flags, int first, int n, unsigned epoch,
                                                unsigned* sched) {
  if (threadIdx.x < 32) {
    const unsigned long long t0 = gtime();
    for (int q = threadIdx.x; q < n; q += 32) {
      const unsigned* p = flags + first + q;
      while (ld_acquire(p) != epoch) {
        __nanosleep(8);
        if (gtime() - t0 > 2000000000ull) {
          atomicOr(&sched[6], 1u);
          break;
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
}

// Dot products of 4 staged Z columns (local kl .. kl+nv-1, column-major with
// leading dimension nr) with the (rows x 3) vector w over rows [r0, r1): lanes
// stride the rows (12 independent chains), then a reduce-scatter butterfly
// (12 -> 6 -> 3 values per lane, then 3 full levels: 18 shuffles instead of
// 60).  On return lane 8j holds column j's three sums in out[0..2].
__device__ __forceinline__ void col4_dots(const double* zt, int nr, const double* w, int kl, int nv, int r0, int r1,
                                          int lane, double (&out)[3]) {
  double a[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) a[q] = 0.0;
  const double* zc = zt + (size_t)kl * nr;
  for (int r = r0 + lane; r < r1; r += 32) {
    const double w0 = w[3 * r + 0], w1 = w[3 * r + 1], w2 = w[3 * r + 2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double l = j < nv ? zc[(size_t)j * nr + r] : 0.0;
      a[3 * j + 0] = fma(l, w0, a[3 * j + 0]);
      a[3 * j + 1] = fma(l, w1, a[3 * j + 1]);
      a[3 * j + 2] = fma(l, w2, a[3 * j + 2]);
    }
  }
  const bool up16 = lane & 16, up8 = lane & 8;
  double b6[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double keep = up16 ? a[i + 6] : a[i], send = up16 ? a[i] : a[i + 6];
    b6[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double keep = up8 ? b6[i + 3] : b6[i], send = up8 ? b6[i] : b6[i + 3];
    out[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i] += __shfl_xor_sync(0xffffffffu, out[i], o);
}

// a += sum over list entries q in [q0, q1) of the update rows u[idx[q]] (3 values each), added in list
// order (bitwise the sequential sum) with the loads of W entries in flight at a time: the sequential
// loop paid one L2 round trip per entry, and these gathers sit on every task's dependent path
template <int W, class Idx>
__device__ __forceinline__ void gather_rows(const double* ub, const Idx* idx, long long q0, long long q1, double& a0,
                                            double& a1, double& a2) {
  long long q = q0;
  for (; q + W <= q1; q += W) {
    double v[W][3];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const double* uc = ub + 3 * (size_t)idx[q + j];
      v[j][0] = __ldcg(uc);
      v[j][1] = __ldcg(uc + 1);
      v[j][2] = __ldcg(uc + 2);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
      a0 += v[j][0];
      a1 += v[j][1];
      a2 += v[j][2];
    }
  }
  const int rem = (int)(q1 - q);
  if (W > 1 && rem > 0) {
    double v[W - 1 > 0 ? W - 1 : 1][3];
#pragma unroll
    for (int j = 0; j < W - 1; ++j)
      if (j < rem) {
        const double* uc = ub + 3 * (size_t)idx[q + j];
        v[j][0] = __ldcg(uc);
        v[j][1] = __ldcg(uc + 1);
        v[j][2] = __ldcg(uc + 2);
      }
#pragma unroll
    for (int j = 0; j < W - 1; ++j)
      if (j < rem) {
        a0 += v[j][0];
        a1 += v[j][1];
        a2 += v[j][2];
      }
  }
}

// publish this task: all of the CTA's global writes are ordered before the flag
// (CTA barrier, then one gpu-scope acq_rel fence — cumulative over the writes
// the barrier ordered — and a relaxed flag store)
__device__ __forceinline__ void publish(unsigned* flag, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
  }
}

// Lookahead ticket pipe of the persistent solve kernels: a CTA holds the ticket
// it works on and the next one, whose 64-byte task descriptor is already being
// copied into shared memory (cp.async, 4 x 16 B) while the current task runs,
// so a task starts without a dependent descriptor load.  Tickets stay
// monotone per CTA and every dependency has a smaller ticket, so the waits
// cannot deadlock (the smallest unfinished ticket is always some CTA's current
// one).
static_assert(sizeof(qn_fdesc) == 64 && sizeof(qn_bdesc) == 64, "descriptor prefetch copies 64 bytes");
struct alignas(16) DescSlot {
  unsigned char bytes[64];
};
__device__ __forceinline__ void desc_prefetch(const FactorView& F, int item, int nfi, int ntt, int total,
                                              DescSlot* dst) {
  if (threadIdx.x < 4 && item < total && !(item >= nfi && item < nfi + ntt)) {
    const unsigned char* src = item < nfi
                                   ? reinterpret_cast<const unsigned char*>(F.fdesc + item / F.nbatch)
                                   : reinterpret_cast<const unsigned char*>(F.bdesc + (item - nfi - ntt) / F.nbatch);
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst->bytes + 16 * threadIdx.x);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 16 * threadIdx.x) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
// Tile prefetch across tasks (tiled factors with ticket lookahead): the Z tile
// buffer of a task is free as soon as its mat-vec has read it, so the bulk copy
// of the CTA's NEXT ticket is issued right there (its descriptor is already in
// shared memory) and streams in behind the epilogue, the flag publication, the
// ticket bookkeeping and the next task's staging / dependency wait.  The
// per-task staging latency (~1.9 of ~6.7 us on c3) leaves the CTA's critical
// path without a second tile buffer.
struct TileAhead {
  bool pre;                  // this task's tile copy is already in flight
  int nxt;                   // the CTA's next ticket (>= total: none)
  const unsigned char* dsc;  // its descriptor in shared memory (null: no lookahead)
};

// Issue the Z tile copy of ticket `item` (descriptor `dsc`, complete and
// visible to the CTA) into zt.  Returns whether a copy is now in flight
// (CTA-uniform: every thread evaluates the same predicate).
template <class IO>
__device__ __forceinline__ bool tile_issue(const FactorView& F, const IO& io, int item, int nfi, int ntt, int total,
                                           const unsigned char* dsc, double* zt, uint64_t* mbar) {
  if (!F.tiled || !dsc || item >= total || !(F.opts & 8)) return false;
  if (item < nfi) {
    const int b = item % F.nbatch;
    if (!io.active(b)) return false;
    if (threadIdx.x == kIssueThread) {
      const qn_fdesc* d = reinterpret_cast<const qn_fdesc*>(dsc);
      const int cnt = (d->hi - d->lo) * (d->hi <= d->nc ? d->hi : d->nc);
      bulk_stage(zt, F.ftile + (size_t)b * F.ftile_n + d->zoff, (unsigned)((cnt + 1) / 2 * 2 * sizeof(double)), mbar,
                 !(F.opts & 16));
    }
    return true;
  }
  if (item < nfi + ntt) return false;  // dense-top tiles stage themselves
  const int b = (item - nfi - ntt) % F.nbatch;
  if (!io.active(b)) return false;
  if (threadIdx.x == kIssueThread) {
    const qn_bdesc* d = reinterpret_cast<const qn_bdesc*>(dsc);
    const int cnt = (d->k1 - d->k0) * d->nr;
    bulk_stage(zt, F.btile + (size_t)b * F.btile_n + d->zoff, (unsigned)((cnt + 1) / 2 * 2 * sizeof(double)), mbar,
               !(F.opts & 16));
  }
  return true;
}

// The CTA's next ticket, taken DURING a task (large factors without lookahead):
// thread kIssueThread issues the counter's atomic before the task's mat-vec and
// turns the ticket into a descriptor copy after it, so the two round trips of
// "take a ticket, read its descriptor" overlap the compute, the epilogue and
// the flag publication instead of following them.  The ticket is held for half
// a task only (a CTA that takes tickets a whole task early delays the tasks it
// holds: measured slower on c3, in the backward sweep above all).
struct NextTicket {
  unsigned* sched;
  int* s_item;     // where the ticket goes
  DescSlot* slot;  // where its descriptor goes
  int nfi, ntt, total;
  bool on;
};
__device__ __forceinline__ void next_take(const NextTicket& n, unsigned& tk) {
  if (n.on && threadIdx.x == kIssueThread) tk = atomicAdd(&n.sched[0], 1u);
}
// the next ticket's descriptor as four 16-byte loads into thread kIssueThread's registers
// (in flight behind the epilogue and the publication; next_store puts them in shared memory)
struct NextRegs {
  unsigned tk;
  uint4 q[4];
};
__device__ __forceinline__ void next_desc(const FactorView& F, const NextTicket& n, NextRegs& r) {
  if (n.on && threadIdx.x == kIssueThread) {
    const int item = (int)r.tk;
    if (item < n.total && !(item >= n.nfi && item < n.nfi + n.ntt)) {
      const uint4* src = item < n.nfi ? reinterpret_cast<const uint4*>(F.fdesc + item / F.nbatch)
                                      : reinterpret_cast<const uint4*>(F.bdesc + (item - n.nfi - n.ntt) / F.nbatch);
#pragma unroll
      for (int q = 0; q < 4; ++q) r.q[q] = __ldg(src + q);
    }
  }
}
__device__ __forceinline__ void next_store(const NextTicket& n, const NextRegs& r) {
  if (n.on && threadIdx.x == kIssueThread) {
    n.s_item[0] = (int)r.tk;
    uint4* dst = reinterpret_cast<uint4*>(n.slot->bytes);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = r.q[q];
  }
}

// What a finished task leaves for the ticket loop to do.
struct TaskDone {
  unsigned* flag;   // completion flag to publish (null: nothing to publish)
  long long tr;     // trace slot of the 'published' stamp (-1: none)
  bool pre;         // the next ticket's tile copy is already in flight
  bool count_fwd;   // fuse_top: count a finished forward task
  bool took;        // the task took the CTA's next ticket (NextTicket)
  NextRegs nx;      // ... and holds its descriptor (thread kIssueThread)
};
__device__ __forceinline__ TaskDone no_task() { return TaskDone{nullptr, -1, false, false, false, NextRegs{}}; }

// publish a finished task (thread 0, after a CTA barrier that followed all of
// the task's global writes): one gpu-scope acq_rel fence — cumulative over the
// writes the barrier ordered — and a relaxed flag store
__device__ __forceinline__ void publish_done(const FactorView& F, const TaskDone& dn, unsigned epoch) {
  if (dn.flag) {
    asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(dn.flag), "r"(epoch) : "memory");
    if (dn.count_fwd) atomicAdd(F.stage_cnt, 1u);  // after the fence
    if (dn.tr >= 0 && F.trace) F.trace[dn.tr] = (unsigned long long)clock64();
  }
}

// The ticket loop of a persistent solve kernel: body(item, descriptor, tile
// prefetch state) runs one task up to (not including) its publication and
// returns a TaskDone.
//
// With lookahead (many tasks per CTA: throughput-bound, e.g. configs[2]) a CTA
// holds three tickets: the one it works on, the next one (descriptor already in
// shared memory) and the one after (its atomic is in flight: issued a task
// early by thread 0 and consumed a task later, so the counter's round trip is
// off the per-task path).  One CTA barrier separates two tasks: it orders the
// finished task's writes before thread 0's fence + flag store and frees the
// task's shared memory; thread 0 publishes AFTER that barrier while the other
// warps already stage the next task (the fence's round trip overlaps their
// loads).  Tickets stay monotone per CTA and every dependency has a smaller
// ticket, so the smallest unfinished ticket is always some CTA's current one
// and the waits cannot deadlock.
// Without lookahead (few tasks per CTA: latency-bound, e.g. configs[1]) a CTA
// never holds a ticket it is not working on, so an idle CTA can start every
// ready task; the task reads its descriptor from global memory.
template <bool kTiled, class Body>
__device__ __forceinline__ void ticket_loop(const FactorView& F, unsigned* sched, int* s_item, int nfi, int ntt,
                                            int total, DescSlot* s_desc, const unsigned& epoch, bool look, Body body) {
  if (look) {
    const bool deep = !(F.opts & 32);  // the ticket after next is taken a task early
    unsigned ahead = 0;  // thread 0: the ticket after next
    if (threadIdx.x == 0) {
      s_item[0] = (int)atomicAdd(&sched[0], 1u);
      s_item[1] = (int)atomicAdd(&sched[0], 1u);
      if (deep) ahead = atomicAdd(&sched[0], 1u);
    }
    __syncthreads();
    int cur = s_item[0], nxt = s_item[1], slot = 0, it = 0;
    desc_prefetch(F, cur, nfi, ntt, total, &s_desc[0]);
    desc_prefetch(F, nxt, nfi, ntt, total, &s_desc[1]);
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // the first descriptor
    __syncthreads();
    bool pre = false;  // cur's Z tile copy was already issued by the previous task (CTA-uniform)
    while (cur < total) {
      const TaskDone dn = body(cur, s_desc[slot].bytes, TileAhead{pre, nxt, s_desc[slot ^ 1].bytes},
                               NextTicket{sched, s_item, s_desc, nfi, ntt, total, false});
      asm volatile("cp.async.wait_group 0;" ::: "memory");  // nxt's descriptor (issued a task ago) has landed
      if (threadIdx.x == 0) s_item[it & 1] = deep ? (int)ahead : (int)atomicAdd(&sched[0], 1u);
      __syncthreads();  // the one barrier between two tasks
      if (threadIdx.x == 0) {
        publish_done(F, dn, epoch);
        if (deep) ahead = atomicAdd(&sched[0], 1u);
      }
      const int nn = s_item[it & 1];
      desc_prefetch(F, nn, nfi, ntt, total, &s_desc[slot]);
      cur = nxt;
      nxt = nn;
      slot ^= 1;
      ++it;
      pre = dn.pre;
    }
  } else {
    const bool late = kTiled && !(F.opts & 128);  // the next ticket is taken during the task (NextTicket)
    bool have = false;
    for (int it = 0;; ++it) {
      if (!have) {
        __syncthreads();  // the previous task is done with shared memory
        if (threadIdx.x == 0) s_item[0] = (int)atomicAdd(&sched[0], 1u);
        __syncthreads();
      }
      const int cur = s_item[0];
      if (cur >= total) break;
      const unsigned char* dp =
          cur >= nfi && cur < nfi + ntt ? nullptr
          : have                        ? s_desc[(it & 1) ^ 1].bytes  // copied by the previous task
          : cur < nfi ? reinterpret_cast<const unsigned char*>(F.fdesc + cur / F.nbatch)
                      : reinterpret_cast<const unsigned char*>(F.bdesc + (cur - nfi - ntt) / F.nbatch);
      const NextTicket nt{sched, s_item, &s_desc[it & 1], nfi, ntt, total, late};
      const TaskDone dn = body(cur, dp, TileAhead{false, total, nullptr}, nt);
      __syncthreads();
      if (threadIdx.x == 0) publish_done(F, dn, epoch);
      have = kTiled && dn.took;
      if (have) {  // the next ticket and its descriptor arrive behind the publication's fence
        next_store(nt, dn.nx);
        __syncthreads();
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// persistent-CTA ticket loop helpers; sched = [ticket, exited, epoch]
__device__ __forceinline__ void cta_exit(unsigned* sched, unsigned epoch, const FactorView& F, int kid) {
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned e = atomicAdd(&sched[1], 1u);
    if (e == gridDim.x - 1) {  // last CTA out: reset for the next launch
      solve_tl(F, kid, 1);
      sched[0] = 0;
      sched[1] = 0;
      if (F.fuse_top) {
        F.stage_cnt[0] = 0;
        F.stage_cnt[1] = 0;
      }
      __threadfence();
      atomicExch(&sched[2], epoch + 1);
    }
  }
}

// IO: struct with
//   __device__ bool active(int b) const;
//   __device__ void rhs(int b, int row, double (&v)[3]) const;   // factor row
//   __device__ void store(int b, int row, const double (&v)[3]) const;
// One forward task (row block of one supernode): stage, wait for the
// children, gather their updates, v = Z f, publish.
template <bool kTiled, class IO>
__device__ __forceinline__ TaskDone fwd_task(const FactorView& F, const IO& io, int item, unsigned epoch, double* sm,
                                             int lane, int warp, uint64_t* mbar, unsigned& phase,
                                             const qn_fdesc* sdesc, const TileAhead& ahead, const NextTicket& nt,
                                             int nfi, int ntt, int total) {
  double* zt = sm;
  const int tid = item / F.nbatch;
  const int b = item % F.nbatch;
  if (!io.active(b)) return no_task();
  trace_mark(F.trace, kTraceSlots * (size_t)item + 0);
  const qn_fdesc d = *sdesc;  // shared memory (lookahead prefetch) or global memory
  const int lo = d.lo, hi = d.hi, rg = d.rg, c0 = d.c0, nc = d.nc, nr = d.nr, blo = d.blo;
  const int R = hi - lo;
  const int kmax = hi <= nc ? hi : nc;  // rows inside the triangle need k <= row only
  // shared memory: [tile (R x kmax, even) | f (nc x 3)] ... [index staging at fwd_entries], whose
  // space the k-slice partial sums reuse once the gathers are done (barrier before the mat-vec)
  double* f = sm + ((R * kmax + 1) & ~1);
  int* sidx = (int*)(sm + F.fwd_entries);
  double* part = (double*)sidx;
  const double* ub = F.u + (size_t)b * F.nupd * 3;
  // ---- stage everything that does not depend on the children ----
  const int nptr_bot = blo < hi ? hi - blo + 1 : 0;
  const int nblob = nc + 1 + nptr_bot + d.ntop + d.nbot;
  const int* gblob = F.fblob + d.blob;
  const bool staged = nblob <= kStageIdx;
  const int* sp_top = staged ? sidx : gblob;  // relative extend-add lists: [sp_top | sp_bot | si_top | si_bot]
  const int* sp_bot = sp_top + nc + 1;
  const int* si_top = sp_bot + nptr_bot;
  const int* si_bot = si_top + d.ntop;
  if (kTiled) {
    // Large factors (throughput-bound): the warps split the roles so that the
    // task's independent round trips overlap — warp 1 issues the tile's bulk
    // copy (rows [lo, hi) x k [0, kmax) = zt[k * R + (r - lo)], one contiguous
    // block), warp 0 polls the children's flags at once, warps 1..7 copy the
    // lists (asynchronously) and load the right-hand side.
    if (threadIdx.x == kIssueThread && !ahead.pre) {
      const int cnt = R * kmax;
      bulk_stage(zt, F.ftile + (size_t)b * F.ftile_n + d.zoff, (unsigned)((cnt + 1) / 2 * 2 * sizeof(double)), mbar,
                 !(F.opts & 16));
    }
    if (warp == 0) {
      poll_flags_warp0(F.flags + (size_t)b * (F.nftask + F.nbtask), F.fdep_idx + d.dep0, d.dep1 - d.dep0, epoch,
                       F.sched);
    } else {
      const int t = threadIdx.x - 32, nt = kSolveThreads - 32;
      if (staged)
        for (int q = t; q < nblob; q += nt) cp_async4(sidx + q, gblob + q);
      for (int p = t; p < nc; p += nt) {
        double v[3];
        io.rhs(b, c0 + p, v);
        f[3 * p + 0] = v[0];
        f[3 * p + 1] = v[1];
        f[3 * p + 2] = v[2];
      }
      cp_async_wait_all();
    }
    trace_mark(F.trace, kTraceSlots * (size_t)item + 1);
    __syncthreads();
  } else {  // small factors: straight from vals, which the backward re-reads from L2
    // lanes over the tile's rows; a tile of R < 32 rows puts 32 / R columns on each warp
    const double* Zg = F.vals + (size_t)b * F.nvals + d.zoff;
    const int Ls = R < 32 ? 32 / R : 1, subs = R < 32 ? lane / R : 0, r0 = R < 32 ? lane - subs * R : lane;
    if (subs < Ls)
      for (int k = warp * Ls + subs; k < kmax; k += kSolveWarps * Ls)
        for (int rr = r0; rr < R; rr += 32) cp_async8(zt + k * R + rr, Zg + (int64_t)k * nr + rr);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (staged)
      for (int q = threadIdx.x; q < nblob; q += blockDim.x) sidx[q] = __ldg(gblob + q);
    for (int p = threadIdx.x; p < nc; p += blockDim.x) {
      double v[3];
      io.rhs(b, c0 + p, v);
      f[3 * p + 0] = v[0];
      f[3 * p + 1] = v[1];
      f[3 * p + 2] = v[2];
    }
    trace_mark(F.trace, kTraceSlots * (size_t)item + 1);
    wait_flags(F.flags + (size_t)b * (F.nftask + F.nbtask), F.fdep_idx + d.dep0, d.dep1 - d.dep0, epoch, F.sched);
  }
  trace_mark(F.trace, kTraceSlots * (size_t)item + 2);
  trace_clock(F.trace, kTraceSlots * (size_t)item + 3);
  // ---- dependent gathers: children's updates on J (f) and on this task's bottom rows ----
  for (int p = threadIdx.x; p < nc; p += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    gather_rows<4>(ub, si_top, sp_top[p], sp_top[p + 1], a0, a1, a2);
    f[3 * p + 0] -= a0;
    f[3 * p + 1] -= a1;
    f[3 * p + 2] -= a2;
  }
  const int rr = lo + threadIdx.x;  // row owned by this thread in the epilogue
  double e0 = 0.0, e1 = 0.0, e2 = 0.0;
  if (threadIdx.x < R && rr >= nc) {
    const int pr = rr - blo;
    gather_rows<4>(ub, si_bot, sp_bot[pr], sp_bot[pr + 1], e0, e1, e2);
  }
  if (kTiled) {
    mbar_wait(mbar, phase);
    phase ^= 1u;
  } else {
    cp_async_wait_all();
  }
  __syncthreads();
  NextRegs nx{};
  if (kTiled) next_take(nt, nx.tk);  // the counter's round trip runs behind the mat-vec
  trace_clock(F.trace, kTraceSlots * (size_t)item + 4);
  // ---- rows of v = Z f from shared memory: warp -> (row group g, k-slice j);
  // a tile of R < 32 rows (wide supernodes) also splits each warp's k-slice
  // over L = 32 / R lane groups (lane = sub R + row), so every lane works ----
  const int lg = __ffs(rg) - 1;  // rg is a power of two: shifts instead of integer divisions
  const int ks = kSolveWarps >> lg;
  const int g = warp >> (3 - lg), j = warp & (ks - 1);
  static_assert(kSolveWarps == 8, "warp -> (row group, k-slice) shifts assume 8 warps");
  // k-slices start at even k, so the f values of two consecutive k (6 doubles) are three aligned
  // 16-byte broadcast loads
  const int per = (((kmax + ks - 1) >> (3 - lg)) + 1) & ~1;
  const int kb = j * per, ke = min(kmax, kb + per);
  const int L = (R < 32 && !(F.opts & 1)) ? 32 / R : 1;  // rg == 1 whenever R < 32
  const int sub = L > 1 ? lane / R : 0;
  const int rl = L > 1 ? lane - sub * R : 32 * g + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  if (g < rg && rl < R && sub < L) {
    // four independent chains per coordinate (k mod 4 within the lane group's pairs): the FP64 FMA
    // latency, not its throughput, bounds a row's dot product
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
    int k = kb + 2 * sub;  // lane group `sub` takes the k pairs sub, sub + L, ...
#pragma unroll 2
    for (; k + 2 * L + 1 < ke; k += 4 * L) {
      const int k2 = k + 2 * L;
      const double l = zt[k * R + rl], m = zt[(k + 1) * R + rl];
      const double n = zt[k2 * R + rl], o = zt[(k2 + 1) * R + rl];
      const double2 f01 = *reinterpret_cast<const double2*>(f + 3 * k);
      const double2 f23 = *reinterpret_cast<const double2*>(f + 3 * k + 2);
      const double2 f45 = *reinterpret_cast<const double2*>(f + 3 * k + 4);
      const double2 g01 = *reinterpret_cast<const double2*>(f + 3 * k2);
      const double2 g23 = *reinterpret_cast<const double2*>(f + 3 * k2 + 2);
      const double2 g45 = *reinterpret_cast<const double2*>(f + 3 * k2 + 4);
      a0 = fma(l, f01.x, a0);
      a1 = fma(l, f01.y, a1);
      a2 = fma(l, f23.x, a2);
      b0 = fma(m, f23.y, b0);
      b1 = fma(m, f45.x, b1);
      b2 = fma(m, f45.y, b2);
      c0 = fma(n, g01.x, c0);
      c1 = fma(n, g01.y, c1);
      c2 = fma(n, g23.x, c2);
      d0 = fma(o, g23.y, d0);
      d1 = fma(o, g45.x, d1);
      d2 = fma(o, g45.y, d2);
    }
    for (; k + 1 < ke; k += 2 * L) {
      const double l = zt[k * R + rl], m = zt[(k + 1) * R + rl];
      const double2 f01 = *reinterpret_cast<const double2*>(f + 3 * k);
      const double2 f23 = *reinterpret_cast<const double2*>(f + 3 * k + 2);
      const double2 f45 = *reinterpret_cast<const double2*>(f + 3 * k + 4);
      a0 = fma(l, f01.x, a0);
      a1 = fma(l, f01.y, a1);
      a2 = fma(l, f23.x, a2);
      b0 = fma(m, f23.y, b0);
      b1 = fma(m, f45.x, b1);
      b2 = fma(m, f45.y, b2);
    }
    if (k < ke) {
      const double l = zt[k * R + rl];
      a0 = fma(l, f[3 * k + 0], a0);
      a1 = fma(l, f[3 * k + 1], a1);
      a2 = fma(l, f[3 * k + 2], a2);
    }
    a0 += c0;
    a1 += c1;
    a2 += c2;
    b0 += d0;
    b1 += d1;
    b2 += d2;
    a0 += b0;
    a1 += b1;
    a2 += b2;
  }
  if (L > 1) {  // lane groups -> group 0, in group order (shuffles, fixed order)
    double s0 = a0, s1 = a1, s2 = a2;
    for (int q = 1; q < L; ++q) {
      const int src = q * R + (lane < R ? lane : 0);
      const double t0 = __shfl_sync(0xffffffffu, a0, src), t1 = __shfl_sync(0xffffffffu, a1, src),
                   t2 = __shfl_sync(0xffffffffu, a2, src);
      s0 += t0;
      s1 += t1;
      s2 += t2;
    }
    a0 = s0;
    a1 = s1;
    a2 = s2;
  }
  part[3 * threadIdx.x + 0] = a0;
  part[3 * threadIdx.x + 1] = a1;
  part[3 * threadIdx.x + 2] = a2;
  trace_clock(F.trace, kTraceSlots * (size_t)item + 7);
  asm volatile("cp.async.wait_group 0;" ::: "memory");  // the next ticket's descriptor has landed
  __syncthreads();
  trace_clock(F.trace, kTraceSlots * (size_t)item + 8);
  // the tile is consumed: the next ticket's copy streams in behind the epilogue and the publication
  const bool issued = tile_issue(F, io, ahead.nxt, nfi, ntt, total, ahead.dsc, zt, mbar);
  if (kTiled) next_desc(F, nt, nx);  // the descriptor's round trip runs behind the epilogue and the publication
  if (threadIdx.x < R) {
    const int gg = threadIdx.x >> 5;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int jj = 0; jj < ks; ++jj) {
      const int t = (gg * ks + jj) * 32 + lane;
      v0 += part[3 * t + 0];
      v1 += part[3 * t + 1];
      v2 += part[3 * t + 2];
    }
    if (rr < nc) {
      double* yg = F.y + ((size_t)b * F.n + c0 + rr) * 3;
      yg[0] = v0;
      yg[1] = v1;
      yg[2] = v2;
    } else {
      double* us = F.u + ((size_t)b * F.nupd + d.upd0 + (rr - nc)) * 3;
      __stcg(us + 0, e0 + v0);
      __stcg(us + 1, e1 + v1);
      __stcg(us + 2, e2 + v2);
    }
  }
  trace_clock(F.trace, kTraceSlots * (size_t)item + 5);
  return TaskDone{F.flags + (size_t)b * (F.nftask + F.nbtask) + tid, (long long)(kTraceSlots * (size_t)item + 6),
                  issued, F.fuse_top != 0, kTiled && nt.on, nx};
}

// One backward task (column block of one supernode).  fused: forward and
// backward share one persistent kernel, so y_J is waited for explicitly.
template <bool kTiled, class IO>
__device__ __forceinline__ TaskDone bwd_task(const FactorView& F, const IO& io, int item, unsigned epoch, double* sm,
                                             int lane, int warp, bool fused, uint64_t* mbar, unsigned& phase,
                                             const qn_bdesc* sdesc, const TileAhead& ahead, const NextTicket& nt,
                                             int nfi, int ntt, int total) {
  double* zt = sm;
  const int tid = item / F.nbatch;
  const int b = item % F.nbatch;
  if (!io.active(b)) return no_task();
  trace_mark(F.trace, kTraceSlots * ((size_t)F.nftask * F.nbatch + item) + 0);
  const qn_bdesc d = *sdesc;  // shared memory (lookahead prefetch) or global memory
  const int k0 = d.k0, k1 = d.k1, c0 = d.c0, nc = d.nc, nr = d.nr;
  const int64_t R0 = d.rows;
  double* w = sm + F.bwd_entries;
  double* pre = w + 3 * nr;  // [kBwdCols][3] y_J part of each column
  double** sdst = (double**)(pre + 3 * kBwdCols);  // [kBwdCols] io destination of each column
  int* srow = (int*)(sdst + kBwdCols);
  const bool staged = nr - nc <= kStageIdx;
  // ---- stage: Z columns [k0, k1) (zeros above the diagonal), y_J, below-row ids ----
  if (kTiled) {  // Z columns [k0, k1) x all rows, zeros above the diagonal: one contiguous block
    if (threadIdx.x == kIssueThread && !ahead.pre) {
      const int cnt = (k1 - k0) * nr;
      bulk_stage(zt, F.btile + (size_t)b * F.btile_n + d.zoff, (unsigned)((cnt + 1) / 2 * 2 * sizeof(double)),
                 mbar, !(F.opts & 16));
    }
  } else {
    const double* Zg = F.vals + (size_t)b * F.nvals + d.zoff;
    const int cnt = (k1 - k0) * nr;
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int kk = e / nr, r = e - kk * nr;
      if (r >= k0 + kk)
        cp_async8(zt + e, Zg + e);
      else
        zt[e] = 0.0;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (fused)  // the forward of s may still be running: y_J must be complete
    wait_flag_range(F.flags + (size_t)b * (F.nftask + F.nbtask), d.fwd0, d.nfwd, epoch, F.sched);
  const double* yg = F.y + ((size_t)b * F.n + c0) * 3;
  if (kTiled && !fused) {
    // y_J and the below-row ids as asynchronous copies: one round trip together with the
    // destinations.  (The 8-byte copies allocate in L1: only in the stand-alone backward
    // kernel, where y is never written; the fused kernel keeps the L2 loads below.)
    for (int q = threadIdx.x; q < 3 * nc; q += blockDim.x) cp_async8(w + q, yg + q);
    if (staged)
      for (int q = threadIdx.x; q < nr - nc; q += blockDim.x) cp_async4(srow + q, F.sup_rows + R0 + nc + q);
    for (int q = threadIdx.x; q < k1 - k0; q += blockDim.x) sdst[q] = io.dest(b, c0 + k0 + q);
    cp_async_wait_all();
  } else {
    for (int q = threadIdx.x; q < nc; q += blockDim.x) {
      w[3 * q + 0] = __ldcg(yg + 3 * q + 0);
      w[3 * q + 1] = __ldcg(yg + 3 * q + 1);
      w[3 * q + 2] = __ldcg(yg + 3 * q + 2);
    }
    if (staged)
      for (int q = threadIdx.x; q < nr - nc; q += blockDim.x) srow[q] = F.sup_rows[R0 + nc + q];
    for (int q = threadIdx.x; q < k1 - k0; q += blockDim.x) sdst[q] = io.dest(b, c0 + k0 + q);
  }
  const size_t tb = kTraceSlots * ((size_t)F.nftask * F.nbatch + item);
  trace_mark(F.trace, tb + 1);
  if (kTiled) {
    mbar_wait(mbar, phase);
    phase ^= 1u;
  } else {
    cp_async_wait_all();
  }
  __syncthreads();
  // ---- before the parent is done: the y_J part of every column, 4 columns per warp.
  // Fewer than kSolveWarps column quads (tall fronts, few columns per task):
  // each quad's rows are split over rs warps and the slices summed in order ----
  const int ncols = k1 - k0;
  const int nquads = (ncols + 3) / 4;
  // tall fronts with few columns per task (the widest separators' children,
  // nr >= 1024): split each quad's rows over the idle warps; on shorter
  // fronts the extra barrier costs more than it saves (c2 -1.8 %)
  const int rs = (nquads >= kSolveWarps || nr < 1024) ? 1 : kSolveWarps / nquads;
  __shared__ double slp[kSolveWarps][4][3];
  if (rs > 1) {
    const int quad = warp / rs, slice = warp % rs, kl = 4 * quad;
    double a[3] = {0.0, 0.0, 0.0};
    if (quad < nquads) {
      const int r0 = k0 + kl, len = nc - r0, per = (len + rs - 1) / rs;
      const int ra = r0 + slice * per, rb = min(nc, ra + per);
      col4_dots(zt, nr, w, kl, min(4, ncols - kl), ra, max(ra, rb), lane, a);
    }
    if ((lane & 7) == 0) {
      slp[warp][lane >> 3][0] = a[0];
      slp[warp][lane >> 3][1] = a[1];
      slp[warp][lane >> 3][2] = a[2];
    }
    __syncthreads();
    if ((int)threadIdx.x < 3 * ncols) {
      const int c = threadIdx.x / 3, q = threadIdx.x - 3 * c;
      double v = 0.0;
      for (int sl = 0; sl < rs; ++sl) v += slp[(c >> 2) * rs + sl][c & 3][q];
      pre[threadIdx.x] = v;
    }
  } else {
    for (int kl = 4 * warp; kl < ncols; kl += 4 * kSolveWarps) {
      double a[3];
      const int j = lane >> 3;
      col4_dots(zt, nr, w, kl, min(4, ncols - kl), k0 + kl, nc, lane, a);
      if ((lane & 7) == 0 && kl + j < ncols) {
        pre[3 * (kl + j) + 0] = a[0];
        pre[3 * (kl + j) + 1] = a[1];
        pre[3 * (kl + j) + 2] = a[2];
      }
    }
  }
  if (d.nwait > 0)
    wait_flag_range(F.flags + (size_t)b * (F.nftask + F.nbtask) + F.nftask, d.wait0, d.nwait, epoch, F.sched);
  if (F.fuse_top && d.top_child) wait_count(F.stage_cnt + 1, (unsigned)F.tnt, F.sched);  // x_T complete
  trace_mark(F.trace, tb + 2);
  trace_clock(F.trace, tb + 3);
  const double* xg = F.x + (size_t)b * F.n * 3;
  for (int q = threadIdx.x; q < nr - nc; q += blockDim.x) {
    const int row = staged ? srow[q] : F.sup_rows[R0 + nc + q];
    w[3 * (nc + q) + 0] = -__ldcg(xg + 3 * row + 0);
    w[3 * (nc + q) + 1] = -__ldcg(xg + 3 * row + 1);
    w[3 * (nc + q) + 2] = -__ldcg(xg + 3 * row + 2);
  }
  __syncthreads();
  NextRegs nx{};
  if (kTiled) next_take(nt, nx.tk);  // the counter's round trip runs behind the second pass
  trace_clock(F.trace, tb + 4);
  // ---- the -x_below part, plus the staged y_J part ----
  if (rs > 1) {
    const int quad = warp / rs, slice = warp % rs, kl = 4 * quad;
    double a[3] = {0.0, 0.0, 0.0};
    if (quad < nquads) {
      const int len = nr - nc, per = (len + rs - 1) / rs;
      const int ra = nc + slice * per, rb = min(nr, ra + per);
      col4_dots(zt, nr, w, kl, min(4, ncols - kl), ra, max(ra, rb), lane, a);
    }
    __syncthreads();  // the y_J pass's slp reads are done
    if ((lane & 7) == 0) {
      slp[warp][lane >> 3][0] = a[0];
      slp[warp][lane >> 3][1] = a[1];
      slp[warp][lane >> 3][2] = a[2];
    }
    __syncthreads();
    if ((int)threadIdx.x < ncols) {
      const int c = threadIdx.x;
      double v[3];
      for (int q = 0; q < 3; ++q) {
        double t = 0.0;
        for (int sl = 0; sl < rs; ++sl) t += slp[(c >> 2) * rs + sl][c & 3][q];
        v[q] = t + pre[3 * c + q];
      }
      double* xo = F.x + ((size_t)b * F.n + c0 + k0 + c) * 3;
      xo[0] = v[0];
      xo[1] = v[1];
      xo[2] = v[2];
      double* d = sdst[c];
      d[0] = v[0];
      d[1] = v[1];
      d[2] = v[2];
    }
  } else {
    for (int kl = 4 * warp; kl < ncols; kl += 4 * kSolveWarps) {
      double a[3];
      const int j = lane >> 3;
      col4_dots(zt, nr, w, kl, min(4, ncols - kl), nc, nr, lane, a);
      if ((lane & 7) == 0 && kl + j < ncols) {
        const int k = k0 + kl + j;
        const double v[3] = {a[0] + pre[3 * (kl + j) + 0], a[1] + pre[3 * (kl + j) + 1],
                             a[2] + pre[3 * (kl + j) + 2]};
        double* xo = F.x + ((size_t)b * F.n + c0 + k) * 3;
        xo[0] = v[0];
        xo[1] = v[1];
        xo[2] = v[2];
        double* d = sdst[kl + j];
        d[0] = v[0];
        d[1] = v[1];
        d[2] = v[2];
      }
    }
  }
  trace_clock(F.trace, tb + 5);
  if (kTiled) next_desc(F, nt, nx);  // the descriptor's round trip runs behind the publication
  bool issued = false;
  if (F.opts & 8) {  // next-tile prefetch (experiment): needs its own barrier after the last tile read
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // the next ticket's descriptor has landed
    __syncthreads();
    issued = tile_issue(F, io, ahead.nxt, nfi, ntt, total, ahead.dsc, zt, mbar);
  }
  return TaskDone{F.flags + (size_t)b * (F.nftask + F.nbtask) + F.nftask + tid, (long long)(tb + 6), issued, false,
                  kTiled && nt.on, nx};
}

template <class IO>
__global__ void __launch_bounds__(kSolveThreads, 3) sptrsv_forward(FactorView F, IO io) {
  pdl_entry();
  // smem: ztile | f[nc*3] (per task) ... index staging (int32) / part[256*3] at fwd_entries
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_item[2];
  __shared__ unsigned s_epoch;
  __shared__ uint64_t s_mbar;
  unsigned phase = 0;
  mbar_init(&s_mbar);
  unsigned* sched = F.sched;
  if (threadIdx.x == 0) s_epoch = *((volatile unsigned*)&sched[2]);
  if (threadIdx.x == 0 && blockIdx.x == 0) solve_tl(F, 4, 0);
  const int total = F.nftask * F.nbatch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ DescSlot s_desc[2];
  auto run = [&](auto tiled) {
    constexpr bool kT = decltype(tiled)::value;
    ticket_loop<kT>(F, sched, s_item, total, 0, total, s_desc, s_epoch, F.lookahead != 0,
                    [&](int cur, const unsigned char* dsc, const TileAhead& ahead, const NextTicket& nt) {
                      return fwd_task<kT>(F, io, cur, s_epoch, sm, lane, warp, &s_mbar, phase,
                                          reinterpret_cast<const qn_fdesc*>(dsc), ahead, nt, total, 0, total);
                    });
  };
  if (F.tiled)
    run(std::true_type{});
  else
    run(std::false_type{});
  cta_exit(sched, s_epoch, F, 4);
}

template <class IO>
__global__ void __launch_bounds__(kSolveThreads, 2) sptrsv_backward(FactorView F, IO io) {
  pdl_entry();
  // smem: ztile[bwd_entries] | w[max_rows*3] = [y_J; -x_below] | pre[kBwdCols*3] | dest[kBwdCols] | row staging
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_item[2];
  __shared__ unsigned s_epoch;
  __shared__ uint64_t s_mbar;
  unsigned phase = 0;
  mbar_init(&s_mbar);
  unsigned* sched = F.sched + 3;
  if (threadIdx.x == 0) s_epoch = *((volatile unsigned*)&sched[2]);
  if (threadIdx.x == 0 && blockIdx.x == 0) solve_tl(F, 5, 0);
  const int total = F.nbtask * F.nbatch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ DescSlot s_desc[2];
  auto run = [&](auto tiled) {
    constexpr bool kT = decltype(tiled)::value;
    ticket_loop<kT>(F, sched, s_item, 0, 0, total, s_desc, s_epoch, F.lookahead && !(F.opts & 64),
                    [&](int cur, const unsigned char* dsc, const TileAhead& ahead, const NextTicket& nt) {
                      return bwd_task<kT>(F, io, cur, s_epoch, sm, lane, warp, false, &s_mbar, phase,
                                          reinterpret_cast<const qn_bdesc*>(dsc), ahead, nt, 0, 0, total);
                    });
  };
  if (F.tiled)
    run(std::true_type{});
  else
    run(std::false_type{});
  cta_exit(sched, s_epoch, F, 5);
}

// ---- dense top: x_T = S^-1 g_T, g_T = b_T - (updates of the subtrees below T) ----
// x_T = S^-1 g_T with the symmetric S^-1 read once from half storage: CTA per
// lower-triangle tile (I, J) (64 x 64, stored with leading dimension 65 so the
// row and the column products both read shared memory without bank
// conflicts; the TMA engine brings the tile in one bulk copy).  A tile gives
// the row-block product S_IJ g_J (-> block I) and, off the diagonal, the
// transposed product S_IJ^T g_I (-> block J).  Each row block receives exactly
// nt partials (slot = the other block index); the CTA that delivers the last
// one (arrival counter) sums them in slot order — a fixed order, so the result
// is bitwise reproducible — and writes x_T.  Half the bytes of the dense K x K
// product (c3: 64 MB instead of 118 MB per solve).  Small CTAs (37 KB of shared
// memory, the partial products reuse the tile buffer) keep 6 tiles in flight
// per SM: the per-tile phases are latency chains, so concurrency matters more
// than pipelining inside one CTA (a persistent double-buffered variant was
// slower: 45 vs 33 us on c3).
constexpr int kTopLD = kTopTile + 1;
constexpr int kTopTileEntries = kTopTile * kTopLD;  // 4160 doubles = 33,280 B (a multiple of 16)

// One tile (I, J) of the symmetric top apply.  st: kTopTileEntries doubles of
// shared memory (the tile, then the partial products), gI / gJ: kTopTile * 3
// each, s_last: 2 ints.  The tile's bulk copy is issued here; with
// `after_forward` (the top-fused persistent solve) the g_T gather waits until
// every forward task has completed (the tile streams in meanwhile) and a
// finalised row block is counted in stage_cnt[1] for the backward tasks.
template <class IO>
__device__ __forceinline__ void top_tile(const FactorView& F, const IO& io, int t, int b, double* st, double* gI,
                                         double* gJ, int* s_last, uint64_t* mbar, unsigned& phase,
                                         bool after_forward) {
  constexpr int T = kTopTile, LD = kTopLD, NQ = kSolveThreads / T;  // NQ = 4 column / row quarters
  double* red = st;  // [2][NQ][T * 3] partial products, after the tile is consumed
  const int K = F.ktop, nt = F.tnt;
  if (threadIdx.x == 0)
    bulk_stage(st, F.stile + (size_t)t * kTopTileEntries, kTopTileEntries * sizeof(double), mbar, !(F.opts & 16));
  int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  const int J = t - I * (I + 1) / 2;
  if (after_forward) wait_count(F.stage_cnt, (unsigned)F.nftask, F.sched);
  // g_T of this tile's two row blocks, formed here (b_T minus the updates of the
  // subtrees below T, in list order) while the tile streams in — no separate
  // gather kernel; each row block's g is formed by every tile that needs it
  const double* ub = F.u + (size_t)b * F.nupd * 3;
  for (int e = threadIdx.x; e < 2 * T; e += blockDim.x) {
    const int blk = e < T ? I : J, r = e < T ? e : e - T;
    double* gd = (e < T ? gI : gJ) + 3 * r;
    const int k = blk * T + r;
    if (k < K) {
      double v[3];
      io.rhs(b, F.tcols[k], v);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      gather_rows<4>(ub, F.tg_idx, F.tg_ptr[k], F.tg_ptr[k + 1], a0, a1, a2);
      gd[0] = v[0] - a0;
      gd[1] = v[1] - a1;
      gd[2] = v[2] - a2;
    } else {
      gd[0] = gd[1] = gd[2] = 0.0;
    }
  }
  mbar_wait(mbar, phase);
  phase ^= 1u;
  __syncthreads();
  const int i = threadIdx.x % T, q = threadIdx.x / T;
  // Row i of S_IJ g_J over the columns of quarter q and, off the diagonal, column i of S_IJ against
  // g_I over the rows of quarter q, two entries per step: the g values of two consecutive rows
  // (6 doubles) are three aligned 16-byte broadcast loads, and every product keeps two FMA chains per
  // coordinate (the kernel is bound by shared-memory wavefronts and by the FP64 FMA latency).
  double r0 = 0.0, r1 = 0.0, r2 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
  {
    double r3 = 0.0, r4 = 0.0, r5 = 0.0, c3 = 0.0, c4 = 0.0, c5 = 0.0;
    const int j0 = q * (T / NQ);
    static_assert((kTopTile / (kSolveThreads / kTopTile)) % 2 == 0, "quarters hold an even number of columns");
#pragma unroll
    for (int t = 0; t < T / NQ; t += 2) {
      const int j = j0 + t;
      const double s0 = st[i + j * LD], s1 = st[i + (j + 1) * LD];
      const double2 a01 = *reinterpret_cast<const double2*>(gJ + 3 * j);
      const double2 a23 = *reinterpret_cast<const double2*>(gJ + 3 * j + 2);
      const double2 a45 = *reinterpret_cast<const double2*>(gJ + 3 * j + 4);
      r0 = fma(s0, a01.x, r0);
      r1 = fma(s0, a01.y, r1);
      r2 = fma(s0, a23.x, r2);
      r3 = fma(s1, a23.y, r3);
      r4 = fma(s1, a45.x, r4);
      r5 = fma(s1, a45.y, r5);
    }
    if (I != J) {
#pragma unroll
      for (int t = 0; t < T / NQ; t += 2) {
        const int r = j0 + t;
        const double u0 = st[r + i * LD], u1 = st[r + 1 + i * LD];
        const double2 b01 = *reinterpret_cast<const double2*>(gI + 3 * r);
        const double2 b23 = *reinterpret_cast<const double2*>(gI + 3 * r + 2);
        const double2 b45 = *reinterpret_cast<const double2*>(gI + 3 * r + 4);
        c0 = fma(u0, b01.x, c0);
        c1 = fma(u0, b01.y, c1);
        c2 = fma(u0, b23.x, c2);
        c3 = fma(u1, b23.y, c3);
        c4 = fma(u1, b45.x, c4);
        c5 = fma(u1, b45.y, c5);
      }
    }
    r0 += r3;
    r1 += r4;
    r2 += r5;
    c0 += c3;
    c1 += c4;
    c2 += c5;
  }
  __syncthreads();  // the tile is consumed: its buffer holds the partial products now
  red[(0 * NQ + q) * T * 3 + 3 * i + 0] = r0;
  red[(0 * NQ + q) * T * 3 + 3 * i + 1] = r1;
  red[(0 * NQ + q) * T * 3 + 3 * i + 2] = r2;
  red[(1 * NQ + q) * T * 3 + 3 * i + 0] = c0;
  red[(1 * NQ + q) * T * 3 + 3 * i + 1] = c1;
  red[(1 * NQ + q) * T * 3 + 3 * i + 2] = c2;
  __syncthreads();
  double* pb = F.tpart + (size_t)b * nt * nt * T * 3;
  for (int e = threadIdx.x; e < T * 3; e += blockDim.x) {
    double v = red[e];
#pragma unroll
    for (int qq = 1; qq < NQ; ++qq) v += red[qq * T * 3 + e];
    __stcg(pb + ((size_t)I * nt + J) * T * 3 + e, v);  // block I, slot J
    if (I != J) {
      double w = red[NQ * T * 3 + e];
#pragma unroll
      for (int qq = 1; qq < NQ; ++qq) w += red[(NQ + qq) * T * 3 + e];
      __stcg(pb + ((size_t)J * nt + I) * T * 3 + e, w);  // block J, slot I
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* cnt = F.tcnt + (size_t)b * nt;
    s_last[0] = atomicAdd(cnt + I, 1u) == (unsigned)nt - 1 ? I : -1;
    s_last[1] = (I != J && atomicAdd(cnt + J, 1u) == (unsigned)nt - 1) ? J : -1;
  }
  __syncthreads();
  for (int w = 0; w < 2; ++w) {
    const int B = s_last[w];
    if (B < 0) continue;
    __threadfence();
    const double* pr = pb + (size_t)B * nt * T * 3;
    for (int e = threadIdx.x; e < T * 3; e += blockDim.x) {
      double v = 0.0;
      int S = 0;
      for (; S + 16 <= nt; S += 16) {  // 16 independent loads in flight, summed in slot order
        double l[16];
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) l[qq] = __ldcg(pr + (size_t)(S + qq) * T * 3 + e);
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) v += l[qq];
      }
      for (; S < nt; ++S) v += __ldcg(pr + (size_t)S * T * 3 + e);
      gI[e] = v;
    }
    __syncthreads();
    if (threadIdx.x < T && B * T + (int)threadIdx.x < K) {
      const int k = B * T + threadIdx.x;
      const double v[3] = {gI[3 * threadIdx.x + 0], gI[3 * threadIdx.x + 1], gI[3 * threadIdx.x + 2]};
      const int row = F.tcols[k];
      double* xo = F.x + ((size_t)b * F.n + row) * 3;
      __stcg(xo + 0, v[0]);
      __stcg(xo + 1, v[1]);
      __stcg(xo + 2, v[2]);
      io.store(b, row, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      F.tcnt[(size_t)b * nt + B] = 0;  // every partial of B has arrived: reset for the next solve
      if (after_forward) {
        __threadfence();
        atomicAdd(F.stage_cnt + 1, 1u);  // row block B of x_T is complete
      }
    }
    __syncthreads();
  }
}

template <class IO>
__global__ void __launch_bounds__(kSolveThreads, 6) sptrsv_top_sym(FactorView F, IO io) {
  pdl_entry();
  __shared__ __align__(16) double st[kTopTileEntries];
  __shared__ __align__(16) double gI[kTopTile * 3], gJ[kTopTile * 3];
  __shared__ int s_last[2];
  __shared__ uint64_t s_mbar;
  const int b = blockIdx.y;
  if (!io.active(b)) return;
  mbar_init(&s_mbar);
  if (threadIdx.x == 0 && blockIdx.x == 0) solve_tl(F, 6, 0);
  unsigned phase = 0;
  top_tile(F, io, (int)blockIdx.x, b, st, gI, gJ, s_last, &s_mbar, phase, false);
  if (threadIdx.x == 0 && (s_last[0] >= 0 || s_last[1] >= 0)) solve_tl_max(F, 6, 1);
}

// Forward, dense-top tiles and backward in ONE persistent kernel: forward
// tickets, then one ticket per S^-1 tile, then backward tickets, so idle CTAs
// stage backward tiles while the forward tail runs, and the top's S^-1 tiles
// stream in while the forward sweep finishes (a tile task issues its bulk copy
// before waiting for the last forward task).  Every dependency has a smaller
// ticket (a backward task waits for its own supernode's forward tasks, its
// parent's backward tasks, and — below the dense top — for every row block
// of x_T), so the waits cannot deadlock.
template <class IO>
__global__ void __launch_bounds__(kSolveThreads, 2) sptrsv_fused(FactorView F, IO io) {
  pdl_entry();
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_item[2];
  __shared__ unsigned s_epoch;
  __shared__ uint64_t s_mbar;
  __shared__ int s_last[2];
  unsigned phase = 0;
  mbar_init(&s_mbar);
  unsigned* sched = F.sched;
  if (threadIdx.x == 0) s_epoch = *((volatile unsigned*)&sched[2]);
  if (threadIdx.x == 0 && blockIdx.x == 0) solve_tl(F, 4, 0);
  const int nfi = F.nftask * F.nbatch;
  const int ntt = F.fuse_top ? F.tnt * (F.tnt + 1) / 2 : 0;  // top tiles (single instance)
  const int total = nfi + ntt + F.nbtask * F.nbatch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ DescSlot s_desc[2];
  auto run = [&](auto tiled) {
    constexpr bool kT = decltype(tiled)::value;
    ticket_loop<kT>(
        F, sched, s_item, nfi, ntt, total, s_desc, s_epoch, F.lookahead != 0,
        [&](int cur, const unsigned char* dsc, const TileAhead& ahead, const NextTicket& nt) {
          if (cur < nfi)
            return fwd_task<kT>(F, io, cur, s_epoch, sm, lane, warp, &s_mbar, phase,
                                reinterpret_cast<const qn_fdesc*>(dsc), ahead, nt, nfi, ntt, total);
          if (cur < nfi + ntt) {
            if (io.active(0))  // same predicate as the forward tasks that the tile waits for
              top_tile(F, io, cur - nfi, 0, sm, sm + kTopTileEntries, sm + kTopTileEntries + 3 * kTopTile, s_last,
                       &s_mbar, phase, true);
            return no_task();
          }
          return bwd_task<kT>(F, io, cur - nfi - ntt, s_epoch, sm, lane, warp, true, &s_mbar, phase,
                              reinterpret_cast<const qn_bdesc*>(dsc), ahead, nt, nfi, ntt, total);
        });
  };
  if (F.tiled)
    run(std::true_type{});
  else
    run(std::false_type{});
  cta_exit(sched, s_epoch, F, 5);
}

// ---- batched small systems (configs[3]): one CTA per instance walks its whole
// tree level by level — forward by height (leaves first), backward by depth
// (root first) — with the independent supernodes of a level on different
// warps and one CTA barrier per level, so the sequential chain is the tree
// height, not the supernode count.  No inter-CTA flags: thousands of
// instances run as thousands of independent CTAs.  The right-hand side of
// every row is staged once; y/x of the instance live in shared memory (x
// overwrites y in place during the backward sweep); each warp keeps its
// supernode's f / y_J in a private shared-memory slice; the update vectors
// stay in the instance's global (L2) slice.
constexpr int kBatchThreads = 128, kBatchWarps = kBatchThreads / 32;
constexpr int kBatchCols = 4;  // backward: columns per pass (12 independent chains per lane)

template <class IO>
__global__ void __launch_bounds__(kBatchThreads, 8) sptrsv_batch(FactorView F, IO io) {
  pdl_entry();
  extern __shared__ double sm[];  // yx[n*3] | fw[kBatchWarps][max_nc*3]
  const int b = blockIdx.x;
  if (!io.active(b)) return;
  const int n = F.n;
  double* yx = sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* fw = sm + 3 * n + (size_t)warp * 3 * F.batch_max_nc;
  double* ub = F.u + (size_t)b * F.nupd * 3;
  const double* vb = F.vals + (size_t)b * F.nvals;
  for (int p = tid; p < n; p += blockDim.x) {  // b for every row (independent loads)
    double v[3];
    io.rhs(b, p, v);
    yx[3 * p + 0] = v[0];
    yx[3 * p + 1] = v[1];
    yx[3 * p + 2] = v[2];
  }
  __syncthreads();
  // ---- forward: y = L^-1 b, one level of independent supernodes at a time ----
  for (int L = 0; L < F.nhlev; ++L) {
    for (int i = F.hlev_ptr[L] + warp; i < F.hlev_ptr[L + 1]; i += kBatchWarps) {
      const int s = F.hlev_sup[i];
      const int c0 = F.sup_col[s], nc = F.sup_col[s + 1] - c0;
      const int64_t R0 = F.sup_row_ptr[s];
      const int nr = (int)(F.sup_row_ptr[s + 1] - R0);
      const double* Z = vb + F.sup_val_ptr[s];
      for (int p = lane; p < nc; p += 32) {  // f = b_J - children updates
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        gather_rows<1>(ub, F.cidx, F.cptr[R0 + p], F.cptr[R0 + p + 1], a0, a1, a2);
        fw[3 * p + 0] = yx[3 * (c0 + p) + 0] - a0;
        fw[3 * p + 1] = yx[3 * (c0 + p) + 1] - a1;
        fw[3 * p + 2] = yx[3 * (c0 + p) + 2] - a2;
      }
      __syncwarp();
      for (int r = lane; r < nr; r += 32) {  // v = Z f (lanes over rows: coalesced Z)
        const int kmax = r < nc ? r + 1 : nc;
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
        if (r >= nc)  // children's updates on this bottom row (independent of the FMAs)
          gather_rows<1>(ub, F.cidx, F.cptr[R0 + r], F.cptr[R0 + r + 1], e0, e1, e2);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        int k = 0;
        for (; k + 8 <= kmax; k += 8) {
          double l[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) l[q] = __ldg(Z + r + (int64_t)(k + q) * nr);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            a0 = fma(l[q], fw[3 * (k + q) + 0], a0);
            a1 = fma(l[q], fw[3 * (k + q) + 1], a1);
            a2 = fma(l[q], fw[3 * (k + q) + 2], a2);
          }
        }
        for (; k < kmax; ++k) {
          const double l = __ldg(Z + r + (int64_t)k * nr);
          a0 = fma(l, fw[3 * k + 0], a0);
          a1 = fma(l, fw[3 * k + 1], a1);
          a2 = fma(l, fw[3 * k + 2], a2);
        }
        if (r < nc) {
          yx[3 * (c0 + r) + 0] = a0;
          yx[3 * (c0 + r) + 1] = a1;
          yx[3 * (c0 + r) + 2] = a2;
        } else {
          double* us = ub + (F.sup_upd_ptr[s] + (r - nc)) * 3;
          __stcg(us + 0, e0 + a0);
          __stcg(us + 1, e1 + a1);
          __stcg(us + 2, e2 + a2);
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  // ---- backward: x = L^-T y (in place over y), root level first ----
  for (int L = 0; L < F.ndlev; ++L) {
    for (int i = F.dlev_ptr[L] + warp; i < F.dlev_ptr[L + 1]; i += kBatchWarps) {
      const int s = F.dlev_sup[i];
      const int c0 = F.sup_col[s], nc = F.sup_col[s + 1] - c0;
      const int64_t R0 = F.sup_row_ptr[s];
      const int nr = (int)(F.sup_row_ptr[s + 1] - R0);
      const double* Z = vb + F.sup_val_ptr[s];
      for (int p = lane; p < 3 * nc; p += 32) fw[p] = yx[3 * c0 + p];  // y_J (x_J overwrites it)
      __syncwarp();
      for (int k0 = 0; k0 < nc; k0 += kBatchCols) {  // kBatchCols columns per pass, lanes over rows
        const int nv = min(kBatchCols, nc - k0);
        double a[kBatchCols][3];
#pragma unroll
        for (int j = 0; j < kBatchCols; ++j) a[j][0] = a[j][1] = a[j][2] = 0.0;
        for (int r = k0 + lane; r < nr; r += 32) {
          double w0, w1, w2;
          if (r < nc) {
            w0 = fw[3 * r + 0];
            w1 = fw[3 * r + 1];
            w2 = fw[3 * r + 2];
          } else {
            const int row = F.sup_rows[R0 + r];
            w0 = -yx[3 * row + 0];
            w1 = -yx[3 * row + 1];
            w2 = -yx[3 * row + 2];
          }
          double l[kBatchCols];
#pragma unroll
          for (int j = 0; j < kBatchCols; ++j)
            l[j] = (j < nv && r >= k0 + j) ? __ldg(Z + r + (int64_t)(k0 + j) * nr) : 0.0;
#pragma unroll
          for (int j = 0; j < kBatchCols; ++j) {
            a[j][0] = fma(l[j], w0, a[j][0]);
            a[j][1] = fma(l[j], w1, a[j][1]);
            a[j][2] = fma(l[j], w2, a[j][2]);
          }
        }
#pragma unroll
        for (int j = 0; j < kBatchCols; ++j) {
          const double v0 = warp_sum(a[j][0]), v1 = warp_sum(a[j][1]), v2 = warp_sum(a[j][2]);
          if (lane == j && j < nv) {
            yx[3 * (c0 + k0 + j) + 0] = v0;
            yx[3 * (c0 + k0 + j) + 1] = v1;
            yx[3 * (c0 + k0 + j) + 2] = v2;
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  for (int p = tid; p < n; p += blockDim.x) {  // x -> caller
    const double v[3] = {yx[3 * p + 0], yx[3 * p + 1], yx[3 * p + 2]};
    io.store(b, p, v);
  }
}

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
  __device__ double* dest(int, int row) const { return X + 3 * (size_t)perm[row]; }
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
  if (f->batch_smem > 0) {  // batched small systems: one CTA per instance
    cudaError_t e = launch_k(sptrsv_batch<IO>, dim3((unsigned)f->nbatch), dim3(kBatchThreads), (size_t)f->batch_smem, stream,
                             f->pdl != 0, v, io);
    (void)e;
    QN_CHECK_LAUNCH();
    return QN_OK;
  }
  const int nf = (int)f->ftask.size() * (int)f->nbatch, nb = (int)f->btask.size() * (int)f->nbatch;
  if (f->fused && (f->ktop == 0 || v.fuse_top)) {
    const int ntt = v.fuse_top ? f->tnt * (f->tnt + 1) / 2 : 0;
    if (nf + nb + ntt > 0) {
      cudaError_t e = launch_k(sptrsv_fused<IO>, dim3((unsigned)std::min(nf + nb + ntt, f->grid_fused)), dim3(kSolveThreads),
                               (size_t)f->smem_fused, stream, f->pdl != 0, v, io);
      (void)e;
      QN_CHECK_LAUNCH();
    }
    return QN_OK;
  }
  if (nf > 0) {
    cudaError_t e = launch_k(sptrsv_forward<IO>, dim3((unsigned)std::min(nf, f->grid_f)), dim3(kSolveThreads),
                             (size_t)f->smem_f, stream, f->pdl != 0, v, io);
    (void)e;
    QN_CHECK_LAUNCH();
  }
  if (f->ktop > 0) {
    const dim3 ga((unsigned)(f->tnt * (f->tnt + 1) / 2), (unsigned)f->nbatch);
    cudaError_t e = launch_k(sptrsv_top_sym<IO>, ga, dim3(kSolveThreads), (size_t)0, stream, f->pdl != 0, v, io);
    (void)e;
    QN_CHECK_LAUNCH();
  }
  if (nb > 0) {
    cudaError_t e = launch_k(sptrsv_backward<IO>, dim3((unsigned)std::min(nb, f->grid_b)), dim3(kSolveThreads),
                             (size_t)f->smem_b, stream, f->pdl != 0, v, io);
    (void)e;
    QN_CHECK_LAUNCH();
  }
  return QN_OK;
}

template <class IO>
int prepare_solve_kernels(qn_factor* f) {
  QN_CUDA(cudaFuncSetAttribute(sptrsv_forward<IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, f->smem_f));
  QN_CUDA(cudaFuncSetAttribute(sptrsv_backward<IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, f->smem_b));
  QN_CUDA(cudaFuncSetAttribute(sptrsv_forward<IO>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  QN_CUDA(cudaFuncSetAttribute(sptrsv_backward<IO>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  if (f->batch_smem > 0)
    QN_CUDA(cudaFuncSetAttribute(sptrsv_batch<IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, f->batch_smem));
  int per_f = 0, per_b = 0, dev = 0, sms = 0;
  QN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_f, sptrsv_forward<IO>, kSolveThreads, f->smem_f));
  QN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_b, sptrsv_backward<IO>, kSolveThreads, f->smem_b));
  QN_CUDA(cudaGetDevice(&dev));
  QN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int gf = std::max(1, per_f) * sms, gb = std::max(1, per_b) * sms;
  if (f->fused) {
    QN_CUDA(cudaFuncSetAttribute(sptrsv_fused<IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, f->smem_fused));
    QN_CUDA(cudaFuncSetAttribute(sptrsv_fused<IO>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_x = 0;
    QN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_x, sptrsv_fused<IO>, kSolveThreads, f->smem_fused));
    const int gx = std::max(1, per_x) * sms;
    f->grid_fused = f->grid_fused ? std::min(f->grid_fused, gx) : gx;
  }
  f->grid_f = f->grid_f ? std::min(f->grid_f, gf) : gf;
  f->grid_b = f->grid_b ? std::min(f->grid_b, gb) : gb;
  // descriptor lookahead pays off when CTAs run many tasks each (c3: 27, c2: 5 per CTA)
  const int64_t tasks = (int64_t)(f->ftask.size() + f->btask.size()) * f->nbatch;
  f->many_tasks = tasks >= 12 * (int64_t)std::max(f->grid_f, 1) ? 1 : 0;
  // Ticket lookahead (a CTA holds its next ticket for a whole task) measured slower than taking the
  // next ticket during the task (NextTicket) once the staging round trips were overlapped: c3 solve
  // 223 vs 207 us.  QN_SOLVE_OPTS bit 1 turns it back on for experiments.
  f->lookahead = (f->many_tasks && (f->solve_opts & 2)) ? 1 : 0;
  return QN_OK;
}

}  // namespace qn

// Device building blocks shared by the single-system frame (qn_solver.cu) and
// the slab-decomposed frame (qn_slab.cu): deterministic last-block
// reductions and the per-tet pass (F = Ds Dm^-1, SVD, VL energy, PK1 corner
// forces) of dynamics.VLGroup.energy / add_gradient (dynamics.py:54-67).
#pragma once

#include "qn_common.cuh"
#include "qn_element.cuh"
#include "qn_element_f32.cuh"
#include "qn_system.h"

namespace qn {

constexpr int kTT = kTetThreads;  // tet-kernel block
constexpr int kTetBlocksPerSm = 7;  // <= 72 registers (swept: 6 -> 7 +6 % on c3 tet, 8 (64 regs, 268 B spills) slower)

// last block of instance b for counter `which`?  (after all partial writes)
// Partials are written by thread 0 before this call; one fence by that thread
// (after the barrier) orders them before the counter increment.  The last
// block reads the partials with L2 loads (__ldcg).
__device__ __forceinline__ bool last_block(unsigned* cnt, int which, int b, int n_inst, int nblk) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned* c = cnt + (size_t)which * n_inst + b;
    const unsigned old = atomicAdd(c, 1u);
    s_last = (old == (unsigned)nblk - 1);
    if (s_last) {
      *c = 0;
      __threadfence();
    }
  }
  __syncthreads();
  return s_last;
}

// Deterministic block-parallel sum of per-block partials (run by every thread of
// the finalising block): out[k] = sum_blk part[blk * stride + k], k < nval
// (nval <= stride <= kNG).  Blocks are processed in chunks: the chunk's
// partial rows (contiguous) are copied to shared memory with every thread
// issuing independent loads, then lane l of the warp owning value k adds the
// chunk's blocks l, l+32, ... into its running sum; a fixed butterfly
// finishes.  Fixed order throughout, so the result is reproducible.
__device__ __forceinline__ void sum_partials(const double* part, int nblk, int stride, int nval, double* out) {
  // thread t < G*nval owns value k = t % nval and blocks t/nval, t/nval + G, ...
  // (8 independent loads in flight per thread); the G per-thread sums of a
  // value are then combined by thread k in index order.
  __shared__ double sums[256];
  const int G = min((int)blockDim.x, 256) / nval;
  const int t = threadIdx.x;
  if (t < G * nval) {
    const int k = t % nval, j0 = t / nval;
    double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int blk = j0;
    for (; blk + 7 * G < nblk; blk += 8 * G) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += __ldcg(part + (size_t)(blk + u * G) * stride + k);
    }
    for (; blk < nblk; blk += G) a[0] += __ldcg(part + (size_t)blk * stride + k);
    sums[t] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  }
  __syncthreads();
  if (t < nval) {
    double s = 0.0;
    for (int j = 0; j < G; ++j) s += sums[j * nval + t];
    out[t] = s;
  }
  __syncthreads();
}

constexpr int kMatSmem = 4;  // materials per instance staged in shared memory

// Material table of instance b: staged in shared memory (block-cooperative
// copy) when kSm (n_mat <= kMatSmem, chosen on the host), else read from
// global memory.  The compile-time choice keeps shared-memory accesses LDS.
template <bool kSm>
__device__ __forceinline__ const qn_material* stage_materials(const SysView& v, int b, qn_material* smat) {
  const qn_material* src = v.mats + (size_t)b * v.n_mat;
  if (!kSm) return src;
  const int words = v.n_mat * (int)(sizeof(qn_material) / 8);
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(smat);
  for (int w = threadIdx.x; w < words; w += blockDim.x) d[w] = __ldg(s + w);
  __syncthreads();
  return smat;
}

constexpr int kFStride = 13;  // padded per-thread stride of the staged corner forces

// Energy and corner forces of tet t (all lanes execute: lanes past the end
// evaluate a clamped tet and do not store, keeping the SVD's warp votes
// convergent).  Tets not in `mat_sel` (>= 0) contribute zero.  The 12 forces
// are staged in shared memory and written block-contiguously (coalesced) by
// store_forces().
// Edge spring (a, b) of a spring network (SpringGroup, dynamics.py:111-151):
// energy w/2 (|d| - r)^2 and forces -+ w (1 - r/|d|) d, w = k (material a.c[0]),
// r = vols[t]; corners 2, 3 of the element stay zero.
__device__ __forceinline__ double spring_thread(const SysView& v, const double* __restrict__ x, int t, int t_raw, int4 tv,
                                             const qn_material* mats, int mat_sel, double* fsm) {
  const int mi = v.tet_mat ? __ldg(v.tet_mat + t) : 0;
  const double w = mats[mi].a.c[0];
  const double r = __ldg(v.vols + t);
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = x[3 * tv.y + a] - x[3 * tv.x + a];
  const double len = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
  const double e = 0.5 * w * ((len - r) * (len - r));
  const double s = w * (1.0 - r / fmax(len, 1e-300));
  const bool sel = mat_sel < 0 || mi == mat_sel;
  double* fs = fsm + threadIdx.x * kFStride;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double rs = s * d[a];
    fs[a] = sel ? -rs : 0.0;
    fs[3 + a] = sel ? rs : 0.0;
    fs[6 + a] = 0.0;
    fs[9 + a] = 0.0;
  }
  return t_raw < v.mt && sel ? e : 0.0;
}

// kAniso: the system has anisotropic-fibre elements (a separate instantiation,
// so the plain per-tet kernel keeps its register allocation)
template <bool kAniso = false, bool kF32 = false>
__device__ __forceinline__ double tet_thread(const SysView& v, const double* __restrict__ x, int b, int t_raw,
                                             const qn_material* mats, int mat_sel, double* fsm) {
  const int t = min(t_raw, v.mt - 1);
  const int4 tv = __ldg(v.tets + t);
  if (v.spring) return spring_thread(v, x, t, t_raw, tv, mats, mat_sel, fsm);
  const int id[4] = {tv.x, tv.y, tv.z, tv.w};
  double xs[4][3];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    xs[k][0] = x[3 * id[k] + 0];
    xs[k][1] = x[3 * id[k] + 1];
    xs[k][2] = x[3 * id[k] + 2];
  }
  double Dm[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) Dm[r][q] = __ldg(v.dminv + (size_t)(r * 3 + q) * v.mt + t);
  const double vol = __ldg(v.vols + t);
  const int mi = v.tet_mat ? __ldg(v.tet_mat + t) : 0;
  double f[4][3];
  // every lane runs the SVD path (its sweeps end on warp votes, so a warp
  // holding both element kinds must not diverge there); fibre elements then
  // replace the result (their VL material evaluates to zero)
  double e;
  if (kF32) {  // the optional fp32 element pass (fp64 storage and gather)
    e = tet_eval_f32(mats[mi], xs, Dm, vol, f);
  } else {
    e = tet_eval<true>(mats[mi], xs, Dm, vol, f);
    if (kAniso && mats[mi].a.kind == QN_FN_ANISO) e = aniso_eval(mats[mi], xs, Dm, vol, f);
  }
  const bool keep = t_raw < v.mt;
  const bool sel = mat_sel < 0 || mi == mat_sel;
  double* fs = fsm + threadIdx.x * kFStride;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a) fs[3 * k + a] = sel ? f[k][a] : 0.0;
  return keep && sel ? e : 0.0;
}

// corner forces of this thread's element to their gather positions: slot
// 4t + c goes to entry slot_pos[4t + c] of the vertex-major gather order
// (v2e), so the gradient gather streams each vertex's contiguous run of
// entries instead of chasing slot ids (same values, same order)
__device__ __forceinline__ void store_forces(const SysView& v, int b, const double* fsm) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= v.mt) return;
  const double* fs = fsm + threadIdx.x * kFStride;
  double* base = v.forces + (size_t)b * v.mt * 12;
  const int4 pos = __ldg(reinterpret_cast<const int4*>(v.slot_pos) + t);
  const int p[4] = {pos.x, pos.y, pos.z, pos.w};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (p[c] < 0) continue;
    double* o = base + 3 * (size_t)p[c];
    o[0] = fs[3 * c + 0];
    o[1] = fs[3 * c + 1];
    o[2] = fs[3 * c + 2];
  }
}

}  // namespace qn

// extern "C" boundary of libqnsim_b200 (declared in include/qnsim_b200.h).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cusolverDn.h>

#include "qn_common.cuh"
#include "qn_factor.h"
#include "qn_sptrsv.cuh"
#include "qn_amg.h"
#include "qn_system.h"

namespace qn {

namespace {
thread_local std::string g_err;
thread_local int g_capturing = 0;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }
void count_launch(int n) {
  if (!g_capturing) g_launches += n;
}
CaptureScope::CaptureScope() { ++g_capturing; }
CaptureScope::~CaptureScope() { --g_capturing; }

// defined in qn_solver.cu
int launch_body(qn_system* S, cudaStream_t st);
int launch_init(qn_system* S, cudaStream_t st);
int launch_finish(qn_system* S, cudaStream_t st);
int build_graph(qn_system* S);
int prepare_kernels(qn_system* S);
int launch_tet_plain(qn_system* S, const double* x, int b, int mat_sel, double* part, cudaStream_t st);
int launch_solve_timing(qn_system* S, cudaStream_t st);
int launch_vcycle(qn_system* S, cudaStream_t st);
int launch_spmv_timing(qn_system* S, cudaStream_t st);
__global__ void k_gather_plain(SysView v, const double* x, const double* y, double* out, int b, int inertia,
                               int zero_fixed, double* part);
__global__ void k_svd(int64_t m, const double* F, double* U, double* s, double* V);
__global__ void k_material(const qn_material* M, int64_t k, const double* sig, double* psi, double* tau);

namespace {

template <class T>
int dev_alloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return QN_ERR_ALLOC;
  }
  e = cudaMemset(*p, 0, count * sizeof(T));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMemset: ") + cudaGetErrorString(e));
    return QN_ERR_CUDA;
  }
  return QN_OK;
}

template <class T>
int dev_upload(T** p, const T* h, size_t count) {
  int rc = dev_alloc(p, count);
  if (rc) return rc;
  if (count) QN_CUDA(cudaMemcpy(*p, h, count * sizeof(T), cudaMemcpyHostToDevice));
  return QN_OK;
}

template <class T>
int sys_alloc(qn_system* S, T** p, size_t count) {
  int rc = dev_alloc(p, count);
  if (rc == QN_OK) S->allocs.push_back((void*)*p);
  return rc;
}

template <class T>
int sys_upload(qn_system* S, T** p, const T* h, size_t count) {
  int rc = dev_upload(p, h, count);
  if (rc == QN_OK) S->allocs.push_back((void*)*p);
  return rc;
}

cudaStream_t pick(qn_system* S, void* stream) { return stream ? (cudaStream_t)stream : S->stream; }

// Dense inverse of the AMG hierarchy's coarsest operator (SPD, a few thousand
// rows) on the device: cuSOLVER Cholesky, then potrs against the identity
// (library factorisation of a setup-time dense block; seconds on the host).
// The result is symmetric, so its column-major layout is the row-major one the
// coarse kernel reads.
int coarse_inverse_device(qn_system* S, const qn::Csr& A, float** out) {
  const int64_t nc = A.n;
  std::vector<double> M((size_t)nc * nc, 0.0);
  for (int64_t i = 0; i < nc; ++i)
    for (int64_t e = A.ptr[i]; e < A.ptr[i + 1]; ++e) M[(size_t)A.col[e] * nc + i] = A.val[e];
  double *dM = nullptr, *dI = nullptr, *work = nullptr;
  int* info = nullptr;
  int rc = QN_OK;
  if ((rc = dev_upload(&dM, M.data(), M.size()))) return rc;
  std::fill(M.begin(), M.end(), 0.0);
  for (int64_t i = 0; i < nc; ++i) M[(size_t)i * nc + i] = 1.0;
  if ((rc = sys_upload(S, &dI, M.data(), M.size()))) {
    cudaFree(dM);
    return rc;
  }
  cusolverDnHandle_t h = nullptr;
  int lwork = 0, hinfo = 0;
  bool ok = cusolverDnCreate(&h) == CUSOLVER_STATUS_SUCCESS &&
            cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)nc, dM, (int)nc, &lwork) ==
                CUSOLVER_STATUS_SUCCESS &&
            cudaMalloc((void**)&work, sizeof(double) * std::max(lwork, 1)) == cudaSuccess &&
            cudaMalloc((void**)&info, sizeof(int)) == cudaSuccess &&
            cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)nc, dM, (int)nc, work, lwork, info) ==
                CUSOLVER_STATUS_SUCCESS &&
            cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && hinfo == 0 &&
            cusolverDnDpotrs(h, CUBLAS_FILL_MODE_LOWER, (int)nc, (int)nc, dM, (int)nc, dI, (int)nc, info) ==
                CUSOLVER_STATUS_SUCCESS &&
            cudaDeviceSynchronize() == cudaSuccess;
  if (h) cusolverDnDestroy(h);
  cudaFree(dM);
  cudaFree(work);
  cudaFree(info);
  if (!ok) {
    set_error(hinfo ? "amg: coarsest operator is not positive definite" : "amg: cuSOLVER coarse inverse failed");
    return hinfo ? QN_ERR_NOT_SPD : QN_ERR_CUDA;
  }
  // stored in fp32: the coarse solve is part of the preconditioner only (a fixed
  // operator; CG still solves the fp64 A_free to pcg_tol), and half the bytes
  // of the per-cycle dense product
  float* f32 = nullptr;
  if ((rc = sys_alloc(S, &f32, (size_t)nc * nc))) return rc;
  std::vector<double> hd((size_t)nc * nc);
  QN_CUDA(cudaMemcpy(hd.data(), dI, sizeof(double) * hd.size(), cudaMemcpyDeviceToHost));
  std::vector<float> hf(hd.begin(), hd.end());
  QN_CUDA(cudaMemcpy(f32, hf.data(), sizeof(float) * hf.size(), cudaMemcpyHostToDevice));
  *out = f32;
  return QN_OK;
}

// three n x 3 vectors for the seam entry points (objective / elements), owned
// by the system and freed with it
int ensure_scratch(qn_system* S) {
  if (S->scratch[0]) return QN_OK;
  const size_t nv = (size_t)S->n * 3;
  for (int i = 0; i < 3; ++i) {
    int rc = sys_alloc(S, &S->scratch[i], nv);
    if (rc) return rc;
  }
  return QN_OK;
}

// copy between a caller buffer (host or device) and a device buffer
int to_device(double* dst, const double* src, size_t count, int32_t mem, cudaStream_t st) {
  QN_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(double),
                          mem == QN_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  return QN_OK;
}
template <class T>
int from_device(T* dst, const T* src, size_t count, int32_t mem, cudaStream_t st) {
  QN_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T),
                          mem == QN_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  return QN_OK;
}

}  // namespace

int factor_upload(qn_factor* f) {
  int rc;
  if ((rc = dev_upload(&f->d_sup_col, f->sup_col.data(), f->sup_col.size()))) return rc;
  if ((rc = dev_upload(&f->d_sup_row_ptr, f->sup_row_ptr.data(), f->sup_row_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_sup_rows, f->sup_rows.data(), f->sup_rows.size()))) return rc;
  if ((rc = dev_upload(&f->d_sup_val_ptr, f->sup_val_ptr.data(), f->sup_val_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_sup_upd_ptr, f->sup_upd_ptr.data(), f->sup_upd_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_parent, f->parent.data(), f->parent.size()))) return rc;
  if ((rc = dev_upload(&f->d_child_ptr, f->child_ptr.data(), f->child_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_child_idx, f->child_idx.data(), f->child_idx.size()))) return rc;
  if ((rc = dev_upload(&f->d_rel_ptr, f->rel_ptr.data(), f->rel_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_rel, f->rel.data(), f->rel.size()))) return rc;
  if ((rc = dev_upload(&f->d_perm, f->perm.data(), f->perm.size()))) return rc;
  if ((rc = dev_upload(&f->d_vals, f->vals.data(), f->vals.size()))) return rc;
  if ((rc = dev_alloc(&f->d_y, (size_t)f->nbatch * f->n * 3))) return rc;
  if ((rc = dev_alloc(&f->d_x, (size_t)f->nbatch * f->n * 3))) return rc;
  if ((rc = dev_alloc(&f->d_u, (size_t)f->nbatch * std::max<int64_t>(f->nupd, 1) * 3))) return rc;
  if ((rc = dev_alloc(&f->d_flags, (size_t)f->nbatch * (f->ftask.size() + f->btask.size())))) return rc;
  if ((rc = dev_upload(&f->d_cptr, f->cptr.data(), f->cptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_cidx, f->cidx.data(), f->cidx.size()))) return rc;
  if ((rc = dev_upload(&f->d_ftask, f->ftask.data(), f->ftask.size()))) return rc;
  if ((rc = dev_upload(&f->d_btask, f->btask.data(), f->btask.size()))) return rc;
  if ((rc = dev_upload(&f->d_bfirst, f->bfirst.data(), f->bfirst.size()))) return rc;
  if ((rc = dev_upload(&f->d_bcount, f->bcount.data(), f->bcount.size()))) return rc;
  if ((rc = dev_upload(&f->d_fdep_ptr, f->fdep_ptr.data(), f->fdep_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_fdep_idx, f->fdep_idx.data(), f->fdep_idx.size()))) return rc;
  if ((rc = dev_upload(&f->d_hlev_ptr, f->hlev_ptr.data(), f->hlev_ptr.size()))) return rc;
  {
    // Task-tiled copies of Z for the persistent solve kernels: every forward /
    // backward task's tile is one contiguous, 16-byte aligned block laid out as
    // the task holds it in shared memory (forward: rows [lo, hi) x k < kmax,
    // column-major with leading dimension hi - lo; backward: columns [k0, k1)
    // x all nr rows, zeros above the diagonal), so one TMA bulk copy stages it.
    // Descriptors' zoff become tile offsets.  Batched mode (one CTA per
    // instance, sptrsv_batch) reads vals directly and needs no copies.
    int max_nc_all = 0;
    for (int s = 0; s < f->nsup; ++s) max_nc_all = std::max(max_nc_all, f->sup_col[s + 1] - f->sup_col[s]);
    const size_t bsm0 = sizeof(double) * 3 * ((size_t)f->n + (size_t)kBatchWarps * max_nc_all);
    const bool batch_mode = f->nbatch > 1 && bsm0 <= 110 * 1024;
    // a factor that fits in L2 next to the frame's vectors keeps one copy: the
    // backward sweep re-reads what the forward sweep pulled into L2 (c2: 30 MB)
    const bool small = (double)f->nbatch * f->nvals * sizeof(double) <= 48.0 * (1 << 20);
    std::vector<qn_fdesc> fd = f->fdesc;
    std::vector<qn_bdesc> bd = f->bdesc;
    if (!batch_mode && !small) {
      int64_t off = 0;
      for (auto& d : fd) {
        const int64_t cnt = (int64_t)(d.hi - d.lo) * std::min(d.hi, d.nc);
        d.zoff = off;
        off += (cnt + 1) / 2 * 2;
      }
      f->ftile_n = std::max<int64_t>(off, 2);
      off = 0;
      for (auto& d : bd) {
        const int64_t cnt = (int64_t)(d.k1 - d.k0) * d.nr;
        d.zoff = off;
        off += (cnt + 1) / 2 * 2;
      }
      f->btile_n = std::max<int64_t>(off, 2);
      std::vector<double> ft((size_t)f->nbatch * f->ftile_n, 0.0), bt((size_t)f->nbatch * f->btile_n, 0.0);
      for (int64_t b = 0; b < f->nbatch; ++b) {
        const double* vb = f->vals.data() + (size_t)b * f->nvals;
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = 0; i < (int64_t)fd.size(); ++i) {
          const qn_fdesc& h = f->fdesc[i];  // host descriptor: zoff = sup_val_ptr[s] + lo
          const int R = h.hi - h.lo, kmax = std::min(h.hi, h.nc);
          double* t = ft.data() + (size_t)b * f->ftile_n + fd[i].zoff;
          for (int k = 0; k < kmax; ++k)
            for (int r = 0; r < R; ++r) t[(size_t)k * R + r] = vb[h.zoff + (int64_t)k * h.nr + r];
        }
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = 0; i < (int64_t)bd.size(); ++i) {
          const qn_bdesc& h = f->bdesc[i];  // zoff = sup_val_ptr[s] + k0 nr
          double* t = bt.data() + (size_t)b * f->btile_n + bd[i].zoff;
          for (int kk = 0; kk < h.k1 - h.k0; ++kk)
            for (int r = 0; r < h.nr; ++r)
              t[(size_t)kk * h.nr + r] = r >= h.k0 + kk ? vb[h.zoff + (int64_t)kk * h.nr + r] : 0.0;
        }
      }
      if ((rc = dev_upload(&f->d_ftile, ft.data(), ft.size()))) return rc;
      if ((rc = dev_upload(&f->d_btile, bt.data(), bt.size()))) return rc;
    }
    if (!fd.empty() && (rc = dev_upload(&f->d_fdesc, fd.data(), fd.size()))) return rc;
    if (!bd.empty() && (rc = dev_upload(&f->d_bdesc, bd.data(), bd.size()))) return rc;
  }
  if (!f->fblob.empty() && (rc = dev_upload(&f->d_fblob, f->fblob.data(), f->fblob.size()))) return rc;
  if ((rc = dev_upload(&f->d_hlev_sup, f->hlev_sup.data(), f->hlev_sup.size()))) return rc;
  if ((rc = dev_upload(&f->d_dlev_ptr, f->dlev_ptr.data(), f->dlev_ptr.size()))) return rc;
  if ((rc = dev_upload(&f->d_dlev_sup, f->dlev_sup.data(), f->dlev_sup.size()))) return rc;
  if (f->ktop > 0) {
    {  // S^-1 is symmetric: only the tiles (I, J), I >= J, are stored (half the bytes of the dense K x K)
      const int64_t K = f->ktop, T = kTopTile, nt = (K + T - 1) / T;
      f->tnt = (int32_t)nt;
      const int64_t LD = T + 1;  // padded leading dimension (bank-conflict-free row and column products)
      std::vector<double> tiles((size_t)(nt * (nt + 1) / 2) * T * LD, 0.0);
      for (int64_t I = 0; I < nt; ++I)
        for (int64_t J = 0; J <= I; ++J) {
          double* t = tiles.data() + (size_t)(I * (I + 1) / 2 + J) * T * LD;
          for (int64_t j = 0; j < T && J * T + j < K; ++j)
            for (int64_t i = 0; i < T && I * T + i < K; ++i)
              t[i + j * LD] = f->sinv[(size_t)(I * T + i) + (size_t)(J * T + j) * K];
        }
      if ((rc = dev_upload(&f->d_stile, tiles.data(), tiles.size()))) return rc;
      if ((rc = dev_alloc(&f->d_tpart, (size_t)f->nbatch * nt * nt * T * 3))) return rc;
      std::vector<unsigned> zero((size_t)f->nbatch * nt, 0u);
      if ((rc = dev_upload(&f->d_tcnt, zero.data(), zero.size()))) return rc;
      const unsigned z2[2] = {0u, 0u};
      if ((rc = dev_upload(&f->d_stage_cnt, z2, 2))) return rc;
    }
    if ((rc = dev_upload(&f->d_tcols, f->tcols.data(), f->tcols.size()))) return rc;
    if ((rc = dev_upload(&f->d_tg_ptr, f->tg_ptr.data(), f->tg_ptr.size()))) return rc;
    if ((rc = dev_upload(&f->d_tg_idx, f->tg_idx.data(), f->tg_idx.size()))) return rc;
  }
  if (const char* e = std::getenv("QN_SOLVE_OPTS")) f->solve_opts = std::atoi(e);  // experiment knob
  const unsigned sched[8] = {0, 0, 1, 0, 0, 1, 0, 0};  // [ticket, exited, epoch] x 2, watchdog
  if ((rc = dev_upload(&f->d_sched, sched, 8))) return rc;
  if ((rc = dev_alloc(&f->d_io, (size_t)f->n * 6))) return rc;
  int max_nc = 0;
  for (int s = 0; s < f->nsup; ++s) max_nc = std::max(max_nc, f->sup_col[s + 1] - f->sup_col[s]);
  // forward: Z tile + f (nc x 3), sized per task (fwd_entries = the largest), + index staging, which the
  // partial sums (256 x 3) reuse after the gathers;
  // backward: Z tile + w (nr x 3) + pre (64 x 3) + destinations (64) + row staging
  static_assert(sizeof(int) * kStageIdx >= sizeof(double) * 3 * kSolveThreads, "partials reuse the index staging");
  f->smem_f = (int)(sizeof(double) * (size_t)f->fwd_entries + sizeof(int) * kStageIdx);
  f->smem_b = (int)(sizeof(double) * (f->bwd_entries + 3 * (size_t)f->task_max_rows + 4 * kBwdCols) + sizeof(int) * kStageIdx);
  QN_REQUIRE(std::max(f->smem_f, f->smem_b) <= 227 * 1024, QN_ERR_UNSUPPORTED,
             "factor: supernode front exceeds shared memory");
  // one persistent kernel for forward (+ dense top tiles) + backward on single systems
  f->fused = !(f->nbatch > 1);
  f->smem_fused = std::max({f->smem_f, f->smem_b,
                             f->ktop > 0 ? (int)(sizeof(double) * (kTopTileEntries + 6 * kTopTile)) : 0});
  // batches of small systems: one CTA per instance when y/x of an instance fits in shared memory
  int64_t zmax = 0;
  for (int s = 0; s < f->nsup; ++s)
    zmax = std::max<int64_t>(zmax, (int64_t)(f->sup_col[s + 1] - f->sup_col[s]) * (f->sup_row_ptr[s + 1] - f->sup_row_ptr[s]));
  f->batch_max_nc = max_nc;
  f->batch_zmax = (int32_t)((zmax + 1) / 2 * 2);  // keep the second buffer 16-byte aligned
  const size_t bsm = sizeof(double) * 3 * ((size_t)f->n + (size_t)kBatchWarps * max_nc);
  f->batch_smem = (f->nbatch > 1 && bsm <= 110 * 1024) ? (int)bsm : 0;
  if ((rc = prepare_solve_kernels<PlainIO>(f))) return rc;
  f->on_device = true;
  return QN_OK;
}

void factor_free_device(qn_factor* f) {
  void* ptrs[] = {f->d_sup_col, f->d_sup_row_ptr, f->d_sup_rows, f->d_sup_val_ptr, f->d_sup_upd_ptr,
                  f->d_parent,  f->d_child_ptr,   f->d_child_idx, f->d_rel_ptr,   f->d_rel,
                  f->d_perm,    f->d_vals,        f->d_y,         f->d_x,         f->d_u,
                  f->d_flags,   f->d_sched,       f->d_io,        f->d_cptr,      f->d_cidx,
                  f->d_ftask,   f->d_btask,       f->d_bfirst,    f->d_bcount,    f->d_fdep_ptr,
                  f->d_fdep_idx, f->d_stile,      f->d_tcols,     f->d_tg_ptr,    f->d_tg_idx,
                  f->d_hlev_ptr,    f->d_hlev_sup,  f->d_dlev_ptr,  f->d_dlev_sup,
                  f->d_fdesc,   f->d_fblob,       f->d_bdesc,     f->d_tpart,     f->d_tcnt,
                  f->d_ftile,   f->d_btile,       f->d_stage_cnt};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  f->on_device = false;
}

// after a synchronised solve: did any dependency wait time out? (sched[6])
int factor_check_watchdog(qn_factor* f) {
  unsigned w = 0;
  QN_CUDA(cudaMemcpy(&w, f->d_sched + 6, sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (w) {
    const unsigned z = 0;
    QN_CUDA(cudaMemcpy(f->d_sched + 6, &z, sizeof(unsigned), cudaMemcpyHostToDevice));
    set_error("supernodal solve: dependency wait timed out (scheduling bug)");
    return QN_ERR_CUDA;
  }
  return QN_OK;
}

int factor_solve_plain(qn_factor* f, int64_t batch, cudaStream_t stream) {
  PlainIO io{f->d_io, f->d_io + 3 * f->n, f->d_perm, (int)batch};
  return launch_solve(f, io, stream);
}

}  // namespace qn

using namespace qn;

extern "C" {

const char* qn_last_error(void) { return get_error(); }
int qn_version(void) { return 1; }

int qn_device_count(int32_t* count) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  cudaGetLastError();
  *count = c;
  return QN_OK;
}

int qn_launch_count(int64_t* count) {
  *count = g_launches.load();
  return QN_OK;
}

// ---------------------------------------------------------------------------
int qn_svd_rv_batch(int64_t m, const double* F, double* U, double* sigma, double* V, int32_t mem, void* stream) {
  QN_REQUIRE(m >= 0 && F && U && sigma && V, QN_ERR_ARG, "svd: bad arguments");
  if (m == 0) return QN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const double *dF = F;
  double *dU = U, *ds = sigma, *dV = V, *buf = nullptr;
  if (mem == QN_MEM_HOST) {
    int rc = dev_alloc(&buf, (size_t)m * 21);
    if (rc) return rc;
    dU = buf;
    dV = buf + 9 * m;
    ds = buf + 18 * m;
    double* tmpF = nullptr;
    rc = dev_upload(&tmpF, F, (size_t)m * 9);
    if (rc) return rc;
    dF = tmpF;
  }
  k_svd<<<div_up(m, 128), 128, 0, st>>>(m, dF, dU, ds, dV);
  QN_CHECK_LAUNCH();
  if (mem == QN_MEM_HOST) {
    QN_CUDA(cudaMemcpyAsync(U, dU, m * 9 * sizeof(double), cudaMemcpyDeviceToHost, st));
    QN_CUDA(cudaMemcpyAsync(V, dV, m * 9 * sizeof(double), cudaMemcpyDeviceToHost, st));
    QN_CUDA(cudaMemcpyAsync(sigma, ds, m * 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    QN_CUDA(cudaStreamSynchronize(st));
    cudaFree(buf);
    cudaFree((void*)dF);
  } else {
    QN_CUDA(cudaStreamSynchronize(st));
  }
  return QN_OK;
}

int qn_material_eval(const qn_material* mat, int64_t k, const double* sigma, double* psi, double* tau, int32_t mem,
                     void* stream) {
  QN_REQUIRE(mat && k >= 0 && sigma && psi && tau, QN_ERR_ARG, "material: bad arguments");
  if (k == 0) return QN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  qn_material* dM = nullptr;
  int rc = dev_upload(&dM, mat, 1);
  if (rc) return rc;
  const double* ds = sigma;
  double *dp = psi, *dt = tau, *buf = nullptr;
  if (mem == QN_MEM_HOST) {
    rc = dev_alloc(&buf, (size_t)k * 7);
    if (rc) return rc;
    QN_CUDA(cudaMemcpy(buf, sigma, k * 3 * sizeof(double), cudaMemcpyHostToDevice));
    ds = buf;
    dp = buf + 3 * k;
    dt = buf + 4 * k;
  }
  k_material<<<div_up(k, 128), 128, 0, st>>>(dM, k, ds, dp, dt);
  QN_CHECK_LAUNCH();
  if (mem == QN_MEM_HOST) {
    QN_CUDA(cudaMemcpyAsync(psi, dp, k * sizeof(double), cudaMemcpyDeviceToHost, st));
    QN_CUDA(cudaMemcpyAsync(tau, dt, k * 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  QN_CUDA(cudaStreamSynchronize(st));
  if (buf) cudaFree(buf);
  cudaFree(dM);
  return QN_OK;
}

// ---------------------------------------------------------------------------
int qn_factor_create(int64_t n, const int64_t* indptr, const int32_t* indices, const double* values, int64_t nbatch,
                     const double* coords, qn_factor** out) {
  QN_REQUIRE(out, QN_ERR_ARG, "factor: null output");
  *out = nullptr;
  qn_factor* f = new qn_factor();
  int rc = factor_build_host(f, n, indptr, indices, values, nbatch, coords);
  if (rc == QN_OK) rc = factor_upload(f);
  if (rc != QN_OK) {
    factor_free_device(f);
    delete f;
    return rc;
  }
  *out = f;
  return QN_OK;
}

int qn_factor_info_get(const qn_factor* f, qn_factor_info* info) {
  QN_REQUIRE(f && info, QN_ERR_ARG, "factor_info: null");
  info->n = f->n;
  info->nnz_a = f->nnz_a;
  info->nnz_l = f->nnz_l;
  info->n_supernodes = f->nsup;
  info->max_front = f->max_rows;
  info->tree_depth = f->depth;
  info->nbatch = f->nbatch;
  info->factor_seconds = f->factor_seconds;
  info->flops = f->flops;
  info->dense_top = f->ktop;
  int64_t sparse = 0;
  for (int s = 0; s < f->nsup; ++s) {
    if (!f->is_top.empty() && f->is_top[s]) continue;
    const int64_t nc = f->sup_col[s + 1] - f->sup_col[s], nr = f->sup_row_ptr[s + 1] - f->sup_row_ptr[s];
    sparse += nr * nc - nc * (nc - 1) / 2;  // L's lower trapezoid of the supernode
  }
  info->nnz_l_sparse = sparse;
  info->sinv_stored = f->ktop > 0 ? (int64_t)f->tnt * (f->tnt + 1) / 2 * kTopTile * (kTopTile + 1) : 0;
  return QN_OK;
}

int qn_factor_solve(qn_factor* f, int64_t batch, const double* B, double* X, int64_t nrhs, int32_t mem,
                    void* stream) {
  QN_REQUIRE(f && B && X && nrhs >= 1 && batch >= 0 && batch < f->nbatch, QN_ERR_ARG, "factor_solve: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = f->n;
  std::vector<double> hb, hx;
  if (mem == QN_MEM_HOST) {
    hb.assign((size_t)n * 3, 0.0);
    hx.resize((size_t)n * 3);
  }
  for (int64_t c0 = 0; c0 < nrhs; c0 += 3) {
    const int64_t nc = std::min<int64_t>(3, nrhs - c0);
    if (mem == QN_MEM_HOST) {
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < 3; ++k) hb[3 * i + k] = k < nc ? B[i * nrhs + c0 + k] : 0.0;
      QN_CUDA(cudaMemcpyAsync(f->d_io, hb.data(), n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    } else {
      QN_REQUIRE(nrhs == 3, QN_ERR_ARG, "factor_solve: device buffers must have 3 columns");
      QN_CUDA(cudaMemcpyAsync(f->d_io, B, n * 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    int rc = factor_solve_plain(f, batch, st);
    if (rc) return rc;
    if (mem == QN_MEM_HOST) {
      QN_CUDA(cudaMemcpyAsync(hx.data(), f->d_io + 3 * n, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
      QN_CUDA(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < nc; ++k) X[i * nrhs + c0 + k] = hx[3 * i + k];
    } else {
      QN_CUDA(cudaMemcpyAsync(X, f->d_io + 3 * n, n * 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
      QN_CUDA(cudaStreamSynchronize(st));
    }
    if ((rc = factor_check_watchdog(f))) return rc;
  }
  return QN_OK;
}

int qn_factor_task_counts(const qn_factor* f, int64_t* n_ftask, int64_t* n_btask) {
  QN_REQUIRE(f && n_ftask && n_btask, QN_ERR_ARG, "task_counts: null");
  *n_ftask = (int64_t)f->ftask.size();
  *n_btask = (int64_t)f->btask.size();
  return QN_OK;
}

int qn_system_solve_trace(qn_system* S, uint64_t* stamps, int32_t* tasks) {
  QN_REQUIRE(S && stamps && tasks, QN_ERR_ARG, "solve_trace: null");
  qn_factor* f = S->factor;
  QN_REQUIRE(f && f->d_trace, QN_ERR_ARG, "solve_trace: no factor or timeline not enabled");
  const size_t nf = f->ftask.size(), nb = f->btask.size(), items = (nf + nb) * (size_t)f->nbatch;
  QN_CUDA(cudaDeviceSynchronize());
  QN_CUDA(cudaMemcpy(stamps, f->d_trace, qn::kTraceSlots * items * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  std::memcpy(tasks, f->ftask.data(), nf * sizeof(int4));
  std::memcpy(tasks + 4 * nf, f->btask.data(), nb * sizeof(int4));
  return QN_OK;
}

int qn_factor_trace_solve(qn_factor* f, uint64_t* stamps, int32_t* tasks) {
  QN_REQUIRE(f && stamps && tasks, QN_ERR_ARG, "trace: null");
  const size_t nf = f->ftask.size(), nb = f->btask.size(), items = (nf + nb) * (size_t)f->nbatch;
  QN_REQUIRE(!f->d_trace, QN_ERR_ARG, "trace: a system timeline is active");
  int rc = dev_alloc(&f->d_trace, qn::kTraceSlots * items);
  if (rc) return rc;
  rc = factor_solve_plain(f, 0, 0);
  if (rc == QN_OK) {
    QN_CUDA(cudaDeviceSynchronize());
    QN_CUDA(cudaMemcpy(stamps, f->d_trace, qn::kTraceSlots * items * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  }
  cudaFree(f->d_trace);
  f->d_trace = nullptr;
  std::memcpy(tasks, f->ftask.data(), nf * sizeof(int4));
  std::memcpy(tasks + 4 * nf, f->btask.data(), nb * sizeof(int4));
  return rc;
}

int qn_factor_destroy(qn_factor* f) {
  if (!f) return QN_OK;
  factor_free_device(f);
  delete f;
  return QN_OK;
}

// ---------------------------------------------------------------------------
void sell_build(int64_t nrows, int64_t ncols, const int64_t* ptr, const int32_t* col, const double* val,
                int64_t ni, int64_t nnz, std::vector<int64_t>& sptr, std::vector<int32_t>& scol,
                std::vector<double>& sval);
static int sell_upload(qn_system* S, int64_t nrows, int64_t ncols, const int64_t* ptr, const int32_t* col,
                       const double* val, qn::SellDevF* out);

int qn_system_create(const qn_system_desc* d, qn_system** out) {
  QN_REQUIRE(d && out, QN_ERR_ARG, "system: null argument");
  *out = nullptr;
  QN_REQUIRE(d->n_verts > 0 && d->n_tets >= 0 && d->n_inst >= 1 && d->n_mat >= 1, QN_ERR_ARG, "system: bad sizes");
  QN_REQUIRE(d->element_kind == QN_ELEM_TET || d->element_kind == QN_ELEM_SPRING, QN_ERR_ARG, "system: element kind");
  QN_REQUIRE(d->n_tets == 0 || (d->tets && (d->Dm_inv || d->element_kind == QN_ELEM_SPRING) && d->vols && d->mats),
             QN_ERR_ARG, "system: missing tets");
  QN_REQUIRE(d->masses && d->a_indptr && d->a_indices && d->a_values, QN_ERR_ARG, "system: missing arrays");
  QN_REQUIRE(d->h > 0, QN_ERR_ARG, "system: h must be positive");
  QN_REQUIRE(d->n_colliders >= 0 && d->n_colliders <= QN_MAX_COLLIDERS && (d->n_colliders == 0 || d->colliders),
             QN_ERR_ARG, "system: colliders");
  for (int64_t k = 0; k < d->n_colliders; ++k)
    QN_REQUIRE(d->colliders[k].kind >= QN_COL_HALFSPACE && d->colliders[k].kind <= QN_COL_TORUS, QN_ERR_ARG,
               "system: unknown collider kind");
  const int64_t n = d->n_verts, mt = d->n_tets, ni = d->n_inst;
  QN_REQUIRE(n * ni < (int64_t)1 << 31 && mt * 4 < (int64_t)1 << 31, QN_ERR_ARG, "system: too large");
  const bool verbose = std::getenv("QN_BUILD_VERBOSE") != nullptr;  // diagnostics: per-phase host times
  auto tp = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!verbose) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "system_create %-16s %8.3f s\n", what, std::chrono::duration<double>(t - tp).count());
    tp = t;
  };
  qn_system* S = new qn_system();
  S->n = n;
  S->mt = mt;
  S->n_inst = ni;
  S->n_mat = d->n_mat;
  S->n_fixed = d->n_fixed;
  S->h = d->h;
  for (int a = 0; a < 3; ++a) S->grav[a] = d->gravity[a];
  S->scale = d->scale;
  S->max_mass = 0;
  for (int64_t i = 0; i < n; ++i) S->max_mass = std::max(S->max_mass, d->masses[i]);
  auto fail = [&](int rc) {
    qn_system_destroy(S);
    return rc;
  };
  // fixed set
  std::vector<uint8_t> is_fixed(n, 0);
  std::vector<int32_t> fixed_pos(n, -1);
  for (int64_t k = 0; k < d->n_fixed; ++k) {
    const int32_t v = d->fixed[k];
    if (v < 0 || v >= n || (k > 0 && d->fixed[k - 1] >= v)) {
      set_error("system: fixed ids must be sorted, unique and in range");
      return fail(QN_ERR_ARG);
    }
    is_fixed[v] = 1;
    fixed_pos[v] = (int32_t)k;
  }
  std::vector<int32_t> free_ids;
  for (int64_t i = 0; i < n; ++i)
    if (!is_fixed[i]) free_ids.push_back((int32_t)i);
  S->n_free = (int64_t)free_ids.size();
  if (S->n_free == 0) {
    set_error("all vertices fixed; nothing to simulate");
    return fail(QN_ERR_ARG);
  }
  phase("fixed set");
  // tets, SoA Dm^-1, gather map (slots 4t + c in increasing order = reference scatter order)
  std::vector<int4> tets(std::max<int64_t>(mt, 1));
  std::vector<double> dminv((size_t)std::max<int64_t>(mt, 1) * 9);
  std::vector<int32_t> v2e_ptr(n + 1, 0), v2e((size_t)std::max<int64_t>(mt, 1) * 4);
  {
    const int corners = d->element_kind == QN_ELEM_SPRING ? 2 : 4;  // springs: (a, b, -1, -1)
    const int64_t stride = d->dminv_stride > 0 ? d->dminv_stride : 9;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t t = 0; t < mt; ++t) {
      const int32_t* tv = d->tets + 4 * t;
      for (int c = 0; c < 4; ++c)
        if (c < corners ? (tv[c] < 0 || tv[c] >= n) : tv[c] != -1) bad = 1;
      tets[t] = make_int4(tv[0], tv[1], tv[2], tv[3]);
      for (int k = 0; k < 9; ++k) dminv[(size_t)k * mt + t] = d->Dm_inv ? d->Dm_inv[stride * t + k] : 0.0;
    }
    if (bad) {
      set_error("system: element vertex out of range");
      return fail(QN_ERR_ARG);
    }
    for (int64_t t = 0; t < mt; ++t)
      for (int c = 0; c < corners; ++c) v2e_ptr[d->tets[4 * t + c] + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) v2e_ptr[i + 1] += v2e_ptr[i];
  {
    std::vector<int32_t> fill(v2e_ptr.begin(), v2e_ptr.end() - 1);
    for (int64_t t = 0; t < mt; ++t)
      for (int c = 0; c < 4; ++c)
        if (d->tets[4 * t + c] >= 0) v2e[fill[d->tets[4 * t + c]]++] = (int32_t)(4 * t + c);
  }
  if (d->tet_mat) {
    for (int64_t t = 0; t < mt; ++t)
      if (d->tet_mat[t] < 0 || d->tet_mat[t] >= d->n_mat) {
        set_error("system: material index out of range");
        return fail(QN_ERR_ARG);
      }
    S->h_tet_mat.assign(d->tet_mat, d->tet_mat + mt);
  }
  phase("tets + gather map");
  SysView& v = S->v;
  int rc = QN_OK;
  std::vector<int32_t> fact_vtx(S->n_free);
  const bool pcg = d->solver == QN_SOLVE_PCG || d->solver == QN_SOLVE_AMG;
  if (!pcg) {
    // factor of A_free (one numeric instance per system instance)
    S->factor = new qn_factor();
    rc = factor_build_host(S->factor, S->n_free, d->a_indptr, d->a_indices, d->a_values, ni, d->free_coords);
    if (rc == QN_OK) rc = factor_upload(S->factor);
    if (rc) return fail(rc);
    for (int64_t r = 0; r < S->n_free; ++r) fact_vtx[r] = free_ids[S->factor->perm[r]];
    v.n_free = (int32_t)S->n_free;  // factor rows (k_solve_rhs)
  } else {
    // PCG: A_free on the device as CSR (free-vertex order), Jacobi preconditioner
    QN_REQUIRE(d->pcg_tol > 0 && d->pcg_maxit > 0, QN_ERR_ARG, "system: PCG needs pcg_tol > 0 and pcg_maxit > 0");
    const int64_t nf = S->n_free, nnz = d->a_indptr[nf];
    std::vector<double> dinv((size_t)ni * nf, 0.0);
    for (int64_t b = 0; b < ni; ++b)
      for (int64_t r = 0; r < nf; ++r)
        for (int64_t p = d->a_indptr[r]; p < d->a_indptr[r + 1]; ++p)
          if (d->a_indices[p] == r) dinv[b * nf + r] = 1.0 / d->a_values[b * nnz + p];
    for (double x : dinv)
      if (!(x > 0.0)) {
        set_error("matrix is not positive definite (non-positive diagonal)");
        return fail(QN_ERR_NOT_SPD);
      }
    for (int64_t r = 0; r < nf; ++r) fact_vtx[r] = free_ids[r];
    const int64_t nsl = (nf + 31) / 32;
    std::vector<int64_t> sptr;
    std::vector<int32_t> scol;
    std::vector<double> sval;
    sell_build(nf, nf, d->a_indptr, d->a_indices, d->a_values, ni, nnz, sptr, scol, sval);
    const int64_t snz = sptr[nsl];
    int64_t* sp;
    int32_t* sc;
    double *sv, *di;
    if ((rc = sys_upload(S, &sp, sptr.data(), sptr.size())) || (rc = sys_upload(S, &sc, scol.data(), scol.size())) ||
        (rc = sys_upload(S, &sv, sval.data(), sval.size())) || (rc = sys_upload(S, &di, dinv.data(), dinv.size())))
      return fail(rc);
    v.sell_ptr = sp;
    v.sell_col = sc;
    v.sell_val = sv;
    v.sell_nnz = snz;
    v.nslice = (int32_t)nsl;
    v.dinv = di;
    v.pcg = d->solver == QN_SOLVE_AMG ? 2 : 1;
    v.n_free = (int32_t)nf;
    v.nblk_p = div_up(nf, 128);
    int dev = 0, nsm = 148;
    QN_CUDA(cudaGetDevice(&dev));
    QN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    v.nblk_spmv = (int32_t)std::min<int64_t>(div_up(nsl, qn::kSpmvWarps), (int64_t)nsm * qn::kSpmvBlocksPerSm);
    v.nblk_upd = (int32_t)std::min<int64_t>(div_up(3 * nf, qn::kUpdThreads), (int64_t)nsm * qn::kUpdBlocksPerSm);
    v.pcg_tol = d->pcg_tol;
    v.pcg_maxit = d->pcg_maxit;
    const size_t fv = (size_t)ni * nf * 3;
    const size_t npart = (size_t)std::max(v.nblk_p, std::max(v.nblk_spmv, v.nblk_upd));
    if ((rc = sys_alloc(S, &v.px, fv)) || (rc = sys_alloc(S, &v.pr, fv)) ||
        (rc = sys_alloc(S, &v.pp, 2 * fv)) || (rc = sys_alloc(S, &v.pq, fv)) ||
        (rc = sys_alloc(S, &v.part_p, (size_t)ni * npart * 8)) ||
        (rc = sys_alloc(S, &v.cnt_p, (size_t)4 * ni + 2)) || (rc = sys_alloc(S, &v.pctl, (size_t)ni)) ||
        (rc = sys_alloc(S, &v.pcg_active, 1)))
      return fail(rc);
    if (v.pcg == 2) {  // AMG hierarchy (host setup once), SELL operators + level vectors on the device
      QN_REQUIRE(ni == 1, QN_ERR_UNSUPPORTED, "system: the AMG solver supports one instance");
      phase("pcg operator");
      qn::AmgHierarchy H;
      H.skip_coarse_inverse = true;  // inverted on the device below (cuSOLVER Cholesky)
      if ((rc = qn::amg_build(nf, d->a_indptr, d->a_indices, d->a_values, &H))) return fail(rc);
      S->amg_setup_s = H.setup_seconds;
      const int nl = (int)H.lv.size();
      S->h_alev.assign(nl, qn::AmgDevLevel{});
      if ((rc = sys_alloc(S, &v.pz, fv))) return fail(rc);
      if ((rc = sys_alloc(S, &v.amg_bar, (size_t)2))) return fail(rc);
      {  // QN_AMG_ZF=0 (experiment knob): keep z in fp64 with the separate r.z kernel
        const char* e = std::getenv("QN_AMG_ZF");
        // (a one-level hierarchy has no smoothing kernel: its dense solve writes the fp64 z)
        if (nl >= 2 && !(e && std::atoi(e) == 0) && (rc = sys_alloc(S, &v.pzf, (size_t)nf))) return fail(rc);
        const char* er = std::getenv("QN_PCG_REC");  // experiment knob: 0 keeps the fused-p SpMV
        S->pcg_rec = v.pzf != nullptr && !(er && std::atoi(er) == 0);
      }
      for (int l = 0; l < nl; ++l) {
        const qn::AmgLevel& L = H.lv[l];
        qn::AmgDevLevel& D = S->h_alev[l];
        S->amg_nnz.push_back(L.A.ptr.empty() ? 0 : L.A.ptr.back());
        S->amg_nnz.push_back(L.P.ptr.empty() ? 0 : L.P.ptr.back());
        S->amg_nnz.push_back(L.R.ptr.empty() ? 0 : L.R.ptr.back());
        D.n = (int32_t)L.A.n;
        D.omega = H.omega_l[l];
        if ((rc = sell_upload(S, L.A.n, L.A.m, L.A.ptr.data(), L.A.col.data(), L.A.val.data(), &D.A))) return fail(rc);
        double* dd;
        if ((rc = sys_upload(S, &dd, L.dinv.data(), L.dinv.size()))) return fail(rc);
        D.dinv = dd;
        if (l + 1 < nl) {
          if ((rc = sell_upload(S, L.P.n, L.P.m, L.P.ptr.data(), L.P.col.data(), L.P.val.data(), &D.P)) ||
              (rc = sell_upload(S, L.R.n, L.R.m, L.R.ptr.data(), L.R.col.data(), L.R.val.data(), &D.R)))
            return fail(rc);
        }
        const size_t lvn = (size_t)L.A.n;
        if (l == 0) {
          D.b = v.pr;  // the CG residual
          D.t = v.pz;  // z = B r
        } else if ((rc = sys_alloc(S, &D.bf, lvn)) || (rc = sys_alloc(S, &D.tf, lvn))) {
          return fail(rc);
        }
        if ((rc = sys_alloc(S, &D.xf, lvn)) || (rc = sys_alloc(S, &D.rf, lvn))) return fail(rc);
        const int64_t nsl_l = (L.A.n + 31) / 32;
        D.nblk = (int32_t)std::max<int64_t>(1, std::min<int64_t>(div_up(nsl_l, qn::kSpmvWarps),
                                                                 (int64_t)nsm * qn::kSpmvBlocksPerSm));
      }
      qn::AmgDevLevel* dl;
      if ((rc = sys_upload(S, &dl, S->h_alev.data(), S->h_alev.size()))) return fail(rc);
      v.alev = dl;
      v.amg_levels = nl;
      v.ncoarse = (int32_t)H.lv.back().A.n;
      phase("amg build + upload");
      float* ci;
      if ((rc = coarse_inverse_device(S, H.lv.back().A, &ci))) return fail(rc);
      v.cinv = ci;
      phase("coarse inverse");
    }
  }

  v.n = (int32_t)n;
  v.mt = (int32_t)mt;
  v.n_inst = (int32_t)ni;
  v.n_mat = (int32_t)d->n_mat;
  v.n_fixed = (int32_t)d->n_fixed;
  v.vt = ni == 1 ? kVertexThreadsMax : kVertexThreads;
  if (const char* e = std::getenv("QN_VERTEX_THREADS"))  // experiment knob: 32 .. kVertexThreadsMax, multiple of 32
    v.vt = std::max(32, std::min(kVertexThreadsMax, (std::atoi(e) / 32) * 32));
  v.nblk_v = div_up(3 * n, v.vt);  // vector kernels run one thread per (vertex, coordinate)
  v.nblk_t = std::max(1, div_up(mt, kTetThreads));
  v.spring = d->element_kind == QN_ELEM_SPRING ? 1 : 0;
  v.aniso = 0;
  for (int64_t q = 0; q < ni * d->n_mat && mt > 0; ++q)
    if (d->mats[q].a.kind == QN_FN_ANISO) v.aniso = 1;
  if (d->n_colliders > 0) {  // colliders: per (instance, vertex, collider) constraint state
    const int64_t nc = d->n_colliders;
    qn_collider* dc;
    if ((rc = sys_upload(S, &dc, d->colliders, (size_t)nc)) ||
        (rc = sys_alloc(S, &v.col_act, (size_t)ni * n * nc)) || (rc = sys_alloc(S, &v.col_t, (size_t)ni * n * nc * 3)) ||
        (rc = sys_alloc(S, &v.col_n, (size_t)ni * n * nc * 3)) || (rc = sys_alloc(S, &v.col_g, (size_t)ni * n * 3)) ||
        (rc = sys_alloc(S, &v.part_c, (size_t)ni * div_up(n, kVertexThreads))) ||
        (rc = sys_alloc(S, &v.cnt_c, (size_t)ni)))
      return fail(rc);
    v.cols = dc;
    v.n_col = (int32_t)nc;
    v.nblk_c = div_up(n, kVertexThreads);
    v.w_col = d->w_col;
  }
  v.h = d->h;
  for (int a = 0; a < 3; ++a) v.grav[a] = d->gravity[a];
  const size_t vec = (size_t)ni * n * 3;
  {
    int4* p;
    if ((rc = sys_upload(S, &p, tets.data(), tets.size()))) return fail(rc);
    v.tets = p;
    double* dm;
    if ((rc = sys_upload(S, &dm, dminv.data(), dminv.size()))) return fail(rc);
    v.dminv = dm;
    double* vol;
    std::vector<double> vols(d->vols ? d->vols : nullptr, d->vols ? d->vols + mt : nullptr);
    if (vols.empty()) vols.push_back(0.0);
    if ((rc = sys_upload(S, &vol, vols.data(), vols.size()))) return fail(rc);
    v.vols = vol;
    if (d->tet_mat) {
      int32_t* tm;
      if ((rc = sys_upload(S, &tm, d->tet_mat, (size_t)mt))) return fail(rc);
      v.tet_mat = tm;
    }
    std::vector<qn_material> mats((size_t)ni * d->n_mat);
    if (d->mats) std::memcpy(mats.data(), d->mats, mats.size() * sizeof(qn_material));
    qn_material* dmats;
    if ((rc = sys_upload(S, &dmats, mats.data(), mats.size()))) return fail(rc);
    v.mats = dmats;
    double* ms;
    if ((rc = sys_upload(S, &ms, d->masses, (size_t)n))) return fail(rc);
    v.masses = ms;
    std::vector<double> w_in(n);
    for (int64_t i = 0; i < n; ++i) w_in[i] = d->masses[i] / (d->h * d->h);  // dynamics.py:472
    double* wi;
    if ((rc = sys_upload(S, &wi, w_in.data(), w_in.size()))) return fail(rc);
    v.w_in = wi;
    uint8_t* fx;
    if ((rc = sys_upload(S, &fx, is_fixed.data(), is_fixed.size()))) return fail(rc);
    v.is_fixed = fx;
    int32_t* fp;
    if ((rc = sys_upload(S, &fp, fixed_pos.data(), fixed_pos.size()))) return fail(rc);
    v.fixed_pos = fp;
    int32_t* vp;
    if ((rc = sys_upload(S, &vp, v2e_ptr.data(), v2e_ptr.size()))) return fail(rc);
    v.v2e_ptr = vp;
    int32_t* ve;
    if ((rc = sys_upload(S, &ve, v2e.data(), v2e.size()))) return fail(rc);
    v.v2e = ve;
    // corner forces are stored in gather order: slot 4t + c -> its v2e position
    std::vector<int32_t> slot_pos((size_t)std::max<int64_t>(mt, 1) * 4, -1);
    for (int64_t k = 0; k < v2e_ptr[n]; ++k) slot_pos[v2e[k]] = (int32_t)k;
    int32_t* sp;
    if ((rc = sys_upload(S, &sp, slot_pos.data(), slot_pos.size()))) return fail(rc);
    v.slot_pos = sp;
    int32_t* fv;
    if ((rc = sys_upload(S, &fv, fact_vtx.data(), fact_vtx.size()))) return fail(rc);
    v.fact_vtx = fv;
  }
  if ((rc = sys_alloc(S, &v.q_l, vec)) || (rc = sys_alloc(S, &v.q_prev, vec)) || (rc = sys_alloc(S, &v.y, vec)) ||
      (rc = sys_alloc(S, &v.X, 3 * vec)) || (rc = sys_alloc(S, &v.Gr, 2 * vec)) ||
      (rc = sys_alloc(S, &v.S, (size_t)(kMaxM + 1) * vec)) || (rc = sys_alloc(S, &v.T, (size_t)(kMaxM + 1) * vec)) ||
      (rc = sys_alloc(S, &v.R0, vec)) || (rc = sys_alloc(S, &v.D, vec)) || (rc = sys_alloc(S, &v.qf, vec)) ||
      (rc = sys_alloc(S, &v.forces, (size_t)ni * std::max<int64_t>(mt, 1) * 12)) ||
      (rc = sys_alloc(S, &v.part_v, (size_t)ni * v.nblk_v * kNG)) ||
      (rc = sys_alloc(S, &v.part_t, (size_t)ni * v.nblk_t)) || (rc = sys_alloc(S, &v.cnt, (size_t)4 * ni + 1)) ||
      (rc = sys_alloc(S, &v.ctl, (size_t)ni)) || (rc = sys_alloc(S, &S->d_cfg, 1)) ||
      (rc = sys_alloc(S, &v.active, 1)) || (rc = sys_alloc(S, &v.passes, 2)) ||
      (rc = sys_alloc(S, &S->d_targets, (size_t)ni * std::max<int64_t>(d->n_fixed, 1) * 3)) ||
      (rc = sys_alloc(S, &S->d_part_plain, (size_t)std::max((int64_t)v.nblk_t * v.n_inst, (int64_t)v.nblk_v) * 2)))
    return fail(rc);
  v.cfg = S->d_cfg;
  v.targets = S->d_targets;
  QN_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
  QN_CUDA(cudaEventCreate(&S->ev0));
  QN_CUDA(cudaEventCreate(&S->ev1));
  S->h_stage_bytes = vec * sizeof(double) * 3;
  QN_CUDA(cudaMallocHost((void**)&S->h_stage, S->h_stage_bytes));
  phase("solver + vectors");
  if ((rc = prepare_kernels(S))) return fail(rc);
  phase("prepare kernels");
  *out = S;
  return QN_OK;
}

int qn_newton_release(qn_system* S);

int qn_system_destroy(qn_system* S) {
  if (!S) return QN_OK;
  qn_newton_release(S);
  if (S->exec) cudaGraphExecDestroy(S->exec);
  if (S->graph) cudaGraphDestroy(S->graph);
  for (void* p : S->allocs) cudaFree(p);
  if (S->factor) qn_factor_destroy(S->factor);
  if (S->h_stage) cudaFreeHost(S->h_stage);
  if (S->h_rec) cudaFreeHost(S->h_rec);
  if (S->ev0) cudaEventDestroy(S->ev0);
  if (S->ev1) cudaEventDestroy(S->ev1);
  if (S->stream) cudaStreamDestroy(S->stream);
  delete S;
  return QN_OK;
}

int qn_system_factor(qn_system* S, qn_factor** out) {
  QN_REQUIRE(S && out, QN_ERR_ARG, "null");
  *out = S->factor;
  return QN_OK;
}

int qn_system_set_precision(qn_system* S, int32_t fp32) {
  QN_REQUIRE(S, QN_ERR_ARG, "set_precision: null");
  QN_REQUIRE(!fp32 || (!S->v.spring && !S->v.aniso), QN_ERR_UNSUPPORTED,
             "set_precision: the fp32 element pass covers Valanis-Landel / ARAP tets");
  S->v.f32 = fp32 ? 1 : 0;
  if (S->exec) {  // the frame graph holds the kernel instantiation
    cudaGraphExecDestroy(S->exec);
    S->exec = nullptr;
    cudaGraphDestroy(S->graph);
    S->graph = nullptr;
  }
  return QN_OK;
}

int qn_system_set_graph_mode(qn_system* S, int32_t use_graph) {
  QN_REQUIRE(S, QN_ERR_ARG, "null");
  S->use_graph = use_graph != 0;
  return QN_OK;
}

int qn_system_last_frame_ms(qn_system* S, double* ms) {
  QN_REQUIRE(S && ms, QN_ERR_ARG, "null");
  *ms = S->last_ms;
  return QN_OK;
}

int qn_system_last_frame_passes(qn_system* S, int64_t* passes) {
  QN_REQUIRE(S && passes, QN_ERR_ARG, "null");
  *passes = S->last_passes;
  return QN_OK;
}

// SELL-32 copy of CSR rows (same entry order within a row, zero padding with
// an in-range column); values of `ni` instances laid out [inst][nnz_sell]
void sell_build(int64_t nrows, int64_t ncols, const int64_t* ptr, const int32_t* col, const double* val,
                int64_t ni, int64_t nnz, std::vector<int64_t>& sptr, std::vector<int32_t>& scol,
                std::vector<double>& sval) {
  const int64_t nsl = (nrows + 31) / 32;
  sptr.assign((size_t)nsl + 1, 0);
  for (int64_t sl = 0; sl < nsl; ++sl) {
    int64_t w = 0;
    for (int64_t r = 32 * sl; r < std::min(nrows, 32 * sl + 32); ++r) w = std::max(w, ptr[r + 1] - ptr[r]);
    sptr[sl + 1] = sptr[sl] + 32 * w;
  }
  const int64_t snz = sptr[nsl];
  scol.assign((size_t)snz, 0);
  sval.assign((size_t)ni * snz, 0.0);
  for (int64_t sl = 0; sl < nsl; ++sl) {
    const int64_t w = (sptr[sl + 1] - sptr[sl]) / 32;
    for (int64_t l = 0; l < 32; ++l) {
      const int64_t r = 32 * sl + l;
      const int64_t p0 = r < nrows ? ptr[r] : 0, len = r < nrows ? ptr[r + 1] - p0 : 0;
      for (int64_t k = 0; k < w; ++k) {
        const int64_t e = sptr[sl] + 32 * k + l;
        scol[e] = k < len ? col[p0 + k] : (int32_t)std::min(r, ncols - 1);
        if (k < len)
          for (int64_t b = 0; b < ni; ++b) sval[b * snz + e] = val[b * nnz + p0 + k];
      }
    }
  }
}

static int sell_upload(qn_system* S, int64_t nrows, int64_t ncols, const int64_t* ptr, const int32_t* col,
                       const double* val, qn::SellDevF* out) {
  // layout by mean row length: short rows -> SELL-32 (lane per row), long rows
  // (Galerkin coarse operators, restriction) -> CSR with K lanes per row
  const int64_t nnz = ptr[nrows];
  const double mean = nrows ? (double)nnz / (double)nrows : 0.0;
  // swept on c5 (QN_AMG_CSR_LANES, V-cycle ms): 4 lanes per row 1.174, 8 1.208, 2 1.282, 16 1.364, 1 1.758
  int kl = mean <= 16.0 ? 0 : mean <= 128.0 ? 4 : 8;
  // experiment knob (off by default, measured neutral on configs[4]): on levels of at most
  // QN_AMG_SMALL_ROWS rows, enough lanes per row that a row is ONE masked batch of 4 entries per lane
  int64_t small_rows = 0;
  if (const char* e = std::getenv("QN_AMG_SMALL_ROWS")) small_rows = std::atoll(e);
  if (kl > 0 && nrows <= small_rows) {
    kl = 4;
    while (kl < 32 && 4.0 * kl < mean) kl *= 2;
  }
  if (const char* e = std::getenv("QN_AMG_CSR_LANES"))  // experiment knob: lanes per row of the CSR levels
    if (kl > 0) kl = std::max(1, std::min(32, std::atoi(e)));
  int dev = 0, nsm = qn::kSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = (int64_t)nsm * qn::kSpmvBlocksPerSm;
  std::vector<int64_t> sp;
  std::vector<int32_t> sc;
  std::vector<double> sv;
  if (kl == 0) {
    sell_build(nrows, ncols, ptr, col, val, 1, nnz, sp, sc, sv);
  } else {
    sp.assign(ptr, ptr + nrows + 1);
    sc.assign(col, col + nnz);
    sv.assign(val, val + nnz);
  }
  std::vector<float> sf(std::max<size_t>(sv.size(), 1), 0.0f);
  for (size_t k = 0; k < sv.size(); ++k) sf[k] = (float)sv[k];
  if (sc.empty()) sc.push_back(0);
  int64_t* dp;
  int32_t* dc;
  float* dv;
  int rc;
  if ((rc = sys_upload(S, &dp, sp.data(), sp.size())) || (rc = sys_upload(S, &dc, sc.data(), sc.size())) ||
      (rc = sys_upload(S, &dv, sf.data(), sf.size())))
    return rc;
  out->ptr = dp;
  out->col = dc;
  out->val = dv;
  out->nslice = kl == 0 ? (int32_t)(sp.size() - 1) : 0;
  out->nrows = (int32_t)nrows;
  out->kl = kl;
  const int64_t units = kl == 0 ? (nrows + 31) / 32 : (nrows + 32 / kl - 1) / (32 / kl);  // warps of work
  out->nblk = (int32_t)std::max<int64_t>(1, std::min<int64_t>((units + qn::kSpmvWarps - 1) / qn::kSpmvWarps, cap));
  return QN_OK;
}

int qn_system_amg_info(qn_system* S, int64_t* out, int64_t cap) {
  QN_REQUIRE(S && out && cap >= 12, QN_ERR_ARG, "amg_info: args");
  std::fill(out, out + cap, 0);
  const int64_t nl = (int64_t)S->h_alev.size();
  out[0] = nl;
  for (int64_t l = 0; l < nl && l < 10; ++l) out[1 + l] = S->h_alev[l].n;
  out[11] = (int64_t)(S->amg_setup_s * 1000.0);
  for (int64_t l = 0; l < nl && l < 10 && 12 + 3 * l + 2 < cap; ++l)  // nnz of A, P, R per level
    for (int k = 0; k < 3; ++k) out[12 + 3 * l + k] = S->amg_nnz[3 * l + k];
  return QN_OK;
}

int qn_frame_records_device(qn_system* S, int32_t iterations, double* g_out, int32_t* status_out, void* stream) {
  QN_REQUIRE(S && g_out && status_out && iterations >= 1 && iterations <= S->rec_cap, QN_ERR_ARG,
             "frame_records_device: args (iterations must not exceed the last frame's record capacity)");
  cudaStream_t st = pick(S, stream);
  QN_CUDA(cudaMemcpy2DAsync(g_out, sizeof(double) * iterations, S->v.rec_g, sizeof(double) * S->rec_cap,
                            sizeof(double) * iterations, S->n_inst, cudaMemcpyDeviceToDevice, st));
  QN_CUDA(cudaMemcpy2DAsync(status_out, sizeof(int32_t), reinterpret_cast<const char*>(S->v.ctl) +
                            offsetof(qn::InstCtl, status), sizeof(qn::InstCtl), sizeof(int32_t), S->n_inst,
                            cudaMemcpyDeviceToDevice, st));
  return QN_OK;
}

int qn_system_set_fault(qn_system* S, int32_t mode, int32_t iteration) {
  QN_REQUIRE(S && mode >= 0 && mode <= 2 && iteration >= 1 && iteration < (1 << 20), QN_ERR_ARG, "set_fault: args");
  S->fault = mode ? (mode | (iteration << 4)) : 0;
  return QN_OK;
}

int qn_system_set_timeline(qn_system* S, int32_t enable) {
  QN_REQUIRE(S, QN_ERR_ARG, "null");
  const size_t cnt = (size_t)qn::kTimelinePasses * qn::kTimelineKernels * 2;
  if (enable && !S->v.ktl) {
    int rc = sys_alloc(S, &S->v.ktl, cnt);
    if (rc) return rc;
  } else if (!enable) {
    S->v.ktl = nullptr;  // buffer stays owned by the system
  }
  if (S->factor) {
    qn_factor* f = S->factor;
    f->d_ktl = S->v.ktl;
    f->d_passes = S->v.passes;
    // the in-graph solves also record their task trace (last solve of a frame wins)
    const size_t items = (f->ftask.size() + f->btask.size()) * (size_t)f->nbatch;
    if (enable && !f->d_trace && items > 0) {
      int rc = dev_alloc(&f->d_trace, qn::kTraceSlots * items);
      if (rc) return rc;
    } else if (!enable && f->d_trace) {
      cudaFree(f->d_trace);
      f->d_trace = nullptr;
    }
  }
  if (S->exec) {  // kernels capture the view by value: rebuild the graph
    cudaGraphExecDestroy(S->exec);
    S->exec = nullptr;
    cudaGraphDestroy(S->graph);
    S->graph = nullptr;
  }
  return QN_OK;
}

int qn_system_timeline(qn_system* S, uint64_t* out, int64_t cap) {
  QN_REQUIRE(S && out, QN_ERR_ARG, "null");
  QN_REQUIRE(S->v.ktl, QN_ERR_ARG, "timeline: not enabled");
  const int64_t cnt = (int64_t)qn::kTimelinePasses * qn::kTimelineKernels * 2;
  QN_REQUIRE(cap >= cnt, QN_ERR_ARG, "timeline: buffer too small");
  QN_CUDA(cudaDeviceSynchronize());
  QN_CUDA(cudaMemcpy(out, S->v.ktl, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return QN_OK;
}

int qn_system_last_frame_cg_iterations(qn_system* S, int64_t* iters) {
  QN_REQUIRE(S && iters, QN_ERR_ARG, "null");
  *iters = 0;
  if (!S->v.pcg) return QN_OK;
  std::vector<qn::PcgCtl> pc((size_t)S->n_inst);
  QN_CUDA(cudaMemcpy(pc.data(), S->v.pctl, pc.size() * sizeof(qn::PcgCtl), cudaMemcpyDeviceToHost));
  for (const auto& p : pc) *iters += p.total;
  return QN_OK;
}

static int stage_in(qn_system* S, double* dst, const double* src, size_t count, int32_t mem, cudaStream_t st) {
  if (mem == QN_MEM_DEVICE) return to_device(dst, src, count, mem, st);
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
    // caller's buffer is page-locked: one stream-ordered DMA, no staging copy
    QN_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyHostToDevice, st));
    return QN_OK;
  }
  (void)cudaGetLastError();
  // pageable: copy into the library's pinned staging buffer first
  QN_REQUIRE(count * sizeof(double) <= S->h_stage_bytes, QN_ERR_ARG, "stage: too large");
  QN_CUDA(cudaStreamSynchronize(st));
  std::memcpy(S->h_stage, src, count * sizeof(double));
  QN_CUDA(cudaMemcpyAsync(dst, S->h_stage, count * sizeof(double), cudaMemcpyHostToDevice, st));
  QN_CUDA(cudaStreamSynchronize(st));
  return QN_OK;
}

int qn_state_set(qn_system* S, const double* q_l, const double* q_prev, int32_t mem, void* stream) {
  QN_REQUIRE(S && q_l && q_prev, QN_ERR_ARG, "state_set: null");
  cudaStream_t st = pick(S, stream);
  const size_t vec = (size_t)S->n_inst * S->n * 3;
  int rc = stage_in(S, S->v.q_l, q_l, vec, mem, st);
  if (rc) return rc;
  return stage_in(S, S->v.q_prev, q_prev, vec, mem, st);
}

int qn_state_get(qn_system* S, double* q_l, double* q_prev, double* y, int32_t mem, void* stream) {
  QN_REQUIRE(S, QN_ERR_ARG, "state_get: null");
  cudaStream_t st = pick(S, stream);
  const size_t vec = (size_t)S->n_inst * S->n * 3;
  int rc;
  if (q_l && (rc = from_device(q_l, S->v.q_l, vec, mem, st))) return rc;
  if (q_prev && (rc = from_device(q_prev, S->v.q_prev, vec, mem, st))) return rc;
  if (y && (rc = from_device(y, S->v.y, vec, mem, st))) return rc;
  QN_CUDA(cudaStreamSynchronize(st));
  return QN_OK;
}

static int ensure_records(qn_system* S, int iterations) {
  if (iterations <= S->rec_cap) return QN_OK;
  int cap = std::max(iterations, 32);
  const size_t ni = (size_t)S->n_inst, cnt = ni * cap;
  const size_t bytes = sizeof(double) * (3 * cnt + ni) + sizeof(int32_t) * (cnt + 2 * ni);
  int rc;
  char* pack = nullptr;
  if ((rc = sys_alloc(S, &pack, bytes))) return rc;
  S->v.rec_g = reinterpret_cast<double*>(pack);
  S->v.rec_alpha = S->v.rec_g + cnt;
  S->v.rec_ms = S->v.rec_alpha + cnt;
  S->v.rec_g0 = S->v.rec_ms + cnt;
  S->v.rec_trials = reinterpret_cast<int32_t*>(S->v.rec_g0 + ni);
  S->v.rec_status = S->v.rec_trials + cnt;
  S->v.rec_fb = S->v.rec_status + ni;
  if (S->h_rec) cudaFreeHost(S->h_rec);
  S->h_rec = nullptr;
  QN_CUDA(cudaMallocHost(&S->h_rec, bytes));
  S->rec_bytes = bytes;
  S->rec_cap = cap;
  S->v.rec_cap = cap;
  if (S->exec) {  // pointers changed: rebuild the graph
    cudaGraphExecDestroy(S->exec);
    S->exec = nullptr;
    cudaGraphDestroy(S->graph);
    S->graph = nullptr;
  }
  return QN_OK;
}

int qn_frame_step(qn_system* S, const qn_solver_config* cfg, const double* fixed_targets, qn_frame_record* rec,
                  int32_t mem, int32_t sync, void* stream) {
  QN_REQUIRE(S && cfg, QN_ERR_ARG, "frame_step: null");
  QN_REQUIRE(cfg->kind >= 0 && cfg->kind <= 2, QN_ERR_UNSUPPORTED, "solver kind not supported on the B200 path");
  QN_REQUIRE(cfg->kind != 2 || (cfg->rho >= 0.0 && cfg->rho < 1.0), QN_ERR_ARG, "frame_step: chebyshev rho");
  QN_REQUIRE(cfg->iterations >= 1 && cfg->m >= 0 && cfg->m <= kMaxM, QN_ERR_ARG, "frame_step: bad iterations/m");
  QN_REQUIRE(cfg->gamma > 0 && cfg->gamma < 1, QN_ERR_ARG, "frame_step: gamma");
  QN_REQUIRE(sync || !rec, QN_ERR_ARG, "frame_step: a record needs sync");
  cudaStream_t st = pick(S, stream);
  int rc = ensure_records(S, cfg->iterations);
  if (rc) return rc;
  DevConfig& c = S->h_cfg;
  c.kind = cfg->kind;
  c.iterations = cfg->iterations;
  c.m = cfg->kind == 1 ? cfg->m : 0;
  c.line_search = cfg->line_search;
  c.gamma = cfg->gamma;
  c.alpha_init = cfg->alpha_init;
  c.shrink = cfg->alpha_shrink;
  c.grad_tol = 1e-12 * S->scale * std::max(1.0, S->max_mass / (S->h * S->h));  // solvers.py:278
  c.cheb_rho = cfg->rho;
  c.cheb_S = cfg->S;
  QN_REQUIRE(cfg->lbfgs_init >= 0 && cfg->lbfgs_init <= 2, QN_ERR_UNSUPPORTED, "frame_step: lbfgs_init");
  QN_REQUIRE(cfg->lbfgs_init == 0 || !S->v.pcg, QN_ERR_UNSUPPORTED,
             "frame_step: this lbfgs_init needs a direct-solver system");
  QN_REQUIRE(cfg->lbfgs_init != 2 || cfg->kind != 1 || (S->v.hrest_inv && S->n_inst == 1), QN_ERR_ARG,
             "frame_step: rest_pose_hessian needs qn_system_rest_hessian first (single instance)");
  c.lbfgs_init = cfg->kind == 1 ? cfg->lbfgs_init : 0;
  c.fault = S->fault;
  c.has_targets = fixed_targets != nullptr && S->n_fixed > 0;
  c.use_graph = S->use_graph ? 1 : 0;
  // Runaway guard: the line search (solvers.py:241-257) shrinks alpha from
  // alpha_init until it accepts or alpha < 1e-12, so one iteration takes at most
  // ceil(log(1e-12 / alpha_init) / log(shrink)) + 1 trials plus one
  // re-evaluation pass; the bound follows the configured alpha_init / shrink.
  QN_REQUIRE(!(cfg->line_search && cfg->alpha_shrink >= 1.0 && cfg->alpha_init >= 1e-12), QN_ERR_UNSUPPORTED,
             "frame_step: alpha_shrink >= 1 never reaches the step floor (the line search cannot terminate)");
  {
    double trials = 1.0;
    if (cfg->line_search && cfg->alpha_shrink > 0.0 && cfg->alpha_init >= 1e-12)
      trials = std::ceil(std::log(1e-12 / cfg->alpha_init) / std::log(cfg->alpha_shrink)) + 1.0;
    const double bound = (double)cfg->iterations * (std::max(trials, 1.0) + 2.0) + 64.0;
    QN_REQUIRE(bound < 2.0e9, QN_ERR_UNSUPPORTED, "frame_step: line-search trial bound too large");
    c.max_passes = (int32_t)bound;
  }
  QN_CUDA(cudaMemcpyAsync(S->d_cfg, &c, sizeof(DevConfig), cudaMemcpyHostToDevice, st));
  if (c.has_targets) {
    rc = stage_in(S, S->d_targets, fixed_targets, (size_t)S->n_inst * S->n_fixed * 3, mem, st);
    if (rc) return rc;
  }
  if (S->v.ktl)
    QN_CUDA(cudaMemsetAsync(S->v.ktl, 0,
                            sizeof(uint64_t) * qn::kTimelinePasses * qn::kTimelineKernels * 2, st));
  QN_CUDA(cudaEventRecord(S->ev0, st));
  if (S->use_graph) {
    const int mb = c.m <= 5 ? 5 : kMaxM;  // kernels are specialised on the history bound
    if (S->exec && (S->graph_m_bound != mb || S->graph_init != c.lbfgs_init)) {
      cudaGraphExecDestroy(S->exec);
      S->exec = nullptr;
      cudaGraphDestroy(S->graph);
      S->graph = nullptr;
    }
    if (!S->exec) {
      if (const char* e = std::getenv("QN_PDL")) S->pdl = std::atoi(e) != 0;  // experiment knob
      if (S->factor) S->factor->pdl = S->pdl ? 1 : 0;
      rc = build_graph(S);
      if (rc && S->pdl) {
        // programmatic edges refused by this driver (e.g. inside the conditional body): abandon the
        // capture and rebuild the frame graph with fully serialised launches
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(st, &dead);
        cudaGetLastError();
        S->pdl = false;
        if (S->factor) S->factor->pdl = 0;
        rc = build_graph(S);
      }
      if (rc) return rc;
      S->graph_m_bound = mb;
      S->graph_init = c.lbfgs_init;
    }
    QN_CUDA(cudaGraphLaunch(S->exec, st));
    count_launch(0);
  } else {
    if ((rc = launch_init(S, st))) return rc;
    for (int pass = 0; pass <= c.max_passes; ++pass) {
      if ((rc = launch_body(S, st))) return rc;
      int32_t act = 0;
      QN_CUDA(cudaMemcpyAsync(&act, S->v.active, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      QN_CUDA(cudaStreamSynchronize(st));
      if (act <= 0) break;
    }
    if ((rc = launch_finish(S, st))) return rc;
  }
  QN_CUDA(cudaEventRecord(S->ev1, st));
  if (!sync) return QN_OK;
  QN_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  QN_CUDA(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
  S->last_ms = ms;
  unsigned long long pe[2] = {0, 0};  // passes, OR of the instances' error bits (2 ascent, 4 CG at pcg_maxit)
  QN_CUDA(cudaMemcpy(pe, S->v.passes, sizeof(pe), cudaMemcpyDeviceToHost));
  const unsigned long long passes = pe[0];
  S->last_passes = (int64_t)passes;
  if (S->use_graph) {  // kernel nodes the graph executed: init + finish + passes + CG iterations
    int64_t cg = 0;
    if (S->v.pcg && S->kernels_per_cg > 0 && qn_system_last_frame_cg_iterations(S, &cg) != QN_OK) cg = 0;
    count_launch((int)(2 + S->kernels_per_pass * (int64_t)passes + S->kernels_per_cg * cg));
  }
  if (S->factor && (rc = factor_check_watchdog(S->factor))) return rc;
  if ((int64_t)passes > (int64_t)c.max_passes) {
    set_error("frame: pass limit exceeded (phase machine did not terminate)");
    return QN_ERR_CUDA;
  }
  if (pe[1] & 8) {
    set_error("frame: the AMG tail kernel's grid barrier timed out (its CTAs were not all resident)");
    return QN_ERR_CUDA;
  }
  if (pe[1] & 4) {  // the direct solve is exact; an unconverged CG direction is reported, not used silently
    set_error("frame: PCG stopped at pcg_maxit before reaching pcg_tol (raise pcg_maxit or pcg_tol)");
    return QN_ERR_ASCENT;
  }
  if ((pe[1] & 2) && !rec) {  // with a record the caller reports the failing instance (status bit 1)
    set_error("line search requires a descent direction (solvers.py:244-246)");
    return QN_ERR_ASCENT;
  }
  if (rec) {
    const int it = cfg->iterations, cap = S->rec_cap;
    const int64_t ni = S->n_inst;
    const size_t cnt = (size_t)ni * cap;
    // one D2H of the packed record arrays (k_finish copied the control blocks' g0 / status / fallbacks)
    QN_CUDA(cudaMemcpyAsync(S->h_rec, S->v.rec_g, S->rec_bytes, cudaMemcpyDeviceToHost, st));
    QN_CUDA(cudaStreamSynchronize(st));
    const double* hg = static_cast<const double*>(S->h_rec);
    const double *g = hg, *al = hg + cnt, *ms_ = hg + 2 * cnt, *hg0 = hg + 3 * cnt;
    const int32_t* tr = reinterpret_cast<const int32_t*>(hg0 + ni);
    const int32_t *hst = tr + cnt, *hfb = hst + ni;
    std::vector<double> g0(hg0, hg0 + ni);
    std::vector<int32_t> status(hst, hst + ni), fallbacks(hfb, hfb + ni);
    std::vector<double> og((size_t)ni * it), oa((size_t)ni * it), om((size_t)ni * it);
    std::vector<int32_t> ot((size_t)ni * it);
    for (int64_t b = 0; b < ni; ++b)
      for (int k = 0; k < it; ++k) {
        og[b * it + k] = g[b * cap + k];
        oa[b * it + k] = al[b * cap + k];
        om[b * it + k] = ms_[b * cap + k];
        ot[b * it + k] = tr[b * cap + k];
      }
    auto put = [&](auto* dst, const auto& src) -> int {
      if (!dst) return QN_OK;
      using T = typename std::decay<decltype(src[0])>::type;
      if (mem == QN_MEM_DEVICE) {
        QN_CUDA(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
      } else {
        std::memcpy(dst, src.data(), src.size() * sizeof(T));
      }
      return QN_OK;
    };
    if ((rc = put(rec->g0, g0)) || (rc = put(rec->g, og)) || (rc = put(rec->ls_trials, ot)) ||
        (rc = put(rec->alphas, oa)) || (rc = put(rec->cum_ms, om)) || (rc = put(rec->status, status)) ||
        (rc = put(rec->fallbacks, fallbacks)))
      return rc;
  }
  return QN_OK;
}

int qn_simulate_frame(qn_system* S, const qn_solver_config* cfg, const double* q_l, const double* q_prev,
                      const double* fixed_targets, double* x_out, double* y_out, qn_frame_record* rec, int32_t mem,
                      void* stream) {
  int rc = qn_state_set(S, q_l, q_prev, mem, stream);
  if (rc) return rc;
  rc = qn_frame_step(S, cfg, fixed_targets, rec, mem, 1, stream);
  if (rc) return rc;
  return qn_state_get(S, x_out, nullptr, y_out, mem, stream);
}

int qn_system_objective(qn_system* S, const double* x, const double* y, double* g_out, double* grad_out, int32_t mem,
                        void* stream) {
  QN_REQUIRE(S && x && y && g_out, QN_ERR_ARG, "objective: null");
  // in order on the caller's stream (device inputs are ready there); scratch is
  // the system's own, so nothing is allocated or leaked per call
  cudaStream_t st = pick(S, stream);
  const size_t nv = (size_t)S->n * 3;
  int rc;
  if ((rc = ensure_scratch(S))) return rc;
  double *dx = S->scratch[0], *dy = S->scratch[1], *dg = S->scratch[2];
  const SysView& v = S->v;
  std::vector<double> pt(v.nblk_t), pv(v.nblk_v);
  for (int64_t b = 0; b < S->n_inst; ++b) {
    if ((rc = to_device(dx, x + b * nv, nv, mem, st)) || (rc = to_device(dy, y + b * nv, nv, mem, st))) return rc;
    if ((rc = launch_tet_plain(S, dx, (int)b, -1, S->d_part_plain, st))) return rc;
    k_gather_plain<<<v.nblk_v, v.vt, 0, st>>>(v, dx, dy, dg, (int)b, 1, 1, S->d_part_plain + v.nblk_t);
    QN_CHECK_LAUNCH();
    QN_CUDA(cudaMemcpyAsync(pt.data(), S->d_part_plain, v.nblk_t * sizeof(double), cudaMemcpyDeviceToHost, st));
    QN_CUDA(cudaMemcpyAsync(pv.data(), S->d_part_plain + v.nblk_t, v.nblk_v * sizeof(double), cudaMemcpyDeviceToHost,
                            st));
    if (grad_out && (rc = from_device(grad_out + b * nv, dg, nv, mem, st))) return rc;
    QN_CUDA(cudaStreamSynchronize(st));
    double e = 0.0, in = 0.0;
    for (double p : pt) e += p;
    for (double p : pv) in += p;
    const double gv = (0.5 / (S->h * S->h)) * in + e;
    if (mem == QN_MEM_DEVICE) {
      QN_CUDA(cudaMemcpyAsync(g_out + b, &gv, sizeof(double), cudaMemcpyHostToDevice, st));
      QN_CUDA(cudaStreamSynchronize(st));
    } else {
      g_out[b] = gv;
    }
  }
  return QN_OK;
}

int qn_system_elements(qn_system* S, int64_t inst, int64_t mat, const double* x, double* energy, double* grad_accum,
                       int32_t mem, void* stream) {
  QN_REQUIRE(S && x && energy && inst >= 0 && inst < S->n_inst && mat < S->n_mat, QN_ERR_ARG, "elements: args");
  cudaStream_t st = pick(S, stream);
  const size_t nv = (size_t)S->n * 3;
  int rc;
  if ((rc = ensure_scratch(S))) return rc;
  double *dx = S->scratch[0], *dg = S->scratch[2];
  const SysView& v = S->v;
  if ((rc = to_device(dx, x, nv, mem, st))) return rc;
  if ((rc = launch_tet_plain(S, dx, (int)inst, (int)mat, S->d_part_plain, st))) return rc;
  if (grad_accum) {
    if ((rc = to_device(dg, grad_accum, nv, mem, st))) return rc;
    k_gather_plain<<<v.nblk_v, v.vt, 0, st>>>(v, dx, nullptr, dg, (int)inst, 0, 0, nullptr);
    QN_CHECK_LAUNCH();
    if ((rc = from_device(grad_accum, dg, nv, mem, st))) return rc;
  }
  std::vector<double> pt(v.nblk_t);
  QN_CUDA(cudaMemcpyAsync(pt.data(), S->d_part_plain, v.nblk_t * sizeof(double), cudaMemcpyDeviceToHost, st));
  QN_CUDA(cudaStreamSynchronize(st));
  double e = 0.0;
  for (double p : pt) e += p;
  if (mem == QN_MEM_DEVICE) {
    QN_CUDA(cudaMemcpyAsync(energy, &e, sizeof(double), cudaMemcpyHostToDevice, st));
    QN_CUDA(cudaStreamSynchronize(st));
  } else {
    *energy = e;
  }
  return QN_OK;
}

int qn_system_time_kernel(qn_system* S, int32_t kernel, int32_t reps, double* avg_ms, void* stream) {
  QN_REQUIRE(S && avg_ms && reps >= 1 && kernel >= 0 && kernel <= 3, QN_ERR_ARG, "time_kernel: args");
  // kernel 3 = one AMG V(1,1) cycle on the resident level vectors: its kernels
  // only run for an instance in the direction phase with an unconverged CG,
  // so the two control words are set for the timing and restored after
  int32_t saved_phase = 0, saved_conv = 0;
  if (kernel == 3) {
    QN_REQUIRE(S->v.pcg == 2, QN_ERR_UNSUPPORTED, "time_kernel: vcycle needs an AMG system");
    QN_CUDA(cudaMemcpy(&saved_phase, &S->v.ctl[0].phase, sizeof(int32_t), cudaMemcpyDeviceToHost));
    QN_CUDA(cudaMemcpy(&saved_conv, &S->v.pctl[0].conv, sizeof(int32_t), cudaMemcpyDeviceToHost));
    const int32_t on = qn::PH_DIR, zero = 0;
    QN_CUDA(cudaMemcpy(&S->v.ctl[0].phase, &on, sizeof(int32_t), cudaMemcpyHostToDevice));
    QN_CUDA(cudaMemcpy(&S->v.pctl[0].conv, &zero, sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  cudaStream_t st = pick(S, stream);
  const SysView& v = S->v;
  int rc;
  auto launch = [&]() -> int {
    if (kernel == 0) {  // per-tet pass (F, SVD, VL energy, PK1 corner forces) at the resident q_l
      int r = launch_tet_plain(S, v.q_l, -1, -1, S->d_part_plain, st);  // every instance
      if (r) return r;
    } else if (kernel == 1) {  // forward + backward supernodal solves with 3 RHS, every instance
      QN_REQUIRE(S->factor, QN_ERR_UNSUPPORTED, "time_kernel: no factor (PCG system)");
      int r = launch_solve_timing(S, st);
      if (r) return r;
    } else if (kernel == 2) {  // the CG's SpMV q = A_free x (PCG / AMG systems)
      QN_REQUIRE(S->v.pcg, QN_ERR_UNSUPPORTED, "time_kernel: spmv needs a PCG system");
      int r = launch_spmv_timing(S, st);
      if (r) return r;
    } else {
      int r = launch_vcycle(S, st);
      if (r) return r;
    }
    return QN_OK;
  };
  if ((rc = launch())) return rc;  // warm-up
  QN_CUDA(cudaStreamSynchronize(st));
  QN_CUDA(cudaEventRecord(S->ev0, st));
  for (int r = 0; r < reps; ++r)
    if ((rc = launch())) return rc;
  QN_CUDA(cudaEventRecord(S->ev1, st));
  QN_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  QN_CUDA(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
  *avg_ms = ms / reps;
  if (kernel == 3) {
    QN_CUDA(cudaMemcpy(&S->v.ctl[0].phase, &saved_phase, sizeof(int32_t), cudaMemcpyHostToDevice));
    QN_CUDA(cudaMemcpy(&S->v.pctl[0].conv, &saved_conv, sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  return QN_OK;
}

}  // extern "C"

// Newton direction on the device (solvers.py:167-234): the reference's
// baseline for reference minima g* (newton_reference, :355-398) and the
// solver kind "newton".
//   1. per element, a 12x12 Hessian block by central differences of the
//      element's corner forces (step = 1e-6 scale, _elem_hessians_fd :170-185),
//      symmetrised, eigenvalues clamped at 1e-8 (project_psd :188-192, cyclic
//      Jacobi per thread);
//   2. the dense free-dof Hessian H = sum of the blocks + M/h^2, each entry a
//      fixed-order sum in the reference's COO order (element, then row-major
//      block entry), the mass term last (newton_hessian_fact :195-225);
//   3. d_free = -H^-1 g_free by a dense Cholesky (cuSOLVER potrf/potrs, a
//      library factorisation of the reference's dense cho_factor);
//      FactorizationError when H is not SPD.
// Meant for the small meshes the reference runs Newton on (dense 3n x 3n).
#include <cusolverDn.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "qn_kernels.cuh"

namespace qn {

constexpr int kNT = 64;  // Newton element-kernel block

// corner forces of element t at corner positions xs (the same branches as the per-tet pass)
__device__ __forceinline__ void elem_forces(const SysView& v, const qn_material& M, int4 tv, const double (&xs)[4][3],
                                            const double (&Dm)[3][3], double vol, double (&f)[4][3]) {
  if (v.spring) {
    const double w = M.a.c[0];
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = xs[1][a] - xs[0][a];
    const double len = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    const double s = w * (1.0 - vol / fmax(len, 1e-300));
    for (int a = 0; a < 3; ++a) {
      f[0][a] = -s * d[a];
      f[1][a] = s * d[a];
      f[2][a] = f[3][a] = 0.0;
    }
    return;
  }
  tet_eval<true>(M, xs, Dm, vol, f);
  if (M.a.kind == QN_FN_ANISO) aniso_eval(M, xs, Dm, vol, f);
}

// symmetric eigen-decomposition by cyclic Jacobi (n = 12 or 6), then
// H = Q max(w, floor) Q^T written back into H (row-major n x n)
__device__ void psd_project(double* H, double* Q, int n, double floor_) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Q[i * n + j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += H[i * n + i] * H[i * n + i];
      for (int j = i + 1; j < n; ++j) off += H[i * n + j] * H[i * n + j];
    }
    if (off <= 1e-32 * diag || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = H[p * n + q];
        if (apq == 0.0) continue;
        const double app = H[p * n + p], aqq = H[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double hkp = H[k * n + p], hkq = H[k * n + q];
          H[k * n + p] = c * hkp - s * hkq;
          H[k * n + q] = s * hkp + c * hkq;
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double hpk = H[p * n + k], hqk = H[q * n + k];
          H[p * n + k] = c * hpk - s * hqk;
          H[q * n + k] = s * hpk + c * hqk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[k * n + p], qkq = Q[k * n + q];
          Q[k * n + p] = c * qkp - s * qkq;
          Q[k * n + q] = s * qkp + c * qkq;
        }
      }
  }
  double w[12];
  for (int i = 0; i < n; ++i) w[i] = fmax(H[i * n + i], floor_);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double a = 0.0;
      for (int k = 0; k < n; ++k) a += Q[i * n + k] * w[k] * Q[j * n + k];
      H[i * n + j] = a;
    }
}

// one element per thread: FD Hessian block (dim = 12 for tets, 6 for springs) -> He[t][144]
__global__ void __launch_bounds__(kNT) k_newton_blocks(SysView v, const double* __restrict__ x, double step,
                                                       double floor_, double* He, double* scratch) {
  const int t_raw = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = min(t_raw, v.mt - 1);  // all lanes run (the SVD's sweeps end on warp votes)
  const int4 tv = __ldg(v.tets + t);
  const int na = v.spring ? 2 : 4, dim = 3 * na;
  const int id[4] = {tv.x, tv.y, v.spring ? tv.x : tv.z, v.spring ? tv.y : tv.w};
  double xs[4][3];
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 3; ++a) xs[k][a] = x[3 * id[k] + a];
  double Dm[3][3];
  for (int r = 0; r < 3; ++r)
    for (int q = 0; q < 3; ++q) Dm[r][q] = v.spring ? 0.0 : __ldg(v.dminv + (size_t)(r * 3 + q) * v.mt + t);
  const double vol = __ldg(v.vols + t);
  const int mi = v.tet_mat ? __ldg(v.tet_mat + t) : 0;
  const qn_material& M = v.mats[mi];
  double* H = scratch + (size_t)t_raw * 288;  // [144] block | [144] eigenvectors
  for (int col = 0; col < 12; ++col) {
    if (col >= dim) break;
    const int vv = col / 3, c = col % 3;
    double fp[4][3], fm[4][3];
    const double x0 = xs[vv][c];
    xs[vv][c] = x0 + step;
    elem_forces(v, M, tv, xs, Dm, vol, fp);
    xs[vv][c] = x0 - step;
    elem_forces(v, M, tv, xs, Dm, vol, fm);
    xs[vv][c] = x0;
    for (int r = 0; r < dim; ++r) H[r * dim + col] = (fp[r / 3][r % 3] - fm[r / 3][r % 3]) / (2.0 * step);
  }
  for (int i = 0; i < dim; ++i)  // 0.5 (H + H^T)
    for (int j = i + 1; j < dim; ++j) {
      const double s = 0.5 * (H[i * dim + j] + H[j * dim + i]);
      H[i * dim + j] = H[j * dim + i] = s;
    }
  psd_project(H, H + 144, dim, floor_);
  if (t_raw < v.mt)
    for (int e = 0; e < dim * dim; ++e) He[(size_t)t_raw * 144 + e] = H[e];
}

// dense free-dof Hessian: entry k of the pattern sums its contributions in
// the reference's order, the diagonal adds M/h^2 last
__global__ void k_newton_assemble(int64_t npat, const int64_t* pat_dst, const int64_t* ptr, const int64_t* src,
                                  const double* He, const double* diag_add, double* Hd) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npat) return;
  double a = 0.0;
  for (int64_t e = ptr[k]; e < ptr[k + 1]; ++e) a += He[src[e]];
  a += diag_add[k];
  Hd[pat_dst[k]] = a;
}

__global__ void k_newton_rhs(int nf3, const int32_t* free3, const double* grad, double* b) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nf3) b[k] = -grad[free3[k]];
}

__global__ void k_newton_put(int nf3, const int32_t* free3, const double* b, double* d) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nf3) d[free3[k]] = b[k];
}

}  // namespace qn

namespace {

struct NewtonWork {
  bool ready = false;
  int64_t nf3 = 0, npat = 0, ncontrib = 0;
  int32_t* free3 = nullptr;
  int64_t *pat_dst = nullptr, *ptr = nullptr, *src = nullptr;
  double *diag_add = nullptr, *He = nullptr, *scratch = nullptr, *H = nullptr, *b = nullptr, *x = nullptr,
         *g = nullptr, *d = nullptr, *work = nullptr;
  int* info = nullptr;
  int lwork = 0;
  cusolverDnHandle_t solver = nullptr;
};

std::vector<std::pair<qn_system*, NewtonWork*>> g_newton;  // per system (released with the system)
std::mutex g_newton_mu;  // guards the table; a system's workspace is used by one thread at a time

NewtonWork* work_of(qn_system* S) {
  std::lock_guard<std::mutex> lock(g_newton_mu);
  for (auto& p : g_newton)
    if (p.first == S) return p.second;
  g_newton.push_back({S, new NewtonWork()});
  return g_newton.back().second;
}

template <class T>
int nalloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    qn::set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return QN_ERR_ALLOC;
  }
  return QN_OK;
}

// pattern of the dense free-dof Hessian from the element dofs (host, once)
int newton_setup(qn_system* S, NewtonWork* W) {
  using namespace qn;
  const SysView& v = S->v;
  const int64_t n = S->n, mt = S->mt;
  std::vector<int4> tets((size_t)std::max<int64_t>(mt, 1));
  QN_CUDA(cudaMemcpy(tets.data(), v.tets, mt * sizeof(int4), cudaMemcpyDeviceToHost));
  std::vector<uint8_t> fixed((size_t)n);
  QN_CUDA(cudaMemcpy(fixed.data(), v.is_fixed, n, cudaMemcpyDeviceToHost));
  std::vector<double> masses((size_t)n);
  QN_CUDA(cudaMemcpy(masses.data(), v.masses, n * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<int64_t> fidx(3 * n, -1);
  std::vector<int32_t> free3;
  for (int64_t i = 0; i < n; ++i)
    if (!fixed[i])
      for (int c = 0; c < 3; ++c) {
        fidx[3 * i + c] = (int64_t)free3.size();
        free3.push_back((int32_t)(3 * i + c));
      }
  const int64_t nf3 = (int64_t)free3.size();
  QN_REQUIRE(nf3 > 0 && nf3 <= 60000, QN_ERR_UNSUPPORTED, "newton: dense Hessian limited to 60000 free dofs");
  // contributions (dst entry, src index) in the reference's COO order
  const int na = v.spring ? 2 : 4, dim = 3 * na;
  std::vector<std::pair<int64_t, int64_t>> con;
  con.reserve((size_t)mt * dim * dim);
  for (int64_t t = 0; t < mt; ++t) {
    const int id[4] = {tets[t].x, tets[t].y, tets[t].z, tets[t].w};
    for (int r = 0; r < dim; ++r) {
      const int64_t fr = fidx[3 * id[r / 3] + r % 3];
      if (fr < 0) continue;
      for (int c = 0; c < dim; ++c) {
        const int64_t fc = fidx[3 * id[c / 3] + c % 3];
        if (fc < 0) continue;
        con.push_back({fr * nf3 + fc, t * 144 + r * dim + c});
      }
    }
  }
  for (int64_t f = 0; f < nf3; ++f) con.push_back({f * nf3 + f, -1});  // the mass diagonal (added last)
  std::stable_sort(con.begin(), con.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<int64_t> pat_dst, ptr{0}, src;
  std::vector<double> diag_add;
  for (size_t e = 0; e < con.size();) {
    size_t f = e;
    double dg = 0.0;
    while (f < con.size() && con[f].first == con[e].first) {
      if (con[f].second >= 0) {
        src.push_back(con[f].second);
      } else {
        const int32_t dof = free3[con[f].first / nf3];
        dg = masses[dof / 3] / (S->h * S->h);
      }
      ++f;
    }
    pat_dst.push_back(con[e].first);
    ptr.push_back((int64_t)src.size());
    diag_add.push_back(dg);
    e = f;
  }
  int rc;
  if ((rc = nalloc(&W->free3, free3.size())) || (rc = nalloc(&W->pat_dst, pat_dst.size())) ||
      (rc = nalloc(&W->ptr, ptr.size())) || (rc = nalloc(&W->src, src.size())) ||
      (rc = nalloc(&W->diag_add, diag_add.size())) || (rc = nalloc(&W->He, (size_t)mt * 144)) ||
      (rc = nalloc(&W->scratch, (size_t)(mt + kNT) * 288)) || (rc = nalloc(&W->H, (size_t)(nf3 * nf3))) ||
      (rc = nalloc(&W->b, (size_t)nf3)) || (rc = nalloc(&W->x, (size_t)3 * n)) || (rc = nalloc(&W->g, (size_t)3 * n)) ||
      (rc = nalloc(&W->d, (size_t)3 * n)) || (rc = nalloc(&W->info, 1)))
    return rc;
  QN_CUDA(cudaMemcpy(W->free3, free3.data(), free3.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  QN_CUDA(cudaMemcpy(W->pat_dst, pat_dst.data(), pat_dst.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  QN_CUDA(cudaMemcpy(W->ptr, ptr.data(), ptr.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  if (!src.empty()) QN_CUDA(cudaMemcpy(W->src, src.data(), src.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  QN_CUDA(cudaMemcpy(W->diag_add, diag_add.data(), diag_add.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (cusolverDnCreate(&W->solver) != CUSOLVER_STATUS_SUCCESS) {
    qn::set_error("newton: cusolverDnCreate failed");
    return QN_ERR_CUDA;
  }
  if (cusolverDnDpotrf_bufferSize(W->solver, CUBLAS_FILL_MODE_LOWER, (int)nf3, W->H, (int)nf3, &W->lwork) !=
      CUSOLVER_STATUS_SUCCESS) {
    qn::set_error("newton: potrf workspace query failed");
    return QN_ERR_CUDA;
  }
  if ((rc = nalloc(&W->work, (size_t)W->lwork))) return rc;
  W->nf3 = nf3;
  W->npat = (int64_t)pat_dst.size();
  W->ready = true;
  return QN_OK;
}

}  // namespace

extern "C" {

int qn_newton_direction(qn_system* S, const double* x, const double* grad, double step, double eig_floor, double* d,
                        int32_t mem, void* stream) {
  using namespace qn;
  QN_REQUIRE(S && x && grad && d && step > 0, QN_ERR_ARG, "newton_direction: args");
  QN_REQUIRE(S->n_inst == 1, QN_ERR_UNSUPPORTED, "newton_direction: one instance");
  QN_REQUIRE(S->v.n_col == 0, QN_ERR_UNSUPPORTED, "newton_direction: colliders are not supported");
  NewtonWork* W = work_of(S);
  int rc;
  if (!W->ready && (rc = newton_setup(S, W))) return rc;
  cudaStream_t st = stream ? (cudaStream_t)stream : S->stream;
  const int64_t n3 = 3 * S->n, nf3 = W->nf3;
  const cudaMemcpyKind h2d = mem == QN_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  QN_CUDA(cudaMemcpyAsync(W->x, x, n3 * sizeof(double), h2d, st));
  QN_CUDA(cudaMemcpyAsync(W->g, grad, n3 * sizeof(double), h2d, st));
  if (S->mt > 0) {
    k_newton_blocks<<<div_up(S->mt, kNT), kNT, 0, st>>>(S->v, W->x, step, eig_floor, W->He, W->scratch);
    QN_CHECK_LAUNCH();
  }
  QN_CUDA(cudaMemsetAsync(W->H, 0, (size_t)nf3 * nf3 * sizeof(double), st));
  k_newton_assemble<<<div_up(W->npat, 256), 256, 0, st>>>(W->npat, W->pat_dst, W->ptr, W->src, W->He, W->diag_add,
                                                           W->H);
  QN_CHECK_LAUNCH();
  k_newton_rhs<<<div_up(nf3, 256), 256, 0, st>>>((int)nf3, W->free3, W->g, W->b);
  QN_CHECK_LAUNCH();
  cusolverDnSetStream(W->solver, st);
  if (cusolverDnDpotrf(W->solver, CUBLAS_FILL_MODE_LOWER, (int)nf3, W->H, (int)nf3, W->work, W->lwork, W->info) !=
      CUSOLVER_STATUS_SUCCESS) {
    set_error("newton: potrf failed to launch");
    return QN_ERR_CUDA;
  }
  int info = 0;
  QN_CUDA(cudaMemcpyAsync(&info, W->info, sizeof(int), cudaMemcpyDeviceToHost, st));
  QN_CUDA(cudaStreamSynchronize(st));
  if (info != 0) {
    set_error("newton: Hessian is not positive definite");
    return QN_ERR_NOT_SPD;
  }
  if (cusolverDnDpotrs(W->solver, CUBLAS_FILL_MODE_LOWER, (int)nf3, 1, W->H, (int)nf3, W->b, (int)nf3, W->info) !=
      CUSOLVER_STATUS_SUCCESS) {
    set_error("newton: potrs failed to launch");
    return QN_ERR_CUDA;
  }
  QN_CUDA(cudaMemsetAsync(W->d, 0, n3 * sizeof(double), st));
  k_newton_put<<<div_up(nf3, 256), 256, 0, st>>>((int)nf3, W->free3, W->b, W->d);
  QN_CHECK_LAUNCH();
  QN_CUDA(cudaMemcpyAsync(d, W->d, n3 * sizeof(double),
                          mem == QN_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  QN_CUDA(cudaStreamSynchronize(st));
  return QN_OK;
}

// rest-pose Hessian (solvers.py:401-407): the Newton Hessian at the rest
// positions with y = rest, Cholesky-factored and inverted once; the frame's
// direction step then applies the dense inverse (k_rest_apply)
int qn_system_rest_hessian(qn_system* S, const double* rest, double step, double eig_floor) {
  using namespace qn;
  QN_REQUIRE(S && rest && step > 0, QN_ERR_ARG, "rest_hessian: args");
  QN_REQUIRE(S->n_inst == 1 && S->v.n_col == 0, QN_ERR_UNSUPPORTED, "rest_hessian: single instance, no colliders");
  NewtonWork* W = work_of(S);
  int rc;
  if (!W->ready && (rc = newton_setup(S, W))) return rc;
  QN_REQUIRE(W->nf3 <= 20000, QN_ERR_UNSUPPORTED, "rest_hessian: dense inverse limited to 20000 free dofs");
  cudaStream_t st = S->stream;
  const int64_t n3 = 3 * S->n, nf3 = W->nf3;
  QN_CUDA(cudaMemcpyAsync(W->x, rest, n3 * sizeof(double), cudaMemcpyHostToDevice, st));
  if (S->mt > 0) {
    k_newton_blocks<<<div_up(S->mt, kNT), kNT, 0, st>>>(S->v, W->x, step, eig_floor, W->He, W->scratch);
    QN_CHECK_LAUNCH();
  }
  QN_CUDA(cudaMemsetAsync(W->H, 0, (size_t)nf3 * nf3 * sizeof(double), st));
  k_newton_assemble<<<div_up(W->npat, 256), 256, 0, st>>>(W->npat, W->pat_dst, W->ptr, W->src, W->He, W->diag_add,
                                                           W->H);
  QN_CHECK_LAUNCH();
  cusolverDnSetStream(W->solver, st);
  if (cusolverDnDpotrf(W->solver, CUBLAS_FILL_MODE_LOWER, (int)nf3, W->H, (int)nf3, W->work, W->lwork, W->info) !=
      CUSOLVER_STATUS_SUCCESS) {
    set_error("rest_hessian: potrf failed to launch");
    return QN_ERR_CUDA;
  }
  int info = 0;
  QN_CUDA(cudaMemcpyAsync(&info, W->info, sizeof(int), cudaMemcpyDeviceToHost, st));
  QN_CUDA(cudaStreamSynchronize(st));
  if (info != 0) {
    set_error("rest_hessian: Hessian is not positive definite");
    return QN_ERR_NOT_SPD;
  }
  // inverse: solve against the identity (column-major == row-major for the symmetric result)
  double* inv;
  if ((rc = nalloc(&inv, (size_t)(nf3 * nf3)))) return rc;
  S->allocs.push_back(inv);
  std::vector<double> eye((size_t)nf3 * nf3, 0.0);
  for (int64_t k = 0; k < nf3; ++k) eye[(size_t)k * nf3 + k] = 1.0;
  QN_CUDA(cudaMemcpy(inv, eye.data(), eye.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (cusolverDnDpotrs(W->solver, CUBLAS_FILL_MODE_LOWER, (int)nf3, (int)nf3, W->H, (int)nf3, inv, (int)nf3,
                       W->info) != CUSOLVER_STATUS_SUCCESS) {
    set_error("rest_hessian: potrs failed to launch");
    return QN_ERR_CUDA;
  }
  QN_CUDA(cudaStreamSynchronize(st));
  double* qb;
  if ((rc = nalloc(&qb, (size_t)nf3))) return rc;
  S->allocs.push_back(qb);
  S->v.hrest_inv = inv;
  S->v.qbuf = qb;
  S->v.free3 = W->free3;
  S->v.nf3 = (int32_t)nf3;
  if (S->exec) {  // views changed: rebuild the frame graph
    cudaGraphExecDestroy(S->exec);
    S->exec = nullptr;
    cudaGraphDestroy(S->graph);
    S->graph = nullptr;
  }
  return QN_OK;
}

int qn_newton_release(qn_system* S) {
  std::lock_guard<std::mutex> lock(g_newton_mu);
  for (size_t i = 0; i < g_newton.size(); ++i)
    if (g_newton[i].first == S) {
      NewtonWork* W = g_newton[i].second;
      for (void* p : {(void*)W->free3, (void*)W->pat_dst, (void*)W->ptr, (void*)W->src, (void*)W->diag_add,
                      (void*)W->He, (void*)W->scratch, (void*)W->H, (void*)W->b, (void*)W->x, (void*)W->g,
                      (void*)W->d, (void*)W->work, (void*)W->info})
        if (p) cudaFree(p);
      if (W->solver) cusolverDnDestroy(W->solver);
      delete W;
      g_newton.erase(g_newton.begin() + i);
      break;
    }
  return QN_OK;
}

}  // extern "C"

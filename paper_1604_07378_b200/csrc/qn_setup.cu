// Device assembly of the system setup: the per-tet
// difference operators and rest volumes (mesh.py:200-216), the lumped vertex
// masses (mesh.py:178-197), L = sum_t w_t G_t G_t^T (dynamics.py:69-70,
// 387-402) and A_free = (L + M/h^2)[free][:, free] (dynamics.py:413) — the
// numpy work of build_system, which dominated the configs[4] build (24 M tets).
//
// Summation orders follow the reference's: masses add the corner shares
// corner-major then element order (the four np.add.at calls), every L entry
// sums its tets' contributions in element order (scipy's COO -> CSR duplicate
// summation); the 3 x 3 inverse is the adjugate over the determinant instead
// of LAPACK's LU, so G (and with it L) agrees with the reference to rounding,
// not bitwise — build_system uses this path for large meshes only.
//
// Pipeline (one thread per tet or per vertex, integer atomics only for counts):
//   k_tetops        G (4 x 3), vol, w G G^T (16) per tet; degenerate-volume check
//   k_count, k_fill incidences per vertex (CUB exclusive scan between them)
//   k_rows          per vertex: slot list sorted by (tet, corner) (so every
//                   later sum is in a fixed order), mass, row length of L
//   k_lrows         CSR columns (sorted) and values of L
//   k_alen, k_afill A_free rows (CUB scan between them)
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "qn_common.cuh"

namespace qn {
namespace {

constexpr int kSetupThreads = 256;
constexpr int kMaxRow = 64;  // neighbours of one vertex (Freudenthal grids: 15)

__global__ void k_tetops(int64_t m, const double* __restrict__ X, const int4* __restrict__ tets,
                         const double* __restrict__ k_of_tet, double* G, double* vols, double* blk, double vol_eps,
                         unsigned long long* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 tv = tets[t];
  const int id[4] = {tv.x, tv.y, tv.z, tv.w};
  double x[4][3];
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 3; ++a) x[k][a] = X[3 * (size_t)id[k] + a];
  double D[3][3];  // Dm[a][j] = (x_{j+1} - x_0)[a]: edge columns
  for (int a = 0; a < 3; ++a)
    for (int j = 0; j < 3; ++j) D[a][j] = x[j + 1][a] - x[0][a];
  const double c00 = D[1][1] * D[2][2] - D[1][2] * D[2][1];
  const double c01 = D[1][2] * D[2][0] - D[1][0] * D[2][2];
  const double c02 = D[1][0] * D[2][1] - D[1][1] * D[2][0];
  const double det = D[0][0] * c00 + D[0][1] * c01 + D[0][2] * c02;
  const double vol = det / 6.0;
  vols[t] = vol;
  if (!(vol >= vol_eps)) atomicMin(bad, (unsigned long long)t);
  const double id_ = 1.0 / det;
  double inv[3][3];  // Dm^-1 = adj(Dm) / det
  inv[0][0] = c00 * id_;
  inv[1][0] = c01 * id_;
  inv[2][0] = c02 * id_;
  inv[0][1] = (D[0][2] * D[2][1] - D[0][1] * D[2][2]) * id_;
  inv[1][1] = (D[0][0] * D[2][2] - D[0][2] * D[2][0]) * id_;
  inv[2][1] = (D[0][1] * D[2][0] - D[0][0] * D[2][1]) * id_;
  inv[0][2] = (D[0][1] * D[1][2] - D[0][2] * D[1][1]) * id_;
  inv[1][2] = (D[0][2] * D[1][0] - D[0][0] * D[1][2]) * id_;
  inv[2][2] = (D[0][0] * D[1][1] - D[0][1] * D[1][0]) * id_;
  double g[4][3];  // G[1:] = Dm^-1, G[0] = -(sum of its rows) (mesh.py:212-215)
  for (int c = 0; c < 3; ++c) {
    g[1][c] = inv[0][c];
    g[2][c] = inv[1][c];
    g[3][c] = inv[2][c];
    g[0][c] = -((inv[0][c] + inv[1][c]) + inv[2][c]);
  }
  for (int k = 0; k < 4; ++k)
    for (int c = 0; c < 3; ++c) G[(size_t)t * 12 + 3 * k + c] = g[k][c];
  const double w = vol * k_of_tet[t];  // dynamics.py:48
  for (int v = 0; v < 4; ++v)
    for (int u = 0; u < 4; ++u)
      blk[(size_t)t * 16 + 4 * v + u] = w * ((g[v][0] * g[u][0] + g[v][1] * g[u][1]) + g[v][2] * g[u][2]);
}

__global__ void k_count(int64_t m, const int4* __restrict__ tets, int32_t* cnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 tv = tets[t];
  atomicAdd(cnt + tv.x, 1);
  atomicAdd(cnt + tv.y, 1);
  atomicAdd(cnt + tv.z, 1);
  atomicAdd(cnt + tv.w, 1);
}

__global__ void k_fill(int64_t m, const int4* __restrict__ tets, const int64_t* __restrict__ ptr, int32_t* cur,
                       int64_t* slots) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 tv = tets[t];
  const int id[4] = {tv.x, tv.y, tv.z, tv.w};
  for (int c = 0; c < 4; ++c) slots[ptr[id[c]] + atomicAdd(cur + id[c], 1)] = 4 * t + c;
}

// per vertex: sort its slots (insertion), mass (corner-major, then element
// order), sorted unique neighbour list length
__global__ void k_rows(int64_t n, const int4* __restrict__ tets, const int64_t* __restrict__ ptr, int64_t* slots,
                       const double* __restrict__ vols, double density, double* masses, int32_t* rowlen, int* err) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t* s = slots + ptr[v];
  const int k = (int)(ptr[v + 1] - ptr[v]);
  for (int i = 1; i < k; ++i) {
    const int64_t key = s[i];
    int j = i - 1;
    while (j >= 0 && s[j] > key) {
      s[j + 1] = s[j];
      --j;
    }
    s[j + 1] = key;
  }
  double mass = 0.0;
  for (int c = 0; c < 4; ++c)  // np.add.at(masses, tets[:, c], share) for c = 0..3
    for (int i = 0; i < k; ++i)
      if ((int)(s[i] & 3) == c) mass += density * vols[s[i] >> 2] / 4.0;
  masses[v] = mass;
  int nb[kMaxRow];
  int cntn = 0;
  for (int i = 0; i < k; ++i) {
    const int4 tv = tets[s[i] >> 2];
    const int id[4] = {tv.x, tv.y, tv.z, tv.w};
    for (int c = 0; c < 4; ++c) {
      const int u = id[c];
      int j = 0;
      while (j < cntn && nb[j] < u) ++j;
      if (j < cntn && nb[j] == u) continue;
      if (cntn == kMaxRow) {
        atomicExch(err, 1);
        rowlen[v] = 0;
        return;
      }
      for (int q = cntn; q > j; --q) nb[q] = nb[q - 1];
      nb[j] = u;
      ++cntn;
    }
  }
  rowlen[v] = k ? cntn : 1;  // an isolated vertex still gets its diagonal (mass check reports it)
}

// CSR of L: sorted columns, each entry the sum of its tets' blocks in element order
__global__ void k_lrows(int64_t n, const int4* __restrict__ tets, const int64_t* __restrict__ ptr,
                        const int64_t* __restrict__ slots, const double* __restrict__ blk,
                        const int64_t* __restrict__ lptr, int32_t* lcol, double* lval) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t* s = slots + ptr[v];
  const int k = (int)(ptr[v + 1] - ptr[v]);
  int32_t* col = lcol + lptr[v];
  double* val = lval + lptr[v];
  const int len = (int)(lptr[v + 1] - lptr[v]);
  int cntn = 0;
  for (int i = 0; i < k; ++i) {  // the same sorted unique list as k_rows
    const int4 tv = tets[s[i] >> 2];
    const int id[4] = {tv.x, tv.y, tv.z, tv.w};
    for (int c = 0; c < 4; ++c) {
      const int u = id[c];
      int j = 0;
      while (j < cntn && col[j] < u) ++j;
      if (j < cntn && col[j] == u) continue;
      for (int q = cntn; q > j; --q) col[q] = col[q - 1];
      col[j] = u;
      ++cntn;
    }
  }
  if (k == 0) col[cntn++] = (int32_t)v;
  for (int j = 0; j < len; ++j) val[j] = 0.0;
  for (int i = 0; i < k; ++i) {  // element order
    const int64_t t = s[i] >> 2;
    const int cv = (int)(s[i] & 3);
    const int4 tv = tets[t];
    const int id[4] = {tv.x, tv.y, tv.z, tv.w};
    for (int cu = 0; cu < 4; ++cu) {
      int j = 0;
      while (col[j] != id[cu]) ++j;
      val[j] += blk[(size_t)t * 16 + 4 * cv + cu];
    }
  }
}

// A_free row lengths, then columns (re-indexed, still sorted) and values L + M/h^2
__global__ void k_alen(int64_t n, const int32_t* __restrict__ newid, const int64_t* __restrict__ lptr,
                       const int32_t* __restrict__ lcol, int32_t* alen) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || newid[v] < 0) return;
  int c = 0;
  for (int64_t p = lptr[v]; p < lptr[v + 1]; ++p) c += newid[lcol[p]] >= 0;
  alen[newid[v]] = c;
}

__global__ void k_afill(int64_t n, const int32_t* __restrict__ newid, const int64_t* __restrict__ lptr,
                        const int32_t* __restrict__ lcol, const double* __restrict__ lval,
                        const double* __restrict__ masses, double inv_h2, const int64_t* __restrict__ aptr,
                        int32_t* acol, double* aval) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || newid[v] < 0) return;
  int64_t o = aptr[newid[v]];
  for (int64_t p = lptr[v]; p < lptr[v + 1]; ++p) {
    const int u = lcol[p];
    if (newid[u] < 0) continue;
    acol[o] = newid[u];
    aval[o] = u == v ? lval[p] + masses[v] * inv_h2 : lval[p];  // (L + diags(m / h^2)), dynamics.py:413
    ++o;
  }
}

template <class T>
int exclusive_scan(const T* in, int64_t* out, int64_t count) {  // out[0..count]
  void* tmp = nullptr;
  size_t bytes = 0;
  QN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, count));
  QN_CUDA(cudaMalloc(&tmp, bytes));
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, count);
  cudaFree(tmp);
  QN_CUDA(e);
  return QN_OK;
}

}  // namespace
}  // namespace qn

struct qn_setup {
  int64_t n = 0, m = 0, nf = 0, nnz_l = 0, nnz_a = 0;
  double *G = nullptr, *vols = nullptr, *masses = nullptr, *lval = nullptr, *aval = nullptr;
  int64_t *lptr = nullptr, *aptr = nullptr;
  int32_t *lcol = nullptr, *acol = nullptr;
};

namespace {
template <class T>
int dalloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    qn::set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return QN_ERR_ALLOC;
  }
  return QN_OK;
}
void setup_free(qn_setup* s) {
  void* p[] = {s->G, s->vols, s->masses, s->lval, s->aval, s->lptr, s->aptr, s->lcol, s->acol};
  for (void* q : p)
    if (q) cudaFree(q);
}
}  // namespace

extern "C" {

int qn_setup_create(int64_t n, const double* verts, int64_t m, const int32_t* tets, double density,
                    const double* k_of_tet, double h, int64_t n_fixed, const int32_t* fixed, double vol_eps,
                    qn_setup** out) {
  using namespace qn;
  QN_REQUIRE(n > 0 && m > 0 && verts && tets && k_of_tet && out && h > 0 && m < ((int64_t)1 << 40), QN_ERR_ARG,
             "setup: args");
  for (int64_t i = 0; i < n_fixed; ++i)
    QN_REQUIRE(fixed[i] >= 0 && fixed[i] < n, QN_ERR_ARG, "setup: fixed vertex out of range");
  qn_setup* S = new qn_setup();
  S->n = n;
  S->m = m;
  double *dX = nullptr, *dk = nullptr, *blk = nullptr;
  int4* dT = nullptr;
  int32_t *cnt = nullptr, *rowlen = nullptr, *newid = nullptr, *alen = nullptr;
  int64_t *ptr = nullptr, *slots = nullptr;
  unsigned long long* bad = nullptr;
  int* err = nullptr;
  int rc = QN_OK;
  auto fail = [&](int r) {
    void* p[] = {dX, dk, blk, dT, cnt, rowlen, newid, alen, ptr, slots, bad, err};
    for (void* q : p)
      if (q) cudaFree(q);
    if (r) {
      setup_free(S);
      delete S;
    }
    return r;
  };
  const unsigned gt = (unsigned)((m + kSetupThreads - 1) / kSetupThreads);
  const unsigned gv = (unsigned)((n + kSetupThreads - 1) / kSetupThreads);
  if ((rc = dalloc(&dX, n * 3)) || (rc = dalloc(&dT, m)) || (rc = dalloc(&dk, m)) || (rc = dalloc(&blk, m * 16)) ||
      (rc = dalloc(&S->G, m * 12)) || (rc = dalloc(&S->vols, m)) || (rc = dalloc(&S->masses, n)) ||
      (rc = dalloc(&cnt, n)) || (rc = dalloc(&ptr, n + 1)) || (rc = dalloc(&slots, 4 * m)) ||
      (rc = dalloc(&rowlen, n)) || (rc = dalloc(&S->lptr, n + 1)) || (rc = dalloc(&bad, 1)) ||
      (rc = dalloc(&err, 1)) || (rc = dalloc(&newid, n)))
    return fail(rc);
  if (cudaMemcpy(dX, verts, sizeof(double) * n * 3, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(dT, tets, sizeof(int4) * m, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(dk, k_of_tet, sizeof(double) * m, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(cnt, 0, sizeof(int32_t) * n) != cudaSuccess || cudaMemset(err, 0, sizeof(int)) != cudaSuccess ||
      cudaMemset(bad, 0xff, sizeof(unsigned long long)) != cudaSuccess) {
    set_error("setup: upload failed");
    return fail(QN_ERR_CUDA);
  }
  // tets must index vertices
  {
    const int32_t* tt = tets;
    int32_t lo = tt[0], hi = tt[0];
    for (int64_t i = 0; i < 4 * m; ++i) {
      lo = std::min(lo, tt[i]);
      hi = std::max(hi, tt[i]);
    }
    if (lo < 0 || hi >= n) {
      set_error("setup: tet vertex index out of range");
      return fail(QN_ERR_ARG);
    }
  }
  k_tetops<<<gt, kSetupThreads>>>(m, dX, dT, dk, S->G, S->vols, blk, vol_eps, bad);
  k_count<<<gt, kSetupThreads>>>(m, dT, cnt);
  if ((rc = exclusive_scan(cnt, ptr, n))) return fail(rc);
  // ptr[n] = 4m
  {
    const int64_t tot = 4 * m;
    if (cudaMemcpy(ptr + n, &tot, sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess) return fail(QN_ERR_CUDA);
  }
  QN_CUDA(cudaMemset(cnt, 0, sizeof(int32_t) * n));
  k_fill<<<gt, kSetupThreads>>>(m, dT, ptr, cnt, slots);
  k_rows<<<gv, kSetupThreads>>>(n, dT, ptr, slots, S->vols, density, S->masses, rowlen, err);
  QN_CUDA(cudaGetLastError());
  unsigned long long badt = 0;
  int herr = 0;
  QN_CUDA(cudaMemcpy(&badt, bad, sizeof(badt), cudaMemcpyDeviceToHost));
  QN_CUDA(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost));
  if (badt != ~0ull) {
    set_error("degenerate rest tet in diff-operator construction (tet " + std::to_string(badt) + ")");
    return fail(QN_ERR_ARG);
  }
  if (herr) {
    set_error("setup: a vertex has more than 64 neighbours (device assembly limit)");
    return fail(QN_ERR_UNSUPPORTED);
  }
  if ((rc = exclusive_scan(rowlen, S->lptr, n))) return fail(rc);
  {
    int64_t last = 0;
    int32_t lastlen = 0;
    QN_CUDA(cudaMemcpy(&last, S->lptr + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    QN_CUDA(cudaMemcpy(&lastlen, rowlen + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
    S->nnz_l = last + lastlen;
    QN_CUDA(cudaMemcpy(S->lptr + n, &S->nnz_l, sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  if ((rc = dalloc(&S->lcol, S->nnz_l)) || (rc = dalloc(&S->lval, S->nnz_l))) return fail(rc);
  k_lrows<<<gv, kSetupThreads>>>(n, dT, ptr, slots, blk, S->lptr, S->lcol, S->lval);
  // free-vertex numbering (host: fixed is small)
  {
    std::vector<int32_t> nid(n, 0);
    for (int64_t i = 0; i < n_fixed; ++i) nid[fixed[i]] = -1;
    int32_t c = 0;
    for (int64_t v = 0; v < n; ++v) nid[v] = nid[v] < 0 ? -1 : c++;
    S->nf = c;
    if (c == 0) {
      set_error("all vertices fixed; nothing to simulate");
      return fail(QN_ERR_ARG);
    }
    QN_CUDA(cudaMemcpy(newid, nid.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  }
  if ((rc = dalloc(&alen, S->nf)) || (rc = dalloc(&S->aptr, S->nf + 1))) return fail(rc);
  k_alen<<<gv, kSetupThreads>>>(n, newid, S->lptr, S->lcol, alen);
  if ((rc = exclusive_scan(alen, S->aptr, S->nf))) return fail(rc);
  {
    int64_t last = 0;
    int32_t lastlen = 0;
    QN_CUDA(cudaMemcpy(&last, S->aptr + S->nf - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    QN_CUDA(cudaMemcpy(&lastlen, alen + S->nf - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
    S->nnz_a = last + lastlen;
    QN_CUDA(cudaMemcpy(S->aptr + S->nf, &S->nnz_a, sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  if ((rc = dalloc(&S->acol, S->nnz_a)) || (rc = dalloc(&S->aval, S->nnz_a))) return fail(rc);
  k_afill<<<gv, kSetupThreads>>>(n, newid, S->lptr, S->lcol, S->lval, S->masses, 1.0 / (h * h), S->aptr, S->acol,
                                 S->aval);
  QN_CUDA(cudaDeviceSynchronize());
  fail(QN_OK);
  *out = S;
  return QN_OK;
}

int qn_setup_sizes(const qn_setup* S, int64_t* nnz_l, int64_t* n_free, int64_t* nnz_a) {
  QN_REQUIRE(S && nnz_l && n_free && nnz_a, QN_ERR_ARG, "setup_sizes: null");
  *nnz_l = S->nnz_l;
  *n_free = S->nf;
  *nnz_a = S->nnz_a;
  return QN_OK;
}

int qn_setup_copy(const qn_setup* S, double* G, double* vols, double* masses, int64_t* l_indptr, int32_t* l_indices,
                  double* l_values, int64_t* a_indptr, int32_t* a_indices, double* a_values) {
  QN_REQUIRE(S, QN_ERR_ARG, "setup_copy: null");
  struct Item {
    void* dst;
    const void* src;
    size_t bytes;
  } items[] = {{G, S->G, sizeof(double) * S->m * 12},          {vols, S->vols, sizeof(double) * S->m},
               {masses, S->masses, sizeof(double) * S->n},        {l_indptr, S->lptr, sizeof(int64_t) * (S->n + 1)},
               {l_indices, S->lcol, sizeof(int32_t) * S->nnz_l},  {l_values, S->lval, sizeof(double) * S->nnz_l},
               {a_indptr, S->aptr, sizeof(int64_t) * (S->nf + 1)}, {a_indices, S->acol, sizeof(int32_t) * S->nnz_a},
               {a_values, S->aval, sizeof(double) * S->nnz_a}};
  for (const Item& it : items)
    if (it.dst) QN_CUDA(cudaMemcpy(it.dst, it.src, it.bytes, cudaMemcpyDeviceToHost));
  return QN_OK;
}

int qn_setup_destroy(qn_setup* S) {
  if (S) {
    setup_free(S);
    delete S;
  }
  return QN_OK;
}

}  // extern "C"

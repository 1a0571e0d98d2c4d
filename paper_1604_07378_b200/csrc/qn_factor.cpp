// Host side of the prefactored solve (replaces linalg.Factorization /
// factorize_spd, linalg.py:23-54, and the dense densify+cho_factor of
// dynamics.py:413-414):
//   1. geometric nested-dissection ordering on the free vertices' rest
//      coordinates (recursive coordinate bisection, vertex separators);
//   2. elimination tree (Liu), postorder, column structures, fundamental
//      supernodes, supernodal tree, parent relative-index maps;
//   3. multifrontal numeric Cholesky per batch instance (OpenMP), then the
//      diagonal blocks are inverted so every device step is a dense
//      mat-vec (no sequential triangular sweeps on the GPU).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "qn_common.cuh"
#include "qn_factor.h"

namespace qn {
namespace {

constexpr int kLeaf = 48;  // ND leaf size (vertices)

struct Graph {
  int64_t n;
  std::vector<int64_t> ptr;
  std::vector<int32_t> adj;  // symmetric adjacency without the diagonal
};

Graph make_graph(int64_t n, const int64_t* indptr, const int32_t* indices) {
  Graph g;
  g.n = n;
  std::vector<int64_t> deg(n, 0);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) {
      const int32_t c = indices[p];
      if (c != r) {
        deg[r]++;
        deg[c]++;
      }
    }
  g.ptr.assign(n + 1, 0);
  for (int64_t r = 0; r < n; ++r) g.ptr[r + 1] = g.ptr[r] + deg[r];
  g.adj.resize(g.ptr[n]);
  std::vector<int64_t> fill(g.ptr.begin(), g.ptr.end() - 1);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) {
      const int32_t c = indices[p];
      if (c != r) {
        g.adj[fill[r]++] = c;
        g.adj[fill[c]++] = (int32_t)r;
      }
    }
  // dedupe (A is given with both triangles)
  std::vector<int64_t> nptr(n + 1, 0);
  int64_t w = 0;
  for (int64_t r = 0; r < n; ++r) {
    auto b = g.adj.begin() + g.ptr[r], e = g.adj.begin() + g.ptr[r + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    nptr[r] = w;
    for (auto it = b; it != u; ++it) g.adj[w++] = *it;
  }
  nptr[n] = w;
  g.adj.resize(w);
  g.ptr.swap(nptr);
  return g;
}

struct ND {
  const Graph& g;
  const double* xyz;
  std::vector<int32_t> side;   // 0 / 1 during a split
  std::vector<int32_t> stamp;  // membership of the current subset
  int32_t next_stamp = 1;
  std::vector<int32_t> order;

  ND(const Graph& g_, const double* c) : g(g_), xyz(c), side(g_.n, 0), stamp(g_.n, 0) {
    order.reserve(g.n);
  }

  void run(std::vector<int32_t> verts) {
    static const int64_t leaf = [] {
      const char* e = std::getenv("QN_ND_LEAF");
      return e ? std::max<int64_t>(8, std::atoll(e)) : (int64_t)kLeaf;
    }();
    if ((int64_t)verts.size() <= leaf) {
      std::sort(verts.begin(), verts.end());
      order.insert(order.end(), verts.begin(), verts.end());
      return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int32_t v : verts)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], xyz[3 * v + a]);
        hi[a] = std::max(hi[a], xyz[3 * v + a]);
      }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
      if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
    std::stable_sort(verts.begin(), verts.end(),
                     [&](int32_t a, int32_t b) { return xyz[3 * a + ax] < xyz[3 * b + ax]; });
    const int64_t n = (int64_t)verts.size();
    // split at the widest coordinate gap near the median (clean grid planes)
    const int64_t mid = n / 2, win = std::max<int64_t>(1, n / 8);
    int64_t best = mid;
    double best_gap = -1.0;
    for (int64_t p = std::max<int64_t>(1, mid - win); p <= std::min<int64_t>(n - 1, mid + win); ++p) {
      const double gap = xyz[3 * verts[p] + ax] - xyz[3 * verts[p - 1] + ax];
      const bool closer = std::llabs(p - mid) < std::llabs(best - mid);
      if (gap > best_gap * (1.0 + 1e-6) || (gap >= best_gap * (1.0 - 1e-6) && closer)) {
        best_gap = gap;
        best = p;
      }
    }
    const int32_t st = next_stamp++;
    for (int64_t p = 0; p < n; ++p) {
      stamp[verts[p]] = st;
      side[verts[p]] = p < best ? 0 : 1;
    }
    std::vector<int32_t> sepL, sepR;
    for (int64_t p = 0; p < n; ++p) {
      const int32_t v = verts[p];
      bool cut = false;
      for (int64_t q = g.ptr[v]; q < g.ptr[v + 1] && !cut; ++q) {
        const int32_t u = g.adj[q];
        cut = stamp[u] == st && side[u] != side[v];
      }
      if (cut) (side[v] == 0 ? sepL : sepR).push_back(v);
    }
    std::vector<int32_t>& sep = sepL.size() <= sepR.size() ? sepL : sepR;
    const int32_t sep_side = (&sep == &sepL) ? 0 : 1;
    for (int32_t v : sep) side[v] = 2;
    std::vector<int32_t> A, B;
    A.reserve(best);
    B.reserve(n - best);
    for (int32_t v : verts) {
      if (side[v] == 0) A.push_back(v);
      else if (side[v] == 1) B.push_back(v);
    }
    (void)sep_side;
    std::vector<int32_t> S = sep;
    std::sort(S.begin(), S.end());
    if (A.empty() || B.empty()) {  // degenerate split: stop recursing
      std::sort(verts.begin(), verts.end());
      order.insert(order.end(), verts.begin(), verts.end());
      return;
    }
    run(std::move(A));
    run(std::move(B));
    order.insert(order.end(), S.begin(), S.end());
  }
};

// permuted symmetric pattern with value indices: rows of the new ordering
struct PermCSR {
  std::vector<int64_t> ptr;
  std::vector<int32_t> col;
  std::vector<int64_t> vidx;  // index into the original values array
};

PermCSR permute(int64_t n, const int64_t* indptr, const int32_t* indices, const std::vector<int32_t>& iperm) {
  PermCSR P;
  P.ptr.assign(n + 1, 0);
  std::vector<int32_t> old_of(n);
  for (int64_t i = 0; i < n; ++i) old_of[iperm[i]] = (int32_t)i;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = old_of[i];
    P.ptr[i + 1] = P.ptr[i] + (indptr[r + 1] - indptr[r]);
  }
  P.col.resize(P.ptr[n]);
  P.vidx.resize(P.ptr[n]);
  std::vector<std::pair<int32_t, int64_t>> tmp;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = old_of[i];
    tmp.clear();
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) tmp.emplace_back(iperm[indices[p]], p);
    std::sort(tmp.begin(), tmp.end());
    int64_t w = P.ptr[i];
    for (auto& t : tmp) {
      P.col[w] = t.first;
      P.vidx[w] = t.second;
      ++w;
    }
  }
  return P;
}

std::vector<int32_t> etree(int64_t n, const PermCSR& P) {
  std::vector<int32_t> parent(n, -1), anc(n, -1);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = P.ptr[i]; p < P.ptr[i + 1]; ++p) {
      int32_t r = P.col[p];
      if (r >= i) continue;
      while (anc[r] != -1 && anc[r] != i) {
        const int32_t nx = anc[r];
        anc[r] = (int32_t)i;
        r = nx;
      }
      if (anc[r] == -1) {
        anc[r] = (int32_t)i;
        parent[r] = (int32_t)i;
      }
    }
  }
  return parent;
}

std::vector<int32_t> postorder(int64_t n, const std::vector<int32_t>& parent) {
  std::vector<int32_t> head(n, -1), next(n, -1), post;
  post.reserve(n);
  // children lists in increasing order: insert in decreasing order at head
  for (int64_t j = n - 1; j >= 0; --j)
    if (parent[j] >= 0) {
      next[j] = head[parent[j]];
      head[parent[j]] = (int32_t)j;
    }
  std::vector<int32_t> stack;
  for (int64_t root = 0; root < n; ++root) {
    if (parent[root] != -1) continue;
    stack.push_back((int32_t)root);
    while (!stack.empty()) {
      const int32_t v = stack.back();
      if (head[v] != -1) {
        const int32_t c = head[v];
        head[v] = next[c];
        stack.push_back(c);
      } else {
        stack.pop_back();
        post.push_back(v);
      }
    }
  }
  return post;
}

}  // namespace

int factor_build_host(qn_factor* f, int64_t n, const int64_t* indptr, const int32_t* indices,
                      const double* values, int64_t nbatch, const double* coords) {
  QN_REQUIRE(n > 0 && indptr && indices && values && nbatch >= 1, QN_ERR_ARG, "factor: bad arguments");
  const auto t0 = std::chrono::steady_clock::now();
  f->n = n;
  f->nnz_a = indptr[n];
  f->nbatch = nbatch;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p)
      QN_REQUIRE(indices[p] >= 0 && indices[p] < n, QN_ERR_ARG, "factor: column index out of range");

  // ---- 1. ordering ----
  Graph g = make_graph(n, indptr, indices);
  std::vector<int32_t> order;
  if (coords) {
    ND nd(g, coords);
    std::vector<int32_t> all(n);
    std::iota(all.begin(), all.end(), 0);
    nd.run(std::move(all));
    order.swap(nd.order);
  } else {
    order.resize(n);
    std::iota(order.begin(), order.end(), 0);
  }
  std::vector<int32_t> iperm(n);
  for (int64_t i = 0; i < n; ++i) iperm[order[i]] = (int32_t)i;

  // ---- 2. etree + postorder (relabel) ----
  PermCSR P = permute(n, indptr, indices, iperm);
  std::vector<int32_t> par = etree(n, P);
  std::vector<int32_t> post = postorder(n, par);
  {
    std::vector<int32_t> order2(n);
    for (int64_t k = 0; k < n; ++k) order2[k] = order[post[k]];
    order.swap(order2);
    for (int64_t i = 0; i < n; ++i) iperm[order[i]] = (int32_t)i;
    P = permute(n, indptr, indices, iperm);
    par = etree(n, P);
  }
  f->perm = order;
  f->iperm = iperm;

  // column structures of L (lower), children before parents
  std::vector<std::vector<int32_t>> cs(n);
  std::vector<std::vector<int32_t>> kids(n);
  for (int64_t j = 0; j < n; ++j)
    if (par[j] >= 0) kids[par[j]].push_back((int32_t)j);
  std::vector<int32_t> mark(n, -1);
  std::vector<int64_t> cnt(n);
  for (int64_t j = 0; j < n; ++j) {
    std::vector<int32_t> s;
    s.push_back((int32_t)j);
    mark[j] = (int32_t)j;
    for (int64_t p = P.ptr[j]; p < P.ptr[j + 1]; ++p) {
      const int32_t i = P.col[p];
      if (i > j && mark[i] != j) {
        mark[i] = (int32_t)j;
        s.push_back(i);
      }
    }
    for (int32_t c : kids[j]) {
      for (int32_t i : cs[c])
        if (i > j && mark[i] != j) {
          mark[i] = (int32_t)j;
          s.push_back(i);
        }
    }
    std::sort(s.begin(), s.end());
    cnt[j] = (int64_t)s.size();
    cs[j].swap(s);
    // children structures are no longer needed once the parent is known,
    // except as the first column of a supernode (kept below)
  }

  // ---- fundamental supernodes, then relaxed amalgamation ----
  // A fundamental supernode continues while parent(j-1) = j and the column
  // counts nest exactly.  Chains are then merged bottom-up into the next
  // supernode when it is the etree parent (contiguous columns), if the
  // explicit zeros stay small (thresholds as in the classic relaxed
  // supernode heuristic: always below 4 columns, <= 80% zeros below 16,
  // <= 10% below 48, <= 5% otherwise).  Fewer, larger supernodes mean a
  // shallower device dependency tree and dense mat-vecs of useful size.
  std::vector<int32_t> fcol;  // fundamental supernode first columns
  for (int64_t j = 0; j < n; ++j) {
    const bool start = j == 0 || !(par[j - 1] == j && cnt[j - 1] == cnt[j] + 1);
    if (start) fcol.push_back((int32_t)j);
  }
  const int32_t nf = (int32_t)fcol.size();
  fcol.push_back((int32_t)n);
  std::vector<int32_t> fsup_of(n);
  for (int32_t s = 0; s < nf; ++s)
    for (int32_t j = fcol[s]; j < fcol[s + 1]; ++j) fsup_of[j] = s;
  auto fparent = [&](int32_t s) {
    const int32_t pc = par[fcol[s + 1] - 1];
    return pc >= 0 ? fsup_of[pc] : -1;
  };
  auto below = [&](int32_t s) {  // rows of the supernode strictly below its columns
    const auto& r = cs[fcol[s]];
    return (int64_t)(r.end() - std::upper_bound(r.begin(), r.end(), fcol[s + 1] - 1));
  };
  f->sup_col.clear();
  std::vector<int32_t> last_f;  // last fundamental supernode of each merged group
  const double relax = [] {      // experiment knob: scales the allowed zero fractions
    const char* e = std::getenv("QN_RELAX_SCALE");
    return e ? std::max(0.0, std::atof(e)) : 1.0;
  }();
  {
    int32_t g0 = 0;       // first fundamental supernode of the open group
    double true_nnz = 0;  // sum of exact column counts of the open group
    for (int32_t s = 0; s < nf; ++s) {
      for (int32_t j = fcol[s]; j < fcol[s + 1]; ++j) true_nnz += (double)cnt[j];
      bool merge = false;
      if (s + 1 < nf && fparent(s) == s + 1) {
        const double ncol = fcol[s + 2] - fcol[g0];
        const double nb = (double)below(s + 1);
        const double merged = ncol * (ncol + 1) / 2 + ncol * nb;
        double tn = true_nnz;
        for (int32_t j = fcol[s + 1]; j < fcol[s + 2]; ++j) tn += (double)cnt[j];
        const double z = (merged - tn) / merged;
        merge = ncol <= 4 || (ncol <= 16 && z <= 0.8) || (ncol <= 48 && z <= 0.1 * relax) || z <= 0.05 * relax;
      }
      if (!merge) {
        f->sup_col.push_back(fcol[g0]);
        last_f.push_back(s);
        g0 = s + 1;
        true_nnz = 0;
      }
    }
  }
  // ---- subtree collapse (single-instance factors) ----
  // The device solve costs about one inter-CTA synchronisation per tree level,
  // so the bottom of the tree is flattened: every subtree of height <=
  // kCollapseHeight whose merged supernode stays small (<= kCollapseCols
  // columns, <= kCollapseGrowth x the Z entries of its parts) becomes ONE
  // supernode (columns contiguous in postorder; its below rows are the
  // subtree root's, by the etree ancestor property).  inv(L11) of the merged
  // block is stored dense, explicit zeros included.
  if (nbatch == 1) {
    // experiment knobs (defaults measured on configs[1..2])
    int32_t collapse_h = kCollapseHeight;
    double collapse_cols = kCollapseCols, collapse_growth = kCollapseGrowth;
    if (const char* e = std::getenv("QN_COLLAPSE_HEIGHT")) collapse_h = std::atoi(e);
    if (const char* e = std::getenv("QN_COLLAPSE_COLS")) collapse_cols = std::atof(e);
    if (const char* e = std::getenv("QN_COLLAPSE_GROWTH")) collapse_growth = std::atof(e);
    const int32_t ng = (int32_t)f->sup_col.size();
    std::vector<int32_t> gcol(f->sup_col);
    gcol.push_back((int32_t)n);
    std::vector<int32_t> gof(n);
    for (int32_t g = 0; g < ng; ++g)
      for (int32_t j = gcol[g]; j < gcol[g + 1]; ++j) gof[j] = g;
    std::vector<int32_t> gpar(ng, -1), ht(ng, 0), gsize(ng, 1);
    std::vector<double> sub_nc(ng), sub_z(ng), below_g(ng);
    for (int32_t g = 0; g < ng; ++g) {
      const int32_t pc = par[gcol[g + 1] - 1];
      gpar[g] = pc >= 0 ? gof[pc] : -1;
      const auto& lr = cs[fcol[last_f[g]]];
      below_g[g] = (double)(lr.end() - std::upper_bound(lr.begin(), lr.end(), gcol[g + 1] - 1));
      const double nc = gcol[g + 1] - gcol[g];
      sub_nc[g] += nc;
      sub_z[g] += nc * (nc + below_g[g]);
    }
    for (int32_t g = 0; g < ng; ++g)  // children precede parents
      if (gpar[g] >= 0) {
        const int32_t p = gpar[g];
        ht[p] = std::max(ht[p], ht[g] + 1);
        sub_nc[p] += sub_nc[g];
        sub_z[p] += sub_z[g];
        gsize[p] += gsize[g];
      }
    std::vector<uint8_t> sel(ng, 0), covered(ng, 0);
    for (int32_t g = ng - 1; g >= 0; --g) {  // parents before children
      const bool pc = gpar[g] >= 0 && covered[gpar[g]];
      const double zm = sub_nc[g] * (sub_nc[g] + below_g[g]);
      const bool ok = gsize[g] > 1 && ht[g] <= collapse_h && sub_nc[g] <= collapse_cols &&
                      zm <= collapse_growth * sub_z[g];
      sel[g] = !pc && ok;
      covered[g] = pc || sel[g];
    }
    std::vector<int32_t> root_at(ng, -1);  // selected subtrees are disjoint: [r - size + 1, r]
    for (int32_t r = 0; r < ng; ++r)
      if (sel[r]) root_at[r - gsize[r] + 1] = r;
    std::vector<int32_t> ncol, nlast;
    for (int32_t g = 0; g < ng;) {
      const int32_t end = root_at[g] >= 0 ? root_at[g] : g;
      ncol.push_back(gcol[g]);
      nlast.push_back(last_f[end]);
      g = end + 1;
    }
    f->sup_col.swap(ncol);
    last_f.swap(nlast);
  }
  std::vector<int32_t> sup_of(n);
  for (size_t s = 0; s < f->sup_col.size(); ++s) {
    const int32_t c1 = s + 1 < f->sup_col.size() ? f->sup_col[s + 1] : (int32_t)n;
    for (int32_t j = f->sup_col[s]; j < c1; ++j) sup_of[j] = (int32_t)s;
  }
  f->nsup = (int32_t)f->sup_col.size();
  f->sup_col.push_back((int32_t)n);
  const int32_t ns = f->nsup;
  f->sup_row_ptr.assign(ns + 1, 0);
  f->sup_val_ptr.assign(ns + 1, 0);
  f->sup_upd_ptr.assign(ns + 1, 0);
  f->parent.assign(ns, -1);
  f->max_rows = 0;
  f->nnz_l = 0;
  std::vector<std::vector<int32_t>> rows_of(ns);
  for (int32_t s = 0; s < ns; ++s) {
    const int32_t c0 = f->sup_col[s], c1 = f->sup_col[s + 1];
    auto& r = rows_of[s];
    for (int32_t j = c0; j < c1; ++j) r.push_back(j);
    const auto& lr = cs[fcol[last_f[s]]];
    for (auto it = std::upper_bound(lr.begin(), lr.end(), c1 - 1); it != lr.end(); ++it) r.push_back(*it);
  }
  for (int32_t s = 0; s < ns; ++s) {
    const int32_t c0 = f->sup_col[s], c1 = f->sup_col[s + 1];
    const int64_t nc = c1 - c0, nr = (int64_t)rows_of[s].size();
    f->sup_row_ptr[s + 1] = f->sup_row_ptr[s] + nr;
    f->sup_val_ptr[s + 1] = f->sup_val_ptr[s] + nc * nc + (nr - nc) * nc;
    f->sup_upd_ptr[s + 1] = f->sup_upd_ptr[s] + (nr - nc);
    f->max_rows = std::max<int32_t>(f->max_rows, (int32_t)nr);
    f->nnz_l += nc * (nc + 1) / 2 + (nr - nc) * nc;
    const int32_t pc = par[c1 - 1];
    f->parent[s] = pc >= 0 ? sup_of[pc] : -1;
  }
  f->sup_rows.resize(f->sup_row_ptr[ns]);
  for (int32_t s = 0; s < ns; ++s)
    std::copy(rows_of[s].begin(), rows_of[s].end(), f->sup_rows.begin() + f->sup_row_ptr[s]);
  std::vector<std::vector<int32_t>>().swap(cs);
  std::vector<std::vector<int32_t>>().swap(rows_of);
  f->nvals = f->sup_val_ptr[ns];
  f->nupd = f->sup_upd_ptr[ns];

  // children lists + relative maps (child's below rows -> parent positions)
  f->child_ptr.assign(ns + 1, 0);
  for (int32_t s = 0; s < ns; ++s)
    if (f->parent[s] >= 0) f->child_ptr[f->parent[s] + 1]++;
  for (int32_t s = 0; s < ns; ++s) f->child_ptr[s + 1] += f->child_ptr[s];
  f->child_idx.resize(f->child_ptr[ns]);
  {
    std::vector<int32_t> fill(f->child_ptr.begin(), f->child_ptr.end() - 1);
    for (int32_t s = 0; s < ns; ++s)
      if (f->parent[s] >= 0) f->child_idx[fill[f->parent[s]]++] = s;
  }
  f->rel_ptr.assign(ns + 1, 0);
  for (int32_t s = 0; s < ns; ++s) {
    const int64_t nc = f->sup_col[s + 1] - f->sup_col[s];
    const int64_t nr = f->sup_row_ptr[s + 1] - f->sup_row_ptr[s];
    f->rel_ptr[s + 1] = f->rel_ptr[s] + (f->parent[s] >= 0 ? nr - nc : 0);
  }
  f->rel.resize(f->rel_ptr[ns]);
  {
    std::vector<int32_t> pos(n, -1);
    for (int32_t p = 0; p < ns; ++p) {
      const int64_t pr0 = f->sup_row_ptr[p], pr1 = f->sup_row_ptr[p + 1];
      for (int64_t k = pr0; k < pr1; ++k) pos[f->sup_rows[k]] = (int32_t)(k - pr0);
      for (int32_t q = f->child_ptr[p]; q < f->child_ptr[p + 1]; ++q) {
        const int32_t c = f->child_idx[q];
        const int64_t nc = f->sup_col[c + 1] - f->sup_col[c];
        const int64_t r0 = f->sup_row_ptr[c] + nc, r1 = f->sup_row_ptr[c + 1];
        for (int64_t k = r0; k < r1; ++k) {
          const int32_t pp = pos[f->sup_rows[k]];
          QN_REQUIRE(pp >= 0, QN_ERR_ARG, "factor: symbolic structure inconsistency");
          f->rel[f->rel_ptr[c] + (k - r0)] = pp;
        }
      }
    }
  }
  // extend-add as a pull: for every front position p of supernode s, the list
  // of children's update rows landing there (child order = deterministic)
  {
    const int64_t tot_rows = f->sup_row_ptr[ns];
    std::vector<int32_t> cnt_p(tot_rows, 0);
    for (int32_t s = 0; s < ns; ++s)
      for (int32_t q = f->child_ptr[s]; q < f->child_ptr[s + 1]; ++q) {
        const int32_t c = f->child_idx[q];
        for (int64_t i = f->rel_ptr[c]; i < f->rel_ptr[c + 1]; ++i) cnt_p[f->sup_row_ptr[s] + f->rel[i]]++;
      }
    f->cptr.assign(tot_rows + 1, 0);
    for (int64_t p = 0; p < tot_rows; ++p) f->cptr[p + 1] = f->cptr[p] + cnt_p[p];
    f->cidx.resize(f->cptr[tot_rows]);
    std::vector<int64_t> fill(f->cptr.begin(), f->cptr.end() - 1);
    for (int32_t s = 0; s < ns; ++s)
      for (int32_t q = f->child_ptr[s]; q < f->child_ptr[s + 1]; ++q) {
        const int32_t c = f->child_idx[q];
        for (int64_t i = f->rel_ptr[c]; i < f->rel_ptr[c + 1]; ++i)
          f->cidx[fill[f->sup_row_ptr[s] + f->rel[i]]++] = (int32_t)(f->sup_upd_ptr[c] + (i - f->rel_ptr[c]));
      }
  }
  // device work items: forward = row blocks of Z per supernode (postorder),
  // backward = column blocks (reverse postorder)
  // Ticket order = level order: forward by height above the leaves, backward
  // by depth below the root.  Tasks that become ready together get adjacent
  // tickets, so resident CTAs are not parked on dependencies while ready work
  // of the same level waits for a slot (a plain postorder serialises subtrees).
  f->ftask.clear();
  f->btask.clear();
  f->fcount.assign(ns, 0);
  f->bcount.assign(ns, 0);
  {
    std::vector<int32_t> height(ns, 0), dep(ns, 0);
    for (int32_t s = 0; s < ns; ++s)
      if (f->parent[s] >= 0) height[f->parent[s]] = std::max(height[f->parent[s]], height[s] + 1);
    for (int32_t s = ns - 1; s >= 0; --s)
      if (f->parent[s] >= 0) dep[s] = dep[f->parent[s]] + 1;
    // Dense top: the top levels of the tree are narrow and strictly serial in
    // both solves.  With T = the supernodes of depth <= d* (closed under
    // ancestors), L_T is the factor of the Schur complement S = A_TT -
    // A_TB A_BB^-1 A_BT, so forward + backward on T collapse into one dense
    // product x_T = S^-1 g_T (g_T = b_T minus the updates of the subtrees
    // hanging below T).  d* = deepest level with |T| <= kTopMax columns.
    f->is_top.assign(ns, 0);
    f->ktop = 0;
    f->tcols.clear();
    if (nbatch == 1) {
      int32_t maxd = 0;
      for (int32_t s = 0; s < ns; ++s) maxd = std::max(maxd, dep[s]);
      std::vector<int64_t> cols_at(maxd + 1, 0), wide_at(maxd + 1, 0);
      for (int32_t s = 0; s < ns; ++s) {
        const int64_t nc = f->sup_col[s + 1] - f->sup_col[s];
        cols_at[dep[s]] += nc;
        wide_at[dep[s]] = std::max(wide_at[dep[s]], nc);
      }
      // Only levels of wide separators go dense: narrow top levels are
      // cheaper as sparse tasks than a K^2 product that also crowds L2
      // (measured: c2 best without a top, c3 best with K ~ 3.8k).
      int64_t top_max = kTopMax, min_wide = kTopMinWidth;  // env: tuning experiments only
      if (const char* e = std::getenv("QN_TOP_MAX")) top_max = std::max<int64_t>(0, std::atoll(e));
      if (const char* e = std::getenv("QN_TOP_MIN_WIDTH")) min_wide = std::max<int64_t>(0, std::atoll(e));
      int32_t dstar = -1;
      int64_t cum = 0;
      for (int32_t d = 0; d <= maxd; ++d) {
        cum += cols_at[d];
        if (cum > top_max || (wide_at[d] < min_wide && n > kTopDenseAll)) break;
        dstar = d;
      }
      if (n <= kTopDenseAll) dstar = maxd;  // small systems: one dense product
      if (dstar >= 0) {
        for (int32_t s = 0; s < ns; ++s) f->is_top[s] = dep[s] <= dstar;
        for (int32_t s = 0; s < ns; ++s)
          if (f->is_top[s])
            for (int32_t c = f->sup_col[s]; c < f->sup_col[s + 1]; ++c) f->tcols.push_back(c);
        f->ktop = (int32_t)f->tcols.size();
      }
    }
    std::vector<int32_t> order(ns);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return height[a] < height[b]; });
    // task size: ~kTaskEntries of Z per task; forward row blocks of 32 rg rows
    // (rg in {1,2,4,8} row groups, 8/rg warps split k), backward 8 cw columns
    // (cw columns per warp)
    auto pow2_floor = [](int64_t v) {
      int64_t p = 1;
      while (p * 2 <= v) p *= 2;
      return (int32_t)p;
    };
    f->ffirst.assign(ns, 0);
    f->bfirst.assign(ns, 0);
    // experiment knobs (<= the compile-time tile bounds)
    auto knob = [](const char* name, int64_t dflt, int64_t hi) {
      const char* e = std::getenv(name);
      return e ? std::max<int64_t>(1, std::min<int64_t>(hi, std::atoll(e))) : dflt;
    };
    const int64_t te_f = knob("QN_FWD_TASK_ENTRIES", kTaskEntries, kTaskEntries);
    const int64_t te_b = knob("QN_BWD_TASK_ENTRIES", kTaskEntries, kTaskEntries);
    const int64_t bcols = knob("QN_BWD_TASK_COLS", kBwdTaskCols, kBwdTaskCols);
    const int64_t fwd_budget = knob("QN_FWD_BUDGET", kFwdBudget, 1 << 20);
    const char* e_bal = std::getenv("QN_FWD_BALANCED");  // experiment knob: 1 = rows split evenly over the fewest tasks
    const bool balanced = e_bal && std::atoi(e_bal) != 0;  // measured: c3 +0.4 %, c2 -1.7 % (the forward is dependency-bound)
    // backward Z tile: as large as kTaskEntries but small enough that two
    // CTAs (each also holding w = nr x 3 of the tallest front) share an SM
    {
      int32_t mr = 0;
      for (int32_t s = 0; s < ns; ++s)
        if (!f->is_top[s]) mr = std::max<int32_t>(mr, (int32_t)(f->sup_row_ptr[s + 1] - f->sup_row_ptr[s]));
      const int64_t rest = 8 * (3 * (int64_t)mr + 4 * kBwdTaskCols) + 4 * 2048;
      const int64_t fit = (kSmemPerCtaPair - rest) / 8;
      f->bwd_entries = std::max<int64_t>(mr, std::min<int64_t>(te_b, fit));
      f->task_max_rows = mr;
    }
    f->fwd_entries = 2;
    for (int32_t s : order) {
      if (f->is_top[s]) continue;
      const int32_t nc = f->sup_col[s + 1] - f->sup_col[s];
      const int32_t nr = (int32_t)(f->sup_row_ptr[s + 1] - f->sup_row_ptr[s]);
      QN_REQUIRE(nc <= kTaskEntries && nr - nc <= (int64_t)1 << 20, QN_ERR_UNSUPPORTED,
                 "factor: supernode too wide for the device solve tiles");
      // a task's shared memory holds its Z tile and f (nc x 3): wide supernodes get
      // smaller tiles so that tile + f stays within kFwdBudget (three CTAs per SM)
      // (only where the forward sweep has its own kernel: the fused forward + backward kernel of
      // factors without a dense top runs two CTAs per SM anyway)
      const int64_t room = fwd_budget - 3 * (int64_t)nc;
      const int64_t te_s = (f->ktop > 0 || nbatch > 1) && room >= 4 * (int64_t)nc ? std::min(te_f, room) : te_f;
      // rows per task: as many as the tile holds (<= 256 = 8 warps x 32 rows), the supernode's rows
      // split evenly over the fewest tasks (a 136-row leaf front is one 5-warp task, not 128 + 8 rows);
      // rg = row groups of 32 rows (power of two: the other 8 / rg warps split k)
      const int64_t rows_cap = std::max<int64_t>(1, std::min<int64_t>(256, te_s / nc));
      const int32_t ntask = (int32_t)((nr + rows_cap - 1) / rows_cap);
      const int32_t rows = balanced ? (nr + ntask - 1) / ntask
                                    : (rows_cap >= 32 ? 32 * pow2_floor(rows_cap / 32) : (int32_t)rows_cap);
      int32_t rg = 1;
      while (32 * rg < rows) rg *= 2;
      f->ffirst[s] = (int32_t)f->ftask.size();
      for (int32_t r = 0; r < nr; r += rows) {
        const int32_t hi = std::min(nr, r + rows);
        f->fwd_entries =
            std::max<int64_t>(f->fwd_entries, ((int64_t)(hi - r) * std::min(hi, nc) + 1) / 2 * 2 + 3 * (int64_t)nc);
        f->ftask.push_back({s, r, std::min(nr, r + rows), rg});
        f->fcount[s]++;
      }
    }
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return dep[a] < dep[b]; });
    for (int32_t s : order) {
      if (f->is_top[s]) continue;
      const int32_t nc = f->sup_col[s + 1] - f->sup_col[s];
      const int32_t nr = (int32_t)(f->sup_row_ptr[s + 1] - f->sup_row_ptr[s]);
      QN_REQUIRE(nr <= f->bwd_entries, QN_ERR_UNSUPPORTED, "factor: supernode front too tall for the device tiles");
      const int32_t cols = (int32_t)std::min<int64_t>(bcols, std::max<int64_t>(1, f->bwd_entries / nr));
      f->bfirst[s] = (int32_t)f->btask.size();
      for (int32_t k = 0; k < nc; k += cols) {
        f->btask.push_back({s, k, std::min(nc, k + cols), 0});
        f->bcount[s]++;
      }
    }
    // forward dependencies of s: every task of every child
    f->fdep_ptr.assign(ns + 1, 0);
    for (int32_t s = 0; s < ns; ++s) {
      int32_t cnt = 0;
      for (int32_t q = f->child_ptr[s]; q < f->child_ptr[s + 1]; ++q) cnt += f->fcount[f->child_idx[q]];
      f->fdep_ptr[s + 1] = f->fdep_ptr[s] + cnt;
    }
    f->fdep_idx.resize(f->fdep_ptr[ns]);
    for (int32_t s = 0; s < ns; ++s) {
      int32_t w = f->fdep_ptr[s];
      for (int32_t q = f->child_ptr[s]; q < f->child_ptr[s + 1]; ++q) {
        const int32_t c = f->child_idx[q];
        for (int32_t t = 0; t < f->fcount[c]; ++t) f->fdep_idx[w++] = f->ffirst[c] + t;
      }
    }
    // forward task descriptors + their relative extend-add lists
    f->fdesc.clear();
    f->fblob.clear();
    for (const int4& t : f->ftask) {
      const int32_t s = t.x, lo = t.y, hi = t.z;
      const int32_t c0 = f->sup_col[s], nc = f->sup_col[s + 1] - c0;
      const int64_t R0 = f->sup_row_ptr[s];
      const int32_t nr = (int32_t)(f->sup_row_ptr[s + 1] - R0);
      const int32_t blo = std::max(lo, nc);
      const int64_t ct0 = f->cptr[R0], ct1 = f->cptr[R0 + nc];
      const int64_t cb0 = f->cptr[R0 + blo], cb1 = blo < hi ? f->cptr[R0 + hi] : cb0;
      qn_fdesc d{};
      d.zoff = f->sup_val_ptr[s] + lo;
      d.lo = lo;
      d.hi = hi;
      d.rg = t.w;
      d.c0 = c0;
      d.nc = nc;
      d.nr = nr;
      d.blo = blo;
      d.ntop = (int32_t)(ct1 - ct0);
      d.nbot = (int32_t)(cb1 - cb0);
      d.upd0 = (int32_t)f->sup_upd_ptr[s];
      d.dep0 = f->fdep_ptr[s];
      d.dep1 = f->fdep_ptr[s + 1];
      QN_REQUIRE(f->fblob.size() < (size_t)INT32_MAX && f->nupd < INT32_MAX, QN_ERR_UNSUPPORTED,
                 "factor: solve lists exceed 32-bit offsets");
      d.blob = (int32_t)f->fblob.size();
      for (int32_t p = 0; p <= nc; ++p) f->fblob.push_back((int32_t)(f->cptr[R0 + p] - ct0));
      if (blo < hi)
        for (int32_t p = 0; p <= hi - blo; ++p) f->fblob.push_back((int32_t)(f->cptr[R0 + blo + p] - cb0));
      for (int64_t q = ct0; q < ct1; ++q) f->fblob.push_back(f->cidx[q]);
      for (int64_t q = cb0; q < cb1; ++q) f->fblob.push_back(f->cidx[q]);
      f->fdesc.push_back(d);
    }
    f->bdesc.clear();
    for (const int4& t : f->btask) {
      const int32_t s = t.x;
      const int32_t nc = f->sup_col[s + 1] - f->sup_col[s];
      const int32_t nr = (int32_t)(f->sup_row_ptr[s + 1] - f->sup_row_ptr[s]);
      const int32_t p = f->parent[s];
      qn_bdesc d{};
      d.zoff = f->sup_val_ptr[s] + (int64_t)t.y * nr;
      d.rows = f->sup_row_ptr[s];
      d.k0 = t.y;
      d.k1 = t.z;
      d.c0 = f->sup_col[s];
      d.nc = nc;
      d.nr = nr;
      d.wait0 = p >= 0 ? f->bfirst[p] : 0;
      d.nwait = p >= 0 ? f->bcount[p] : 0;
      d.fwd0 = f->ffirst[s];
      d.nfwd = f->fcount[s];
      d.top_child = (p >= 0 && !f->is_top.empty() && f->is_top[p]) ? 1 : 0;
      f->bdesc.push_back(d);
    }
    // level lists for the batched per-instance solve: forward by height
    // (leaves first), backward by depth (root first); supernodes of one level
    // are independent and run on different warps of the instance's CTA
    {
      int32_t mh = 0, md = 0;
      for (int32_t s = 0; s < ns; ++s) {
        mh = std::max(mh, height[s]);
        md = std::max(md, dep[s]);
      }
      auto bucket = [&](const std::vector<int32_t>& key, int32_t nl, std::vector<int32_t>& ptr,
                        std::vector<int32_t>& list) {
        ptr.assign(nl + 2, 0);
        for (int32_t s = 0; s < ns; ++s) ptr[key[s] + 1]++;
        for (int32_t l = 0; l <= nl; ++l) ptr[l + 1] += ptr[l];
        list.assign(ns, 0);
        std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
        for (int32_t s = 0; s < ns; ++s) list[fill[key[s]]++] = s;
      };
      bucket(height, mh, f->hlev_ptr, f->hlev_sup);
      bucket(dep, md, f->dlev_ptr, f->dlev_sup);
    }
    // g_T gather lists: every non-top supernode whose parent is top passes all
    // of its subtree's updates to top columns in its update vector u_s
    if (f->ktop > 0) {
      std::vector<int32_t> tpos(n, -1);
      for (int32_t k = 0; k < f->ktop; ++k) tpos[f->tcols[k]] = k;
      std::vector<std::vector<int32_t>> lists(f->ktop);
      for (int32_t s = 0; s < ns; ++s) {
        if (f->is_top[s] || f->parent[s] < 0 || !f->is_top[f->parent[s]]) continue;
        const int32_t nc = f->sup_col[s + 1] - f->sup_col[s];
        const int64_t r0 = f->sup_row_ptr[s] + nc, r1 = f->sup_row_ptr[s + 1];
        for (int64_t r = r0; r < r1; ++r) {
          const int32_t k = tpos[f->sup_rows[r]];
          QN_REQUIRE(k >= 0, QN_ERR_ARG, "factor: update row outside the dense top");
          lists[k].push_back((int32_t)(f->sup_upd_ptr[s] + (r - r0)));
        }
      }
      f->tg_ptr.assign(f->ktop + 1, 0);
      for (int32_t k = 0; k < f->ktop; ++k) f->tg_ptr[k + 1] = f->tg_ptr[k] + (int32_t)lists[k].size();
      f->tg_idx.clear();
      for (auto& l : lists) f->tg_idx.insert(f->tg_idx.end(), l.begin(), l.end());
    }
  }
  // tree depth
  {
    std::vector<int32_t> d(ns, 1);
    f->depth = 0;
    for (int32_t s = ns - 1; s >= 0; --s) {
      if (f->parent[s] >= 0) d[s] = d[f->parent[s]] + 1;
      f->depth = std::max(f->depth, d[s]);
    }
  }

  // ---- 3. numeric multifrontal factorisation per batch instance ----
  f->vals.assign((size_t)nbatch * f->nvals, 0.0);
  // lower-triangle entries of each factor column, as (row, value index)
  std::vector<int64_t> lptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = P.ptr[i]; p < P.ptr[i + 1]; ++p)
      if (P.col[p] <= i) lptr[P.col[p] + 1]++;
  for (int64_t j = 0; j < n; ++j) lptr[j + 1] += lptr[j];
  std::vector<int32_t> lrow(lptr[n]);
  std::vector<int64_t> lvi(lptr[n]);
  {
    std::vector<int64_t> fill(lptr.begin(), lptr.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = P.ptr[i]; p < P.ptr[i + 1]; ++p)
        if (P.col[p] <= i) {
          const int64_t q = fill[P.col[p]]++;
          lrow[q] = (int32_t)i;
          lvi[q] = P.vidx[p];
        }
  }
  double flops = 0.0;
  for (int32_t s = 0; s < ns; ++s) {
    const double nc = f->sup_col[s + 1] - f->sup_col[s];
    const double nr = (double)(f->sup_row_ptr[s + 1] - f->sup_row_ptr[s]);
    flops += nc * nc * nc / 3.0 + (nr - nc) * nc * nc + (nr - nc) * (nr - nc) * nc;
  }
  f->flops = flops;

  int err = QN_OK;
  std::string errmsg;
  const bool par_batch = nbatch > 1;
  std::vector<int32_t> ttpos;  // factor column -> top index (dense top only; nbatch == 1)
  std::vector<double> LT;
  if (f->ktop > 0) {
    ttpos.assign(n, -1);
    for (int32_t k = 0; k < f->ktop; ++k) ttpos[f->tcols[k]] = k;
    LT.assign((size_t)f->ktop * f->ktop, 0.0);
  }
#pragma omp parallel for schedule(dynamic, 1) if (par_batch)
  for (int64_t b = 0; b < nbatch; ++b) {
    if (err != QN_OK) continue;
    const double* av = values + (size_t)b * f->nnz_a;
    double* out = f->vals.data() + (size_t)b * f->nvals;
    std::vector<std::vector<double>> upd(ns);
    std::vector<int32_t> pos(n, -1);
    std::vector<double> F;
    for (int32_t s = 0; s < ns; ++s) {
      const int32_t c0 = f->sup_col[s];
      const int64_t nc = f->sup_col[s + 1] - c0;
      const int64_t r0 = f->sup_row_ptr[s];
      const int64_t nr = f->sup_row_ptr[s + 1] - r0;
      const int64_t mb = nr - nc;
      for (int64_t k = 0; k < nr; ++k) pos[f->sup_rows[r0 + k]] = (int32_t)k;
      F.assign((size_t)nr * nr, 0.0);
      // assemble A's columns J_s (lower part)
      for (int64_t jj = 0; jj < nc; ++jj) {
        const int64_t j = c0 + jj;
        for (int64_t q = lptr[j]; q < lptr[j + 1]; ++q) F[pos[lrow[q]] + jj * nr] += av[lvi[q]];
      }
      // extend-add children's update matrices (lower, column-major mc x mc)
      for (int32_t q = f->child_ptr[s]; q < f->child_ptr[s + 1]; ++q) {
        const int32_t c = f->child_idx[q];
        const int64_t mc = f->rel_ptr[c + 1] - f->rel_ptr[c];
        const int32_t* rl = f->rel.data() + f->rel_ptr[c];
        const double* U = upd[c].data();
        for (int64_t jb = 0; jb < mc; ++jb) {
          double* Fc = F.data() + (size_t)rl[jb] * nr;
          for (int64_t ib = jb; ib < mc; ++ib) Fc[rl[ib]] += U[ib + jb * mc];
        }
        std::vector<double>().swap(upd[c]);
      }
      // partial Cholesky of the nc pivot columns (right-looking within the panel)
      for (int64_t k = 0; k < nc; ++k) {
        double* Fk = F.data() + k * nr;
        const double d = Fk[k];
        if (!(d > 0.0) || !std::isfinite(d)) {
#pragma omp critical
          {
            err = QN_ERR_NOT_SPD;
            errmsg = "matrix is not positive definite (pivot " + std::to_string(d) + " at factor column " +
                     std::to_string(c0 + k) + ")";
          }
          break;
        }
        const double l = std::sqrt(d);
        Fk[k] = l;
        const double il = 1.0 / l;
        for (int64_t i = k + 1; i < nr; ++i) Fk[i] *= il;
        for (int64_t j = k + 1; j < nc; ++j) {
          const double a = Fk[j];
          double* Fj = F.data() + j * nr;
          for (int64_t i = j; i < nr; ++i) Fj[i] -= Fk[i] * a;
        }
      }
      if (err != QN_OK) break;
      // Schur complement U = F22 - L21 L21^T (lower), handed to the parent
      if (mb > 0 && f->parent[s] >= 0) {
        std::vector<double>& U = upd[s];
        U.assign((size_t)mb * mb, 0.0);
        for (int64_t jb = 0; jb < mb; ++jb)
          for (int64_t ib = jb; ib < mb; ++ib) U[ib + jb * mb] = F[(nc + ib) + (nc + jb) * nr];
        const bool big = mb * mb * nc > (int64_t)1 << 22 && !par_batch;
#pragma omp parallel for schedule(dynamic, 8) if (big)
        for (int64_t jb = 0; jb < mb; ++jb) {
          double* Uj = U.data() + jb * mb;
          for (int64_t k = 0; k < nc; ++k) {
            const double* Lk = F.data() + k * nr + nc;
            const double a = Lk[jb];
            if (a == 0.0) continue;
            for (int64_t ib = jb; ib < mb; ++ib) Uj[ib] -= Lk[ib] * a;
          }
        }
      }
      // dense top: copy this supernode's columns of L into L_T
      if (f->ktop > 0 && f->is_top[s]) {
        for (int64_t j = 0; j < nc; ++j) {
          const int64_t tj = ttpos[c0 + j];
          for (int64_t i = j; i < nr; ++i) LT[(size_t)ttpos[f->sup_rows[r0 + i]] + (size_t)tj * f->ktop] = F[i + j * nr];
        }
      }
      // store Z = [inv(L11); L21 inv(L11)] (nr x nc, column-major): the forward
      // step of this supernode is then v = Z f (y = top, update = bottom) and
      // the backward step x = Z^T [y; -x_below] — dense, row/column parallel.
      double* Z = out + f->sup_val_ptr[s];
      for (int64_t j = 0; j < nc; ++j) {
        double* Zj = Z + j * nr;
        Zj[j] = 1.0 / F[j + j * nr];
        for (int64_t i = j + 1; i < nc; ++i) {
          double acc = 0.0;
          for (int64_t k = j; k < i; ++k) acc += F[i + k * nr] * Zj[k];
          Zj[i] = -acc / F[i + i * nr];
        }
        double* Wj = Zj + nc;
        for (int64_t ib = 0; ib < mb; ++ib) Wj[ib] = 0.0;
        for (int64_t k = j; k < nc; ++k) {
          const double a = Zj[k];
          const double* Lk = F.data() + k * nr + nc;
          for (int64_t ib = 0; ib < mb; ++ib) Wj[ib] += Lk[ib] * a;
        }
      }
    }
  }
  if (err != QN_OK) {
    set_error(errmsg);
    return err;
  }
  // S^-1 = L_T^-T L_T^-1 (symmetric, stored full, column-major)
  if (f->ktop > 0) {
    const int64_t K = f->ktop;
    std::vector<double> M((size_t)K * K, 0.0);  // L_T^-1 (lower)
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < K; ++j) {  // column j of L_T^-1: solve L_T m = e_j
      double* Mj = M.data() + (size_t)j * K;
      Mj[j] = 1.0;
      for (int64_t k = j; k < K; ++k) {
        const double* Lk = LT.data() + (size_t)k * K;
        Mj[k] /= Lk[k];
        const double mk = Mj[k];
        if (mk != 0.0)
          for (int64_t i = k + 1; i < K; ++i) Mj[i] -= Lk[i] * mk;
      }
    }
    f->sinv.assign((size_t)K * K, 0.0);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < K; ++j) {
      const double* Mj = M.data() + (size_t)j * K;
      for (int64_t i = j; i < K; ++i) {
        const double* Mi = M.data() + (size_t)i * K;
        double acc = 0.0;
        for (int64_t k = i; k < K; ++k) acc += Mi[k] * Mj[k];  // rows >= max(i, j)
        f->sinv[(size_t)i + (size_t)j * K] = acc;
        f->sinv[(size_t)j + (size_t)i * K] = acc;
      }
    }
  }
  f->factor_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return QN_OK;
}

}  // namespace qn

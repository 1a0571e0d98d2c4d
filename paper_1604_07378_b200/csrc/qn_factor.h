// Supernodal Cholesky factor of the constant system matrix A = M/h^2 + L on
// the free DOFs (dynamics.py:413-414), shared by all frames; the device holds
// per supernode s (columns J_s = [col0, col0 + nc), rows R_s, |R_s| = nr):
//   vals[s] = [ inv(L_ss) (nc x nc, column-major) | L_Bs ((nr - nc) x nc, column-major) ]
// and the multifrontal triangular solve exchanges per-supernode update
// vectors u_s (nr - nc rows x 3 RHS) with the parent through `rel` maps.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "qnsim_b200.h"

// Forward solve task descriptor: everything a task needs before its first
// dependent load, in one 64-byte record (one round trip instead of a chain
// task -> supernode -> row pointers -> extend-add lists).
struct alignas(16) qn_fdesc {
  int64_t zoff;                 // Z tile origin: sup_val_ptr[s] + lo
  int32_t lo, hi, rg, c0;       // rows [lo, hi), row groups, first column
  int32_t nc, nr, blo, ntop;    // supernode shape, first bottom row, #top list entries
  int32_t nbot, upd0, dep0, dep1;  // #bottom list entries, update rows offset, fdep range
  int32_t blob, pad;            // offset of [sp_top | sp_bot | si_top | si_bot] in fblob
};

// Backward solve task descriptor (same idea as qn_fdesc).
struct alignas(16) qn_bdesc {
  int64_t zoff;                 // column k0 of Z: sup_val_ptr[s] + k0 nr
  int64_t rows;                 // sup_row_ptr[s] (row ids in sup_rows)
  int32_t k0, k1, c0, nc;
  int32_t nr, wait0, nwait, fwd0;  // parent's backward tasks [wait0, wait0 + nwait); own forward tasks from fwd0
  int32_t nfwd, top_child, pad1, pad2;  // ... nfwd of them (fused kernel); parent is in the dense top
};

struct qn_factor {
  // ---- symbolic (host) ----
  int64_t n = 0, nnz_a = 0, nbatch = 1;
  std::vector<int32_t> perm;      // factor row -> original (free) row
  std::vector<int32_t> iperm;     // original -> factor row
  int32_t nsup = 0;
  std::vector<int32_t> sup_col;   // (nsup+1) first column of each supernode
  std::vector<int64_t> sup_row_ptr;  // (nsup+1) into sup_rows
  std::vector<int32_t> sup_rows;  // R_s (factor row ids), J_s first
  std::vector<int64_t> sup_val_ptr;  // (nsup+1) into vals (per batch)
  std::vector<int64_t> sup_upd_ptr;  // (nsup+1) into the u buffer (rows)
  std::vector<int32_t> parent;    // supernodal etree parent (-1 = root)
  std::vector<int32_t> child_ptr, child_idx;  // children in increasing order
  std::vector<int64_t> rel_ptr;   // (nsup+1) per child: its below rows -> parent front positions
  std::vector<int32_t> rel;
  std::vector<int64_t> cptr;      // (total front rows + 1): pull lists of the extend-add
  std::vector<int32_t> cidx;      // children's update-row ids
  std::vector<int4> ftask, btask; // {supernode, lo, hi, 0}: forward row blocks / backward column blocks
  std::vector<int32_t> fcount, bcount;  // tasks per supernode
  std::vector<int32_t> ffirst, bfirst;  // first task of each supernode
  std::vector<int32_t> fdep_ptr, fdep_idx;  // forward: all tasks of the children of s
  std::vector<qn_fdesc> fdesc;              // per forward task
  std::vector<qn_bdesc> bdesc;              // per backward task
  std::vector<int32_t> fblob;               // per-task relative extend-add lists
  std::vector<int32_t> hlev_ptr, hlev_sup;  // supernodes grouped by height (batched forward levels)
  std::vector<int32_t> dlev_ptr, dlev_sup;  // supernodes grouped by depth (batched backward levels)
  // dense top: the supernodes within the top levels of the tree (K columns)
  // are solved together as x_T = S^-1 g_T, S = Schur complement on T
  std::vector<uint8_t> is_top;
  int32_t ktop = 0;
  std::vector<int32_t> tcols;           // factor column of each top index
  std::vector<int32_t> tg_ptr, tg_idx;  // update rows (of the top's child subtrees) landing on each top column
  std::vector<double> sinv;             // K x K, symmetric (column-major)
  int64_t nvals = 0, nupd = 0, nnz_l = 0;
  int32_t max_rows = 0, depth = 0;
  int32_t task_max_rows = 0;   // tallest front among the supernodes solved by tasks (not the dense top)
  int64_t bwd_entries = 8192;  // Z entries per backward task tile (<= kTaskEntries, set by the task builder)
  int64_t fwd_entries = 8192;  // forward task shared memory in doubles: largest (even tile + f = nc x 3) over the tasks
  double flops = 0.0, factor_seconds = 0.0;
  // ---- numeric (host, nbatch x nvals) ----
  std::vector<double> vals;

  // ---- device ----
  int32_t* d_sup_col = nullptr;
  int64_t* d_sup_row_ptr = nullptr;
  int32_t* d_sup_rows = nullptr;
  int64_t* d_sup_val_ptr = nullptr;
  int64_t* d_sup_upd_ptr = nullptr;
  int32_t* d_parent = nullptr;
  int32_t* d_child_ptr = nullptr;
  int32_t* d_child_idx = nullptr;
  int64_t* d_rel_ptr = nullptr;
  int32_t* d_rel = nullptr;
  int32_t* d_perm = nullptr;      // factor row -> original row
  double* d_vals = nullptr;       // nbatch x nvals
  double* d_y = nullptr;          // nbatch x n x 3 (forward result, factor order)
  double* d_x = nullptr;          // nbatch x n x 3 (backward result, factor order)
  double* d_u = nullptr;          // nbatch x nupd x 3
  int64_t* d_cptr = nullptr;
  int32_t* d_cidx = nullptr;
  int4* d_ftask = nullptr;
  int4* d_btask = nullptr;
  int32_t* d_bfirst = nullptr;
  int32_t* d_bcount = nullptr;
  int32_t* d_fdep_ptr = nullptr;
  int32_t* d_fdep_idx = nullptr;
  qn_fdesc* d_fdesc = nullptr;
  qn_bdesc* d_bdesc = nullptr;
  int32_t* d_fblob = nullptr;
  int32_t* d_hlev_ptr = nullptr;
  int32_t* d_hlev_sup = nullptr;
  int32_t* d_dlev_ptr = nullptr;
  int32_t* d_dlev_sup = nullptr;
  unsigned* d_flags = nullptr;    // nbatch x (n_ftask + n_btask) completion epochs
  double* d_ftile = nullptr;      // task-tiled Z copies of the persistent solve (see factor_upload)
  double* d_btile = nullptr;
  int64_t ftile_n = 0, btile_n = 0;  // entries per instance
  double* d_stile = nullptr;      // S^-1 as packed lower-triangle tiles (kTopTile^2 each, tile (I,J), I >= J)
  double* d_tpart = nullptr;      // nbatch x nt x nt x kTopTile x 3 partial products of the symmetric top apply
  unsigned* d_tcnt = nullptr;     // nbatch x nt arrival counters of the partials per row block
  unsigned* d_stage_cnt = nullptr;  // [forward tasks done, top blocks done] (top-fused solve)
  int32_t tnt = 0;                // row blocks of the top (ceil(K / kTopTile))
  int32_t* d_tcols = nullptr;
  int32_t* d_tg_ptr = nullptr;
  int32_t* d_tg_idx = nullptr;
  unsigned* d_sched = nullptr;    // [ticket_f, done_f, epoch_f, ticket_b, done_b, epoch_b]
  double* d_io = nullptr;         // staging for the plain solve API (n x 3 in, out)
  unsigned long long* d_trace = nullptr;  // diagnostics only (qn_factor_trace_solve)
  unsigned long long* d_ktl = nullptr;    // diagnostics only (qn_system_timeline; owned by the system)
  const unsigned long long* d_passes = nullptr;
  int smem_f = 0, smem_b = 0;     // dynamic shared memory of the forward / backward solve kernels
  int grid_f = 0, grid_b = 0;     // persistent solve grids (co-resident CTAs)
  bool fused = false;             // forward + backward in one persistent kernel (no dense top)
  int smem_fused = 0, grid_fused = 0;
  int batch_smem = 0;             // > 0: batched mode, one CTA per instance (bytes of shared memory)
  int32_t batch_max_nc = 0, batch_zmax = 0;  // batched mode: widest supernode, largest Z block (entries)
  bool on_device = false;
  int32_t lookahead = 0;          // persistent solve ticket lookahead (prepare_solve_kernels)
  int32_t pdl = 0;                // solve kernels launched with programmatic stream serialization (set by the system)
  int32_t many_tasks = 0;         // throughput-bound factor: many tasks per CTA (rhs formed once by k_solve_rhs)
  int32_t solve_opts = 0;         // QN_SOLVE_OPTS experiment knob (see FactorView::opts)
};

namespace qn {
constexpr int64_t kTaskEntries = 8192;  // Z entries per solve task (64 KB shared-memory tile)
constexpr int64_t kTopMax = 4096;
constexpr int kTopTile = 64;            // symmetric top apply: S^-1 stored as 64 x 64 lower-triangle tiles       // max columns of the dense top block (S^-1 <= 134 MB)
constexpr int64_t kTopDenseAll = 1536;  // systems this small are solved entirely as x = A^-1 b (dense)
constexpr int64_t kTopMinWidth = 600;   // a level joins the dense top only if its widest supernode has >= this many columns
constexpr int64_t kBwdTaskCols = 64;    // max columns of a backward task
// forward tasks: tile + f doubles so that three CTAs (tile + f + 8 KB of list / partial-sum staging + static)
// share an SM's 228 KB
constexpr int64_t kFwdBudget = (74 * 1024 - 8192) / 8;
constexpr int64_t kSmemPerCtaPair = 110 * 1024;  // dynamic smem per CTA with two CTAs per SM (228 KB - reserved/static)
// bottom-of-tree subtree collapse (see factor_build_host)
constexpr int32_t kCollapseHeight = 2;  // swept on c1-c3 with the current solve kernels: 2 > 3 (+3.6 % at c2), 1 and 4 slower
constexpr double kCollapseCols = 512;
constexpr double kCollapseGrowth = 2.5;

// host: ordering + symbolic + numeric factorisation; returns QN_OK / QN_ERR_*
int factor_build_host(qn_factor* f, int64_t n, const int64_t* indptr, const int32_t* indices,
                      const double* values, int64_t nbatch, const double* coords);
int factor_upload(qn_factor* f);
void factor_free_device(qn_factor* f);

// Functors describing where the solve reads its right-hand side and writes its result.
struct SolveIO {
  // plain API: B (n x 3, original order) -> X (n x 3, original order)
  const double* B = nullptr;
  double* X = nullptr;
};

// Forward + backward solve on `stream` for all batch instances whose `active`
// entry is non-zero (active == nullptr => all). The L-BFGS variant forms its
// RHS on the fly (see qn_solver.cu) via the templated kernels in qn_sptrsv.cuh.
int factor_solve_plain(qn_factor* f, int64_t batch, cudaStream_t stream);
}  // namespace qn

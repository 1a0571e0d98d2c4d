// Shared device/host helpers for the qnsim B200 library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "qnsim_b200.h"

namespace qn {

// diagnostics timeline (qn_system_timeline): per body pass, globaltimer ns at
// the entry of block 0 and at the end of the finalising block / last CTA of
// k_grad, k_eta, k_vec, k_tet, sptrsv_forward, sptrsv_backward
constexpr int kTimelinePasses = 512, kTimelineKernels = 7;


// ---- error plumbing (thread-local message for qn_last_error) ---------------
void set_error(const std::string& msg);
const char* get_error();
void count_launch(int n = 1);
// while a graph is being captured, QN_CHECK_LAUNCH records nodes, not launches
struct CaptureScope {
  CaptureScope();
  ~CaptureScope();
};

#define QN_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::qn::set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" __FILE__); \
      return QN_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

#define QN_CHECK_LAUNCH()                                                                   \
  do {                                                                                      \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ != cudaSuccess) {                                                                \
      ::qn::set_error(std::string("kernel launch: ") + cudaGetErrorString(e_) + " @" __FILE__); \
      return QN_ERR_CUDA;                                                                   \
    }                                                                                       \
    ::qn::count_launch();                                                                   \
  } while (0)

#define QN_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) {                  \
      ::qn::set_error(msg);         \
      return (code);                \
    }                               \
  } while (0)

constexpr int kSMs = 148;

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Programmatic dependent launch (PDL) between consecutive kernels of a frame
// (experiment, off by default: QN_PDL=1): a kernel launched through launch_k
// with pdl = true may be scheduled while its predecessor in the stream (or
// frame graph) drains, and pdl_entry(), the first statement of such kernels,
// blocks until the predecessor grid has completed and its writes are visible.
// Nothing runs before pdl_entry(), so results are those of the serialised
// launches.  Measured on the B200: back-to-back stream launches gain (c3
// stand-alone solve 215 -> 208 us) but inside the frame graph the kernel
// boundaries are already short — neutral with the implicit trigger (c3 2.73 k
// it/s either way), and 2-8 % SLOWER with an early griddepcontrol.launch_dependents
// (the dependents' resident CTAs slow the predecessor's tail).  Launched
// without the attribute, pdl_entry() returns at once.
__device__ __forceinline__ void pdl_entry() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <class... KArgs, class... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}

// ---- device helpers ----------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide reduction of K doubles per thread; result valid in thread 0.
// Fixed order (warp butterfly then warps in index order) => deterministic.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* smem /* >= K*32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) smem[k * 32 + warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < K) {  // thread k finishes value k (warps in index order)
    double a = 0.0;
    for (int w = 0; w < nw; ++w) a += smem[threadIdx.x * 32 + w];
    smem[threadIdx.x * 32] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = smem[k * 32];
  }
  __syncthreads();
}

// block_sum for the entries whose bit is set in `used` (K <= 64); others are
// left untouched in thread 0.  `used` must be uniform across the block.
template <int K>
__device__ __forceinline__ void block_sum_masked(double (&v)[K], double* smem, unsigned long long used) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if ((used >> k) & 1ull) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((used >> k) & 1ull) smem[k * 32 + warp] = v[k];
  }
  __syncthreads();
  // thread k finishes value k (warps in index order) into smem[k * 32]
  if (threadIdx.x < K && ((used >> threadIdx.x) & 1ull)) {
    double a = 0.0;
    for (int w = 0; w < nw; ++w) a += smem[threadIdx.x * 32 + w];
    smem[threadIdx.x * 32] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((used >> k) & 1ull) v[k] = smem[k * 32];
  }
  __syncthreads();
}

#endif  // __CUDACC__

}  // namespace qn

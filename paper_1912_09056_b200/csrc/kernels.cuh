// Device-side building blocks shared by the kernels.
#pragma once

#include <atomic>
#include "common.cuh"

namespace camg {

extern std::atomic<int64_t> g_launches;
// per-thread count (kernels recorded into a graph by this thread's capture)
extern thread_local int64_t g_thread_launches;
inline void note_launch(int n = 1) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  g_thread_launches += n;
}

constexpr double kDropTol = 1e-300;  // sparse.py:21 DROP_TOL
constexpr int kDotBlocks = 592;      // 4 x 148 SMs
constexpr int64_t kSellMinBlockRows = 50000;  // fewer block rows: lanes cannot fill 148 SMs
constexpr int64_t kSellPairSlices = 5000;  // below: two lanes per block row (C5: level-1 passes faster one lane per row)
constexpr int64_t kSellQuadBlocks = int64_t(1) << 40;  // ... or rows averaging this many blocks (R at 117: measured slower, opt-in)
constexpr int64_t kSellQuadSlices = 0;  // below: four lanes per block row (measured slower on C5 level 1: opt-in)
constexpr int64_t kMcgsCtaRows = 24576;  // S~ up to this size: single-CTA MC-SGS (x in 192 KB smem)
constexpr int64_t kMcgsCtaNnz = 131072;
constexpr int64_t kGsSellMinRows = 30000;
constexpr int64_t kGsSellMinNodesPerColour = 16384;  // ... and this many nodes per colour
constexpr double kChebRatio = 30.0;  // Chebyshev predictor: lower bound lmax / 30 (Ifpack2 / MueLu default)
constexpr double kChebBoost = 1.1;   // ... upper bound 1.1 lmax  // MC-SGS predictor: colour-ordered SELL from this many K rows  // ... and this many non-zeros (one SM streams it per colour pass)

// Programmatic dependent launch (PDL): V-cycle kernels let their successor
// launch as soon as every CTA of theirs runs (launch_dependents) and wait for
// the predecessor's completion before touching produced data (wait), so the
// launch latency of the ~500 kernels of a cycle overlaps the previous tail.
// Without the PDL launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define CAMG_PDL_ENTRY() \
  do {                    \
    pdl_launch_dependents(); \
    pdl_wait();           \
  } while (0)

bool use_pdl();  // CAMG_PDL=0 disables

template <class K, class... Args>
inline void launch_k(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  if (!use_pdl()) {
    kernel<<<grid, block, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CAMG_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// lanes per row for vector-CSR kernels, from the mean row length
inline int group_for(double avg) {
  if (avg <= 1.5) return 1;
  if (avg <= 3.0) return 2;
  if (avg <= 6.0) return 4;
  if (avg <= 12.0) return 8;
  if (avg <= 24.0) return 16;
  return 32;
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if (G == 32) return 0xffffffffu;
  const unsigned lane = threadIdx.x & 31;
  return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
}

template <int G>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, G);
  return v;
}

// x_j read from the u part (j < split) or the lambda part (j >= split; a null
// lambda pointer reads zeros)
template <bool SPLIT>
__device__ __forceinline__ double xload(const double* __restrict__ xu, const double* __restrict__ xl,
                                        int64_t split, int32_t c) {
  if (!SPLIT) return __ldg(xu + c);
  if (c < split) return __ldg(xu + c);
  return xl ? __ldg(xl + (c - split)) : 0.0;
}

template <int G, bool SPLIT>
__device__ __forceinline__ double row_dot(const CsrView& A, int64_t row, const double* __restrict__ xu,
                                          const double* __restrict__ xl, int64_t split, int lane) {
  const int64_t s = A.rowptr[row], e = A.rowptr[row + 1];
  double acc = 0.0;
  for (int64_t p = s + lane; p < e; p += G) {
    const int32_t c = __ldcs(A.col + p);
    CAMG_DCHECK(c >= 0 && c < A.n_cols, "csr column index out of range");
    acc = fma(__ldcs(A.val + p), xload<SPLIT>(xu, xl, split, c), acc);
  }
  return acc;
}

// deterministic block reduction (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (w == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

void vec_axpy(int64_t n, double a, const double* x, double* y, cudaStream_t s);
void vec_scale(int64_t n, double a, double* y, cudaStream_t s);
void dot_device(int64_t n, const double* x, const double* y, double* out_dev, double* part, cudaStream_t s);
Csr* csr_axpby(double alpha, const Csr* A, double beta, const Csr* B, cudaStream_t s);
Csr* csr_scale_rows(const Csr* A, const double* sc, cudaStream_t s);
Csr* csr_saddle_merge(const Csr* K, const Csr* B1, const Csr* B2, const Csr* Cz, cudaStream_t s);
Csr* spgemm(const Csr* A, const Csr* B, cudaStream_t s);
Csr* galerkin(const Csr* R, const Csr* A, const Csr* P, cudaStream_t s);

}  // namespace camg

// Block smoothers, levels and the V-cycle on device.
//
// Replaces BlockSmoother (smoothers.py:245-329) with Jacobi / dense-direct
// inner solves, Hierarchy.solve_coarsest / apply (hierarchy.py:96-120) and
// vcycle (hierarchy.py:272-287).  All vectors are merged [u; lambda].
//
// One smoother step = one fused sweep over the top block row [K | B1] (the
// residual, the first predictor sweep and the u update in one pass over K),
// plus a few small kernels on the lambda side and on the interface rows of B1.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>
#include <utility>
#include <mutex>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "common.cuh"
#include "pointsolve.cuh"
#include "kernels.cuh"
#include "sell.cuh"

namespace camg {

Csr* schur(const Csr* B2, const Csr* Cz, const Csr* B1, const double* ainv, double scale, cudaStream_t s);
void recip(int64_t n, const double* d, double* out, cudaStream_t s);

// ---------------------------------------------------------------------------
// fused row kernels

struct RowEpi {
  const double* b;       // rhs (merged indexing)
  const double* x;       // current iterate (merged indexing), null = zero
  double* out_r;         // residual (optional)
  const double* dscale;  // d = dscale[i] * r (optional)
  double* out_d;         // (optional)
  double* out_x;         // xmode 0: x[i] + coef*d ; xmode 1: x0 + coef*((x + d) - x0)
  double coef;
  const double* x0 = nullptr;  // relaxation origin for xmode 1 (null = 0)
  int xmode = 0;
  double* out_y = nullptr;     // Jacobi iterate y = x + d (optional)
  const double* dprev = nullptr;  // Chebyshev: d = c1*dprev + c2*dscale*r
  double c1 = 0.0, c2 = 1.0;
};

// r_i = b_i - A_i x for rows [row0, row0+nrows), x split at `split` into
// (xu, xl); optional jacobi-style epilogue.
template <int G, bool ZERO, bool SPLIT>
__global__ void __launch_bounds__(256) k_resid(CsrView A, int64_t row0, int64_t nrows, const double* __restrict__ xu,
                                               const double* __restrict__ xl, int64_t split, RowEpi e) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  for (int64_t rr = tid / G; rr < nrows; rr += stride) {
    const int64_t i = row0 + rr;
    double acc = 0.0;
    if (!ZERO) {
      acc = row_dot<G, SPLIT>(A, i, xu, xl, split, lane);
      acc = group_sum<G>(acc, mask);
    }
    if (lane == 0) {
      const double r = e.b[i] - acc;
      if (e.out_r) e.out_r[i] = r;
      if (e.dscale) {
        double d = e.dscale[i] * r;
        if (e.dprev) d = e.c1 * e.dprev[i] + e.c2 * d;
        else if (e.c2 != 1.0) d = e.c2 * d;
        if (e.out_d) e.out_d[i] = d;
        const double xi = (ZERO || !e.x) ? 0.0 : e.x[i];
        const double y = xi + d;
        if (e.out_y) e.out_y[i] = y;
        if (e.out_x) {
          if (e.xmode) {
            const double o = e.x0 ? e.x0[i] : 0.0;
            e.out_x[i] = o + e.coef * (y - o);
          } else {
            e.out_x[i] = xi + e.coef * d;
          }
        }
      }
    }
  }
}

// extra Jacobi sweep on K (rows < nu): d_new = d + dinv*(r - K d); optional x update
template <int G>
__global__ void __launch_bounds__(256) k_jacobi(CsrView A, int64_t nu, const double* __restrict__ d,
                                                const double* __restrict__ r, const double* __restrict__ dinv,
                                                double* __restrict__ d_new, const double* __restrict__ x,
                                                double* __restrict__ out_x, double coef) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  for (int64_t i = tid / G; i < nu; i += stride) {
    double acc = row_dot<G, true>(A, i, d, nullptr, nu, lane);
    acc = group_sum<G>(acc, mask);
    if (lane == 0) {
      const double dn = d[i] + dinv[i] * (r[i] - acc);
      d_new[i] = dn;
      if (out_x) out_x[i] = (x ? x[i] : 0.0) + coef * dn;
    }
  }
}

// lambda-side: rc_q = (A_bot [vu; vl])_q - c_q, q in [0, nl)
template <int G>
__global__ void __launch_bounds__(256) k_lam_rhs(CsrView A, int64_t nu, int64_t nl, const double* __restrict__ vu,
                                                 const double* __restrict__ vl, const double* __restrict__ c,
                                                 double* __restrict__ rc) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  for (int64_t q = tid / G; q < nl; q += stride) {
    double acc = row_dot<G, true>(A, nu + q, vu, vl, nu, lane);
    acc = group_sum<G>(acc, mask);
    if (lane == 0) rc[q] = acc - c[q];
  }
}

// corrector Jacobi sweep on S~ : first sweep from zero (dl = dinv*rc) or
// dl_new = dl + dinv*(rc - S dl)
template <int G, bool FIRST>
__global__ void __launch_bounds__(256) k_corr_jacobi(CsrView S, const double* __restrict__ rc,
                                                     const double* __restrict__ dinv, const double* __restrict__ dl,
                                                     double* __restrict__ dl_new) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  for (int64_t q = tid / G; q < S.n_rows; q += stride) {
    if (FIRST) {
      if (lane == 0) dl_new[q] = dinv[q] * rc[q];
    } else {
      double acc = row_dot<G, false>(S, q, dl, nullptr, S.n_cols, lane);
      acc = group_sum<G>(acc, mask);
      if (lane == 0) dl_new[q] = dl[q] + dinv[q] * (rc[q] - acc);
    }
  }
}

// Multicolour (node-block) Gauss-Seidel kernels for the CSR path (levels
// without a colour-ordered SELL) and for one-CTA sweeps of small operators.
// One lane group per node of one colour: the BS rows of the node are
// accumulated together with the values from before this pass (independent
// loads, one reduction per row), then the node's DOFs are updated in order
// (backward: reverse) through its stored diagonal block,
//   dv_d = dinv_d * (b_d - acc_d - sum_{e before d} K_de dv_e),  y_d += dv_d,
// which is the sequential Gauss-Seidel update (smoothers.py:155-164) on the
// colour-permuted operator.  Columns >= split read xl (lambda; null = 0).
// Rows of one colour share no entries, so no address a group writes is read
// by another group of the same launch.
template <int BS, bool FWD>
__device__ __forceinline__ void node_delta(const double* acc, const double* __restrict__ db,
                                           const double* __restrict__ b, const double* __restrict__ dinv,
                                           int64_t base, double* dv) {
#pragma unroll
  for (int dd = 0; dd < BS; ++dd) {
    const int d = FWD ? dd : BS - 1 - dd;
    double corr = 0.0;
#pragma unroll
    for (int ee = 0; ee < dd; ++ee) {
      const int e = FWD ? ee : BS - 1 - ee;
      corr = fma(db[d * BS + e], dv[e], corr);
    }
    dv[d] = dinv[base + d] * ((b[base + d] - acc[d]) - corr);
  }
}

// The colour passes form a chain of small kernels: each lets its successor
// launch at once and the successor loads its constant operands (node list,
// row structure, the first matrix entries) before waiting (PDL, kernels.cuh),
// so the launch gap and the matrix-load latency leave the critical path.
template <int G, int BS, bool FWD>
__global__ void __launch_bounds__(256) k_mcgs_node(CsrView A, const int32_t* __restrict__ nodes, int64_t nn,
                                                   const double* __restrict__ dblk, const double* __restrict__ xl,
                                                   int64_t split, const double* __restrict__ b,
                                                   const double* __restrict__ dinv, double* y) {
  pdl_launch_dependents();
  constexpr int PRE = BS == 1 ? 4 : (BS <= 3 ? 2 : 1);  // entries per row and lane loaded before the wait
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  const double* __restrict__ yr = y;
  bool waited = false;
  for (int64_t k = tid / G; k < nn; k += stride) {
    const int64_t node = nodes[k];
    const int64_t base = node * BS;
    int64_t p0[BS];
    int len[BS];
    int maxlen = 0;
#pragma unroll
    for (int r = 0; r < BS; ++r) {
      p0[r] = A.rowptr[base + r];
      len[r] = (int)(A.rowptr[base + r + 1] - p0[r]);
      maxlen = max(maxlen, len[r]);
    }
    int32_t pc[BS][PRE];
    double pv[BS][PRE];
#pragma unroll
    for (int r = 0; r < BS; ++r)
#pragma unroll
      for (int j = 0; j < PRE; ++j) {
        const int t = lane + j * G;
        pc[r][j] = t < len[r] ? __ldcs(A.col + p0[r] + t) : -1;
        pv[r][j] = t < len[r] ? __ldcs(A.val + p0[r] + t) : 0.0;
      }
    if (!waited) {
      pdl_wait();  // y, b and lambda come from the preceding kernels
      waited = true;
    }
    double acc[BS];
#pragma unroll
    for (int r = 0; r < BS; ++r) {
      acc[r] = 0.0;
#pragma unroll
      for (int j = 0; j < PRE; ++j) {
        const int32_t c = pc[r][j];
        if (c >= 0) {
          const double xv = c < split ? __ldg(yr + c) : (xl ? __ldg(xl + (c - split)) : 0.0);
          acc[r] = fma(pv[r][j], xv, acc[r]);
        }
      }
    }
    for (int t = lane + PRE * G; t < maxlen; t += G) {
#pragma unroll
      for (int r = 0; r < BS; ++r) {
        if (t < len[r]) {
          const int32_t c = __ldcs(A.col + p0[r] + t);
          const double xv = c < split ? __ldg(yr + c) : (xl ? __ldg(xl + (c - split)) : 0.0);
          acc[r] = fma(__ldcs(A.val + p0[r] + t), xv, acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < BS; ++r) acc[r] = group_sum<G>(acc[r], mask);
    if (lane == 0) {
      double dv[BS];
      node_delta<BS, FWD>(acc, dblk + node * (BS * BS), b, dinv, base, dv);
#pragma unroll
      for (int d = 0; d < BS; ++d) y[base + d] = yr[base + d] + dv[d];
    }
  }
}

// Whole sweeps (all colours forward then backward, __syncthreads between
// colours) of a small square operator in one CTA, the iterate in shared
// memory: replaces 2 x ncolours tiny launches per sweep on coarse levels.
template <int G, int BS>
__global__ void __launch_bounds__(1024) k_mcgs_node_cta(CsrView A, const int32_t* __restrict__ nodes,
                                                        const int64_t* __restrict__ cptr, int ncol, int sweeps,
                                                        bool zero, const double* __restrict__ dblk,
                                                        const double* __restrict__ b,
                                                        const double* __restrict__ dinv, double* __restrict__ yg) {
  CAMG_PDL_ENTRY();
  extern __shared__ double xs[];
  const int64_t n = A.n_rows;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int grp = threadIdx.x / G, ngrp = blockDim.x / G;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) xs[i] = zero ? 0.0 : yg[i];
  __syncthreads();
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int dir = 0; dir < 2; ++dir) {
      for (int cc = 0; cc < ncol; ++cc) {
        const int c = dir == 0 ? cc : ncol - 1 - cc;
        for (int64_t k = cptr[c] + grp; k < cptr[c + 1]; k += ngrp) {
          const int64_t node = nodes[k];
          const int64_t base = node * BS;
          int64_t p0[BS];
          int len[BS];
          int maxlen = 0;
#pragma unroll
          for (int r = 0; r < BS; ++r) {
            p0[r] = A.rowptr[base + r];
            len[r] = (int)(A.rowptr[base + r + 1] - p0[r]);
            maxlen = max(maxlen, len[r]);
          }
          double acc[BS];
#pragma unroll
          for (int r = 0; r < BS; ++r) acc[r] = 0.0;
          for (int t = lane; t < maxlen; t += G) {
#pragma unroll
            for (int r = 0; r < BS; ++r)
              if (t < len[r]) acc[r] = fma(A.val[p0[r] + t], xs[A.col[p0[r] + t]], acc[r]);
          }
#pragma unroll
          for (int r = 0; r < BS; ++r) acc[r] = group_sum<G>(acc[r], mask);
          if (lane == 0) {
            double dv[BS];
            if (dir == 0) node_delta<BS, true>(acc, dblk + node * (BS * BS), b, dinv, base, dv);
            else node_delta<BS, false>(acc, dblk + node * (BS * BS), b, dinv, base, dv);
#pragma unroll
            for (int d = 0; d < BS; ++d) xs[base + d] = xs[base + d] + dv[d];
          }
        }
        __syncthreads();
      }
    }
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) yg[i] = xs[i];
}

// diagonal node blocks of rows [0, nn*bs): dblk[node][r][c] (zeros where absent)
__global__ void k_extract_dblk(CsrView A, int64_t nn, int bs, double* __restrict__ dblk) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nn * bs; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = q / bs;
    const int r = (int)(q % bs);
    for (int64_t p = A.rowptr[q]; p < A.rowptr[q + 1]; ++p) {
      const int64_t c = A.col[p] - node * bs;
      if (c >= 0 && c < bs) dblk[(node * bs + r) * bs + c] = A.val[p];
    }
  }
}

template <int G, int BS>
static void launch_mcgs_node(const Csr* A, const int32_t* nodes, int64_t nn, const double* dblk, const double* xl,
                             int64_t split, const double* b, const double* dinv, double* y, bool fwd, cudaStream_t s) {
  unsigned grid = grid_for(nn * G, 256, int64_t(kNumSMs) * 16);
  note_launch();
  if (fwd) launch_k(k_mcgs_node<G, BS, true>, grid, 256, 0, s, view(A), nodes, nn, dblk, xl, split, b, dinv, y);
  else launch_k(k_mcgs_node<G, BS, false>, grid, 256, 0, s, view(A), nodes, nn, dblk, xl, split, b, dinv, y);
}

template <int G>
struct LaunchMcgsNode {
  static void run(const Csr* A, const int32_t* nodes, int64_t nn, int bs, const double* dblk, const double* xl,
                  int64_t split, const double* b, const double* dinv, double* y, bool fwd, cudaStream_t s) {
    if (nn <= 0) return;
    constexpr int GG = G < 4 ? 4 : G;
    switch (bs) {
      case 1: return launch_mcgs_node<GG, 1>(A, nodes, nn, dblk, xl, split, b, dinv, y, fwd, s);
      case 2: return launch_mcgs_node<GG, 2>(A, nodes, nn, dblk, xl, split, b, dinv, y, fwd, s);
      case 3: return launch_mcgs_node<GG, 3>(A, nodes, nn, dblk, xl, split, b, dinv, y, fwd, s);
      case 6: return launch_mcgs_node<GG, 6>(A, nodes, nn, dblk, xl, split, b, dinv, y, fwd, s);
      default: throw Error(CAMG_ERR_NATIVE, "unsupported node block size");
    }
  }
};

template <int G, int BS>
static void launch_mcgs_cta(const Csr* A, const int32_t* nodes, const int64_t* cptr, int ncol, int sweeps, bool zero,
                            const double* dblk, const double* b, const double* dinv, double* y, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    CAMG_CUDA(cudaFuncSetAttribute(k_mcgs_node_cta<G, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * kMcgsCtaRows)));
    attr = true;
  }
  note_launch();
  k_mcgs_node_cta<G, BS><<<1, 1024, sizeof(double) * A->n_rows, s>>>(view(A), nodes, cptr, ncol, sweeps, zero, dblk, b,
                                                                     dinv, y);
}

template <int G>
struct LaunchMcgsCta {
  static void run(const Csr* A, const int32_t* nodes, const int64_t* cptr, int ncol, int bs, int sweeps, bool zero,
                  const double* dblk, const double* b, const double* dinv, double* y, cudaStream_t s) {
    constexpr int GG = G < 4 ? 4 : G;
    switch (bs) {
      case 1: return launch_mcgs_cta<GG, 1>(A, nodes, cptr, ncol, sweeps, zero, dblk, b, dinv, y, s);
      case 2: return launch_mcgs_cta<GG, 2>(A, nodes, cptr, ncol, sweeps, zero, dblk, b, dinv, y, s);
      case 3: return launch_mcgs_cta<GG, 3>(A, nodes, cptr, ncol, sweeps, zero, dblk, b, dinv, y, s);
      case 6: return launch_mcgs_cta<GG, 6>(A, nodes, cptr, ncol, sweeps, zero, dblk, b, dinv, y, s);
      default: throw Error(CAMG_ERR_NATIVE, "unsupported node block size");
    }
  }
};

// Multicolour Gauss-Seidel sweeps of a small square operator (point colouring)
// on one 16-CTA thread-block cluster: every CTA keeps the rows it owns (the
// p-th node of each colour goes to CTA p mod 16) and a replica of the iterate
// in shared memory; a row update is stored into all 16 replicas through
// distributed shared memory and the colours are separated by cluster
// barriers.  The matrix is read from L2/HBM once per launch instead of once
// per colour pass, and a pass costs ~1 us instead of a kernel launch.  Same
// visiting order and update as k_mcgs_node<G, 1>.
constexpr int kMcgsCluster = 16;

template <int G>
__global__ void __launch_bounds__(1024, 1) k_mcgs_cl(int n, int ncol, int sweeps, const int32_t* __restrict__ nd_all,
                                                     const int32_t* __restrict__ rp_all,
                                                     const uint16_t* __restrict__ col_all,
                                                     const double* __restrict__ val_all,
                                                     const int64_t* __restrict__ off_nd,
                                                     const int64_t* __restrict__ off_nz,
                                                     const int32_t* __restrict__ cp_all, const double* __restrict__ b,
                                                     const double* __restrict__ dinv, double* __restrict__ y) {
  CAMG_PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int64_t nloc = off_nd[r + 1] - off_nd[r];
  const int64_t nz = off_nz[r + 1] - off_nz[r];
  double* x = reinterpret_cast<double*>(smraw);
  double* val = x + n;
  int32_t* rp = reinterpret_cast<int32_t*>(val + nz);
  int32_t* nd = rp + nloc + 1;
  int32_t* cp = nd + nloc;
  uint16_t* col = reinterpret_cast<uint16_t*>(cp + ncol + 1);
  for (int64_t i = threadIdx.x; i < nz; i += blockDim.x) {
    val[i] = val_all[off_nz[r] + i];
    col[i] = col_all[off_nz[r] + i];
  }
  for (int64_t i = threadIdx.x; i <= nloc; i += blockDim.x) rp[i] = rp_all[off_nd[r] + r + i];
  for (int64_t i = threadIdx.x; i < nloc; i += blockDim.x) nd[i] = nd_all[off_nd[r] + i];
  for (int i = threadIdx.x; i <= ncol; i += blockDim.x) cp[i] = cp_all[(int64_t)r * (ncol + 1) + i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = 0.0;
  cl.sync();
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int grp = threadIdx.x / G, ngrp = blockDim.x / G;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int dir = 0; dir < 2; ++dir) {
      for (int cc = 0; cc < ncol; ++cc) {
        const int c = dir == 0 ? cc : ncol - 1 - cc;
        for (int k = cp[c] + grp; k < cp[c + 1]; k += ngrp) {
          const int i = nd[k];
          double acc = 0.0;
          for (int p = rp[k] + lane; p < rp[k + 1]; p += G) acc = fma(val[p], x[col[p]], acc);
          acc = group_sum<G>(acc, mask);
          const double xn = x[i] + dinv[i] * (b[i] - acc);
          for (int t = lane; t < kMcgsCluster; t += G) *cl.map_shared_rank(x + i, t) = xn;
        }
        cl.sync();
      }
    }
  }
  if (r == 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = x[i];
}

template <int G>
struct LaunchMcgsCl {
  static void run(int n, int ncol, int sweeps, const int32_t* nd, const int32_t* rp, const uint16_t* col,
                  const double* val, const int64_t* off_nd, const int64_t* off_nz, const int32_t* cp, size_t smem,
                  const double* b, const double* dinv, double* y, cudaStream_t s) {
    constexpr int GG = G < 4 ? 4 : G;
    static bool attr = false;
    if (!attr) {
      CAMG_CUDA(cudaFuncSetAttribute(k_mcgs_cl<GG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      CAMG_CUDA(cudaFuncSetAttribute(k_mcgs_cl<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kMcgsCluster);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kMcgsCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    note_launch();
    CAMG_CUDA(cudaLaunchKernelEx(&cfg, k_mcgs_cl<GG>, n, ncol, sweeps, nd, rp, col, val, off_nd, off_nz, cp, b, dinv,
                                 y));
  }
};

// y = x_u (zero if x is null), g = b_u
__global__ void k_gs_init(int64_t nu, const double* __restrict__ x, const double* __restrict__ b,
                          double* __restrict__ y, double* __restrict__ g) {
  CAMG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nu; i += (int64_t)gridDim.x * blockDim.x) {
    y[i] = x ? x[i] : 0.0;
    g[i] = b[i];
  }
}

// g_i -= B1_i . lam on the nonempty rows of B1 (g = b_u - B1 lam)
__global__ void k_b1_sub(CsrView B1, const int64_t* __restrict__ rows, int64_t nrows, const double* __restrict__ lam,
                         double* __restrict__ g) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 7;
  const unsigned mask = group_mask<8>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / 8;
  for (int64_t k = tid / 8; k < nrows; k += stride) {
    const int64_t i = rows[k];
    double acc = row_dot<8, false>(B1, i, lam, nullptr, B1.n_cols, lane);
    acc = group_sum<8>(acc, mask);
    if (lane == 0) g[i] = g[i] - acc;
  }
}

// Uzawa relaxation: out = x0 + alpha (y - x0)   (x0 null = 0)
__global__ void k_relax(int64_t n, const double* __restrict__ x0, const double* __restrict__ y, double alpha,
                        double* __restrict__ out) {
  CAMG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double o = x0 ? x0[i] : 0.0;
    out[i] = o + alpha * (y[i] - o);
  }
}

// x_out_lam = x_lam + coef*dl
__global__ void k_lam_update(int64_t nl, const double* __restrict__ xl, const double* __restrict__ dl, double coef,
                             double* __restrict__ out) {
  CAMG_PDL_ENTRY();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nl; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = (xl ? xl[q] : 0.0) + coef * dl[q];
}

// x_u[i] -= mult * ainv[i] * (B1_i . dl) on the nonempty rows of B1
__global__ void k_b1_correct(CsrView B1, const int64_t* __restrict__ rows, int64_t nrows,
                             const double* __restrict__ ainv, const double* __restrict__ dl, double mult,
                             double* __restrict__ xu) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 7;
  const unsigned mask = group_mask<8>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / 8;
  for (int64_t k = tid / 8; k < nrows; k += stride) {
    const int64_t i = rows[k];
    double acc = row_dot<8, false>(B1, i, dl, nullptr, B1.n_cols, lane);
    acc = group_sum<8>(acc, mask);
    if (lane == 0) xu[i] = xu[i] - mult * (ainv[i] * acc);
  }
}

// small dense LU solve (LAPACK getrf factors, column-major, 0-based pivots)
__global__ void __launch_bounds__(1024) k_lu_solve(int n, const double* __restrict__ LU, const int32_t* __restrict__ piv,
                                                   const double* __restrict__ b, double* __restrict__ xg) {
  CAMG_PDL_ENTRY();
  extern __shared__ double xs[];
  const bool sh = n <= 12288;
  double* x = sh ? xs : xg;
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = b[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      int p = piv[i];
      if (p != i) { double t = x[i]; x[i] = x[p]; x[p] = t; }
    }
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {  // unit lower
    const double xj = x[j];
    const double* colj = LU + (size_t)j * n;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) x[i] -= colj[i] * xj;
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {  // upper
    if (threadIdx.x == 0) x[j] /= LU[(size_t)j * n + j];
    __syncthreads();
    const double xj = x[j];
    const double* colj = LU + (size_t)j * n;
    for (int i = threadIdx.x; i < j; i += blockDim.x) x[i] -= colj[i] * xj;
    __syncthreads();
  }
  if (sh)
    for (int i = threadIdx.x; i < n; i += blockDim.x) xg[i] = x[i];
}

// Same solve with the factors staged in shared memory (n^2 + 2n doubles fit):
// every substitution step reads shared memory instead of L2, one barrier per
// step.  Identical operations to k_lu_solve.
__global__ void __launch_bounds__(1024) k_lu_solve_smem(int n, const double* __restrict__ LU,
                                                        const int32_t* __restrict__ piv, const double* __restrict__ b,
                                                        double* __restrict__ xg) {
  CAMG_PDL_ENTRY();
  extern __shared__ double sm[];
  double* lu = sm;
  double* x = sm + (size_t)n * n;
  double* y = x + n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) lu[i] = LU[i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = b[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      int p = piv[i];
      if (p != i) { double t = x[i]; x[i] = x[p]; x[p] = t; }
    }
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {  // unit lower
    const double xj = x[j];
    const double* colj = lu + (size_t)j * n;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) x[i] -= colj[i] * xj;
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {  // upper: y_j = x_j / u_jj, then eliminate it
    const double yj = x[j] / lu[(size_t)j * n + j];
    const double* colj = lu + (size_t)j * n;
    for (int i = threadIdx.x; i < j; i += blockDim.x) x[i] -= colj[i] * yj;
    if (threadIdx.x == 0) y[j] = yj;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) xg[i] = y[i];
}

// Dense LU solve of a larger coarsest operator (n_c^2 doubles do not fit in
// shared memory; C2: n_c = 2448, 48 MB of factors) on many SMs: one CTA per
// block of kLuB rows.  Forward: CTA i accumulates L_ik y_k over the earlier
// row blocks k as each one is published (release/acquire flags), then solves
// its unit-lower diagonal block by substitution in one warp and publishes
// y_i.  Backward, in reverse block order, the same with U and a non-unit
// diagonal.  The factors are read once (each CTA streams its row panel);
// the critical path is one diagonal-block solve + one flag hand-off per row
// block and direction.  Same LAPACK factors and pivots as k_lu_solve; the
// accumulation order within a row differs (parity bar 1e-10 on the V-cycle).
// flags[0..nb) forward, [nb..2nb) backward, flags[2nb] = finished CTAs: the
// last CTA to finish resets them for the next launch.
constexpr int kLuB = 64;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) k_lu_solve_blk(int n, const double* __restrict__ LU,
                                                      const int32_t* __restrict__ perm, const double* __restrict__ b,
                                                      double* y, double* x, unsigned* flags) {
  CAMG_PDL_ENTRY();
  __shared__ double acc[4][kLuB];
  __shared__ double diag[kLuB][kLuB + 1];  // diagonal block, [row][col]
  __shared__ double v[kLuB];
  const int nb = (n + kLuB - 1) / kLuB;
  const int i = blockIdx.x;
  const int r0 = i * kLuB;
  const int rows = min(kLuB, n - r0);
  const int t = threadIdx.x, rr = t & (kLuB - 1), cq = t >> 6;  // row in block, column quarter
  for (int dir = 0; dir < 2; ++dir) {
    const bool fwd = dir == 0;
    // diagonal block of L (fwd) / U (bwd) into shared memory
    for (int e = t; e < kLuB * kLuB; e += blockDim.x) {
      const int c = e / kLuB, r = e % kLuB;
      diag[r][c] = (r < rows && c < rows) ? LU[(size_t)(r0 + c) * n + (r0 + r)] : 0.0;
    }
    double a = 0.0;
    const double* src = fwd ? y : x;  // published blocks of the vector being solved for
    for (int q = 0; q < nb - 1; ++q) {
      const int k = fwd ? q : nb - 1 - q;  // blocks in publication order
      if (fwd ? k >= i : k <= i) break;
      const int c0 = k * kLuB, cols = min(kLuB, n - c0);
      if (t == 0)
        while (ld_acquire(flags + (fwd ? 0 : nb) + k) == 0) __nanosleep(64);
      __syncthreads();
      if (rr < rows)
        for (int c = cq; c < cols; c += 4)
          a = fma(LU[(size_t)(c0 + c) * n + (r0 + rr)], __ldcg(src + c0 + c), a);
    }
    acc[cq][rr] = a;
    __syncthreads();
    if (t < kLuB) {
      const double base = fwd ? (t < rows ? b[perm[r0 + t]] : 0.0) : (t < rows ? y[r0 + t] : 0.0);
      v[t] = base - (((acc[0][t] + acc[1][t]) + acc[2][t]) + acc[3][t]);
    }
    __syncthreads();
    if (t < 32) {  // substitution on the diagonal block: lane owns rows t, t+32
      double v0 = v[t], v1 = v[t + 32];
      if (fwd) {
        for (int j = 0; j < rows; ++j) {
          const double xj = __shfl_sync(0xffffffffu, j < 32 ? v0 : v1, j & 31);
          if (t > j) v0 = fma(-diag[t][j], xj, v0);
          if (t + 32 > j) v1 = fma(-diag[t + 32][j], xj, v1);
        }
      } else {
        for (int j = rows - 1; j >= 0; --j) {
          double xj = __shfl_sync(0xffffffffu, j < 32 ? v0 : v1, j & 31);
          xj = xj / diag[j][j];
          if (t == (j & 31)) {
            if (j < 32) v0 = xj; else v1 = xj;
          }
          if (t < j) v0 = fma(-diag[t][j], xj, v0);
          if (t + 32 < j) v1 = fma(-diag[t + 32][j], xj, v1);
        }
      }
      double* dst = fwd ? y : x;
      if (t < rows) dst[r0 + t] = v0;
      if (t + 32 < rows) dst[r0 + t + 32] = v1;
      __threadfence();
      __syncwarp();
      if (t == 0) st_release(flags + (fwd ? 0 : nb) + i, 1u);
    }
    __syncthreads();
  }
  if (t == 0) {
    __threadfence();
    if (atomicAdd(flags + 2 * nb, 1u) == (unsigned)(nb - 1)) {  // last CTA: reset for the next launch
      for (int k = 0; k < 2 * nb; ++k) flags[k] = 0u;
      __threadfence();
      flags[2 * nb] = 0u;
    }
  }
}

// Coarsest solve through the explicit inverse of the merged coarse operator
// (computed once at setup from the same LAPACK LU factors): x0 = A^-1 b,
// r = b - A x0 (sparse coarse operator), x = x0 + A^-1 r.  Two dense GEMVs
// (every row of A^-1 one warp, b staged in shared memory) replace 2 n
// dependent substitution steps; the refinement step brings the forward
// error back to the LU solve's O(eps cond(A)).  out = add + M v.
__global__ void __launch_bounds__(256) k_dense_gemv(int n, const double* __restrict__ M, const double* __restrict__ v,
                                                    const double* __restrict__ add, double* __restrict__ out) {
  CAMG_PDL_ENTRY();
  CAMG_DCHECK(n >= 0 && n <= 4096, "dense gemv size beyond its shared-memory staging");
  extern __shared__ double vs[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) vs[i] = v[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const double* row = M + (size_t)r * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = lane;
    for (; c + 96 < n; c += 128) {
      a0 = fma(__ldg(row + c), vs[c], a0);
      a1 = fma(__ldg(row + c + 32), vs[c + 32], a1);
      a2 = fma(__ldg(row + c + 64), vs[c + 64], a2);
      a3 = fma(__ldg(row + c + 96), vs[c + 96], a3);
    }
    for (; c < n; c += 32) a0 = fma(__ldg(row + c), vs[c], a0);
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = add ? add[r] + acc : acc;
  }
}

constexpr int kCoarseInvMax = 4096;  // n^2 doubles <= 128 MB (about the L2)

// ---------------------------------------------------------------------------
// Device factorization of the coarsest merged operator (hierarchy.py:242-249:
// scipy.linalg.lu_factor, i.e. LAPACK dgetrf semantics: P A = L U with
// partial pivoting, the first maximal |a_ik| as pivot (idamax), whole rows
// swapped, 0-based pivot rows in ipiv order), for hosts without LAPACK
// (camg_hierarchy_coarse_factor).  Right-looking, one cooperative grid with
// three grid-wide barriers per column: (1) every CTA finds the pivot
// redundantly and the grid swaps rows k and p; (2) multipliers l_i =
// a_ik / a_kk; (3) rank-1 update of the trailing block.  The factors differ
// from dgetrf's blocked order only in rounding.

__global__ void k_csr_to_dense_colmajor(CsrView A, double* __restrict__ D) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n_rows; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = A.rowptr[i]; p < A.rowptr[i + 1]; ++p) D[(size_t)A.col[p] * A.n_rows + i] = A.val[p];
}

__global__ void __launch_bounds__(256) k_dense_lu(int n, double* __restrict__ A, int32_t* __restrict__ piv,
                                                  double* __restrict__ lk) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[8];
  __shared__ int si[8];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < n; ++k) {
    // (1) pivot: first maximal |a_ik|, i >= k (every CTA, same result)
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      const double a = fabs(A[(size_t)k * n + i]);
      if (a > best) { best = a; bi = i; }  // i ascending per thread: first max kept
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { sv[w] = best; si[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
        if (sv[q] > sv[0] || (sv[q] == sv[0] && si[q] < si[0])) { sv[0] = sv[q]; si[0] = si[q]; }
    }
    __syncthreads();
    const int p = si[0] < n ? si[0] : k;
    if (tid == 0) piv[k] = p;
    if (p != k)
      for (int64_t j = tid; j < n; j += nthr) {
        const double t = A[(size_t)j * n + k];
        A[(size_t)j * n + k] = A[(size_t)j * n + p];
        A[(size_t)j * n + p] = t;
      }
    grid.sync();
    // (2) multipliers
    const double akk = A[(size_t)k * n + k];
    for (int64_t i = k + 1 + tid; i < n; i += nthr) {
      const double l = akk != 0.0 ? A[(size_t)k * n + i] / akk : 0.0;
      lk[i] = l;
      A[(size_t)k * n + i] = l;
    }
    grid.sync();
    // (3) trailing update A[i][j] -= l_i a_kj, i, j > k (column-major: i fastest)
    const int64_t m = n - k - 1;
    for (int64_t e = tid; e < m * m; e += nthr) {
      const int64_t j = k + 1 + e / m, i = k + 1 + e % m;
      A[(size_t)j * n + i] -= lk[i] * A[(size_t)j * n + k];
    }
    grid.sync();
  }
}

// X = A^-1 (row-major) from LAPACK-style factors on one cooperative grid:
// X = P I, then the unit-lower forward elimination row by row (X[i] -= l_ik
// X[k], i > k) and the backward one (X[k] /= u_kk; X[i] -= u_ik X[k], i < k),
// every step a rank-1 row update spread over the grid (coalesced rows).
__global__ void __launch_bounds__(256) k_lu_inverse_coop(int n, const double* __restrict__ LU,
                                                         const int32_t* __restrict__ piv, double* __restrict__ X,
                                                         int32_t* __restrict__ perm) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {  // row i of P A is row perm[i] of A (LAPACK's sequential swaps)
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = 0; i < n; ++i) {
      const int p = piv[i];
      const int32_t t = perm[i];
      perm[i] = perm[p];
      perm[p] = t;
    }
  }
  grid.sync();
  for (int64_t e = tid; e < (int64_t)n * n; e += nthr) {  // X = P (rows of the identity)
    const int64_t i = e / n, j = e % n;
    X[e] = (perm[i] == j) ? 1.0 : 0.0;
  }
  grid.sync();
  for (int k = 0; k < n - 1; ++k) {
    const int64_t m = n - k - 1;
    for (int64_t e = tid; e < m * n; e += nthr) {
      const int64_t i = k + 1 + e / n, j = e % n;
      X[i * n + j] -= LU[(size_t)k * n + i] * X[(int64_t)k * n + j];
    }
    grid.sync();
  }
  for (int k = n - 1; k >= 0; --k) {
    const double ukk = LU[(size_t)k * n + k];
    for (int64_t j = tid; j < n; j += nthr) X[(int64_t)k * n + j] /= ukk;
    grid.sync();
    for (int64_t e = tid; e < (int64_t)k * n; e += nthr) {
      const int64_t i = e / n, j = e % n;
      X[i * n + j] -= LU[(size_t)k * n + i] * X[(int64_t)k * n + j];
    }
    grid.sync();
  }
}

static void dense_gemv(int n, const double* M, const double* v, const double* add, double* out, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    CAMG_CUDA(cudaFuncSetAttribute(k_dense_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * kCoarseInvMax)));
    attr = true;
  }
  note_launch();
  launch_k(k_dense_gemv, grid_for((int64_t)n * 32, 256, int64_t(kNumSMs) * 4), 256, sizeof(double) * n, s, n, M, v,
           add, out);
}

// Explicit inverse X = (L U)^-1 of the MC-ILU(0) factors of a small S~
// (setup): thread j solves L U x = e_j over the rows in colour order
// (forward: unit L, backward: U with diagonal udiag), x = column j of X,
// stored row-major (X[i][j] at i*n + j: a warp's 32 columns are one
// coalesced 256-byte row segment; every thread of the warp walks the same
// factor row, so the factor loads are broadcasts).
__global__ void __launch_bounds__(128) k_ilu_inverse(int n, const int32_t* __restrict__ nd, CsrView L, CsrView U,
                                                     const double* __restrict__ udiag, double* __restrict__ X) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int r = 0; r < n; ++r) {
    const int i = nd[r];
    double acc = (i == j) ? 1.0 : 0.0;
    for (int64_t p = L.rowptr[i]; p < L.rowptr[i + 1]; ++p) acc -= L.val[p] * X[(size_t)L.col[p] * n + j];
    X[(size_t)i * n + j] = acc;
  }
  for (int r = n - 1; r >= 0; --r) {
    const int i = nd[r];
    double acc = X[(size_t)i * n + j];
    for (int64_t p = U.rowptr[i]; p < U.rowptr[i + 1]; ++p) acc -= U.val[p] * X[(size_t)U.col[p] * n + j];
    X[(size_t)i * n + j] = acc / udiag[i];
  }
}

// dl = X rc and the lambda update xo_l = xl + cl dl in one GEMV (warp per
// row); with M2 (n_b1 rows: mult diag(ainv) B1 X on the interface rows) the
// B1 correction xo_u[r_k] -= (M2 rc)_k runs in the same launch
__global__ void __launch_bounds__(256) k_dense_gemv_lam(int n, const double* __restrict__ M,
                                                        const double* __restrict__ v, const double* __restrict__ xl,
                                                        double cl, double* __restrict__ dl, double* __restrict__ xo_l,
                                                        const double* __restrict__ M2, const int64_t* __restrict__ b1_rows,
                                                        int n_b1, double* __restrict__ xo_u) {
  CAMG_PDL_ENTRY();
  CAMG_DCHECK(n >= 0 && n <= 4096, "dense gemv size beyond its shared-memory staging");
  extern __shared__ double vs[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) vs[i] = v[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n + n_b1; r += nw) {
    const double* row = r < n ? M + (size_t)r * n : M2 + (size_t)(r - n) * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = lane;
    for (; c + 96 < n; c += 128) {
      a0 = fma(__ldg(row + c), vs[c], a0);
      a1 = fma(__ldg(row + c + 32), vs[c + 32], a1);
      a2 = fma(__ldg(row + c + 64), vs[c + 64], a2);
      a3 = fma(__ldg(row + c + 96), vs[c + 96], a3);
    }
    for (; c < n; c += 32) a0 = fma(__ldg(row + c), vs[c], a0);
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (r < n) {
        dl[r] = acc;
        xo_l[r] = (xl ? xl[r] : 0.0) + cl * acc;
      } else {
        const int64_t u = b1_rows[r - n];
        xo_u[u] = xo_u[u] - acc;
      }
    }
  }
}

// M2[k][j] = mult ainv[r_k] sum_i B1[r_k, i] X[i][j] (r_k = b1_rows[k])
__global__ void k_b1_dense(int n, int64_t n_b1, const int64_t* __restrict__ b1_rows, CsrView B1,
                           const double* __restrict__ ainv, double mult, const double* __restrict__ X,
                           double* __restrict__ M2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_b1 * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / n, j = e % n;
    const int64_t r = b1_rows[k];
    double acc = 0.0;
    for (int64_t p = B1.rowptr[r]; p < B1.rowptr[r + 1]; ++p) acc = fma(B1.val[p], X[(size_t)B1.col[p] * n + j], acc);
    M2[e] = mult * (ainv[r] * acc);
  }
}

// the blocked multi-CTA solve needs all nb CTAs resident (they wait on each
// other): used from kLuBlkMin rows up to 148 row blocks
constexpr int kLuBlkMin = 192;
constexpr int kLuBlkMaxBlocks = 148;

// dense LU solve on one CTA: factors in shared memory when they fit
void lu_solve(int n, const double* LU, const int32_t* piv, const double* b, double* x, cudaStream_t s) {
  const size_t need = sizeof(double) * ((size_t)n * n + 2 * (size_t)n);
  note_launch();
  if (need <= size_t(220) * 1024) {
    static bool attr = false;
    if (!attr) {
      CAMG_CUDA(cudaFuncSetAttribute(k_lu_solve_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      attr = true;
    }
    launch_k(k_lu_solve_smem, 1, 1024, need, s, n, LU, piv, b, x);
    return;
  }
  const size_t sh = n <= 12288 ? sizeof(double) * n : 0;
  launch_k(k_lu_solve, 1, 1024, sh, s, n, LU, piv, b, x);
}

__global__ void k_first_zero(int64_t n, const double* __restrict__ d, unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (d[i] == 0.0) atomicMin(out, (unsigned long long)i);
}

__global__ void k_scaled_recip(int64_t n, const double* __restrict__ d, double num, double mul, double* __restrict__ o) {
  // o = num / (mul * d)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __ddiv_rn(num, __dmul_rn(mul, d[i]));
}

__global__ void k_nonempty_flags(const int64_t* __restrict__ rowptr, int64_t n, int32_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = rowptr[i + 1] > rowptr[i];
}

__global__ void k_copy(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  CAMG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// ---------------------------------------------------------------------------
// launch helpers with group-size dispatch

template <template <int> class F, class... Args>
void dispatch_g(double avg, Args&&... args) {
  switch (group_for(avg)) {
    case 1: F<1>::run(args...); break;
    case 2: F<2>::run(args...); break;
    case 4: F<4>::run(args...); break;
    case 8: F<8>::run(args...); break;
    case 16: F<16>::run(args...); break;
    default: F<32>::run(args...); break;
  }
}

template <int G>
struct LaunchResid {
  static void run(const Csr* A, int64_t row0, int64_t nrows, const double* xu, const double* xl, int64_t split,
                  const RowEpi& e, bool zero, cudaStream_t s) {
    if (nrows <= 0) return;
    unsigned grid = grid_for(nrows * G, 256, int64_t(kNumSMs) * 16);
    note_launch();
    if (zero) launch_k(k_resid<G, true, false>, grid, 256, 0, s, view(A), row0, nrows, xu, xl, split, e);
    else if (split < A->n_cols) launch_k(k_resid<G, false, true>, grid, 256, 0, s, view(A), row0, nrows, xu, xl, split, e);
    else launch_k(k_resid<G, false, false>, grid, 256, 0, s, view(A), row0, nrows, xu, xl, split, e);
  }
};

template <int G>
struct LaunchJacobi {
  static void run(const Csr* A, int64_t nu, const double* d, const double* r, const double* dinv, double* dn,
                  const double* x, double* ox, double coef, cudaStream_t s) {
    unsigned grid = grid_for(nu * G, 256, int64_t(kNumSMs) * 16);
    note_launch();
    launch_k(k_jacobi<G>, grid, 256, 0, s, view(A), nu, d, r, dinv, dn, x, ox, coef);
  }
};

template <int G>
struct LaunchLamRhs {
  static void run(const Csr* A, int64_t nu, int64_t nl, const double* vu, const double* vl, const double* c,
                  double* rc, cudaStream_t s) {
    if (nl <= 0) return;
    unsigned grid = grid_for(nl * G, 256, int64_t(kNumSMs) * 16);
    note_launch();
    launch_k(k_lam_rhs<G>, grid, 256, 0, s, view(A), nu, nl, vu, vl, c, rc);
  }
};

template <int G>
struct LaunchCorr {
  static void run(const Csr* S, const double* rc, const double* dinv, const double* dl, double* dn, bool first,
                  cudaStream_t s) {
    if (S->n_rows <= 0) return;
    unsigned grid = grid_for(S->n_rows * G, 256, int64_t(kNumSMs) * 16);
    note_launch();
    if (first) launch_k(k_corr_jacobi<G, true>, grid, 256, 0, s, view(S), rc, dinv, dl, dn);
    else launch_k(k_corr_jacobi<G, false>, grid, 256, 0, s, view(S), rc, dinv, dl, dn);
  }
};


static SellEpi sell_epi(const RowEpi& e) {
  SellEpi se;
  se.b = e.b; se.x = e.x; se.out_r = e.out_r; se.dscale = e.dscale; se.out_d = e.out_d;
  se.out_x = e.out_x; se.coef = e.coef; se.x0 = e.x0; se.xmode = e.xmode; se.out_y = e.out_y;
  se.dprev = e.dprev; se.c1 = e.c1; se.c2 = e.c2;
  return se;
}

// residual over rows [row0, row0+nrows): SELL mirror for the rows it covers,
// CSR for the rest
static void resid_rows(const Csr* A, int64_t row0, int64_t nrows, const double* xu, const double* xl,
                       int64_t split, const RowEpi& e, bool zero, cudaStream_t s) {
  if (A->sell && row0 == 0 && nrows >= A->sell->rows()) {
    const SellEpi se = sell_epi(e);
    sell_launch(A->sell, 1, zero, xu, xl, split < A->n_cols ? split : -1, se, s);
    const int64_t done = A->sell->rows();
    row0 += done;
    nrows -= done;
    if (nrows <= 0) return;
  }
  dispatch_g<LaunchResid>(A->avg_row, A, row0, nrows, xu, xl, split, e, zero, s);
}

static void jacobi_rows(const Csr* A, int64_t nu, const double* d, const double* r, const double* dinv, double* dn,
                        const double* x, double* ox, double coef, cudaStream_t s) {
  if (A->sell && A->sell->rows() == nu) {
    SellEpi se;
    se.d = d; se.r = r; se.dscale = dinv; se.out_d = dn; se.x = x; se.out_x = ox; se.coef = coef;
    sell_launch(A->sell, 2, false, d, nullptr, nu, se, s);
    return;
  }
  dispatch_g<LaunchJacobi>(A->avg_row, A, nu, d, r, dinv, dn, x, ox, coef, s);
}

Csr* block_graph_sym(const Csr* K, int bs, int64_t nn);

// Greedy colouring of the nodes (bs consecutive DOFs) of K in natural node
// order over the symmetrised node graph (nodes p != q coupled by a non-zero
// K entry); the multicolour predictor's colouring, emulated by the oracle.
static std::vector<int32_t> node_colors(const Csr* K, int64_t nu, int bs) {
  const int64_t nn = nu / bs;
  std::unique_ptr<Csr> Gs(block_graph_sym(K, bs, nn));
  std::vector<int64_t> rp(nn + 1);
  std::vector<int32_t> ci(Gs->nnz);
  CAMG_CUDA(cudaMemcpy(rp.data(), Gs->rowptr, sizeof(int64_t) * (nn + 1), cudaMemcpyDeviceToHost));
  if (Gs->nnz) CAMG_CUDA(cudaMemcpy(ci.data(), Gs->col, sizeof(int32_t) * Gs->nnz, cudaMemcpyDeviceToHost));
  if (getenv("CAMG_DEBUG"))
    fprintf(stderr, "[camg] node graph: %lld nodes, %lld edges\n", (long long)nn, (long long)Gs->nnz);
  std::vector<int32_t> color(nn, -1);
  std::vector<int64_t> seen(64, -1);  // seen[c] == i: colour c is taken by a neighbour of i
  for (int64_t i = 0; i < nn; ++i) {
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t c = color[ci[k]];
      if (c >= 0) {
        if (c >= (int32_t)seen.size()) seen.resize(2 * c + 2, -1);
        seen[c] = i;
      }
    }
    int32_t c = 0;
    while (c < (int32_t)seen.size() && seen[c] == i) ++c;
    color[i] = c;
  }
  return color;
}

// Multicolour (node-block) Gauss-Seidel on the rows [0, nu) of an operator
// whose leading nu x nu block is K: greedy node colouring, and for large K a
// colour-ordered block SELL of K (rhs g) instead of the CSR kernel (rhs b and
// the lambda columns of the merged rows).
struct McgsK {
  int64_t nu = 0;
  int bs = 1;
  std::vector<int64_t> col_ptr, col_slice;
  DBuf<int64_t> col_ptr_dev;
  DBuf<int32_t> nodes;
  DBuf<double> dblk;  // diagonal node blocks (CSR / CTA paths)
  Sell* sell = nullptr;
  DBuf<double> g;
  bool cta = false;  // small square operator: whole sweeps in one CTA
  // small square operators with point colouring: whole sweeps on one
  // 16-CTA cluster with the rows in distributed shared memory
  bool cl = false;
  size_t cl_smem = 0;
  DBuf<int32_t> cl_nd, cl_rp, cl_cp;
  DBuf<uint16_t> cl_col;
  DBuf<double> cl_val;
  DBuf<int64_t> cl_offnd, cl_offnz;
  double cl_avg = 0.0;
  ~McgsK() { delete sell; }
  int colors() const { return (int)col_ptr.size() - 1; }

  void setup(const Csr* K, int node_block, cudaStream_t s) {
    nu = K->n_rows;
    bs = node_block > 1 ? node_block : 1;
    if (nu % bs) bs = 1;
    const int64_t nn = nu / bs;
    std::vector<int32_t> color = node_colors(K, nu, bs);
    int ncol = 0;
    for (int32_t c : color) ncol = std::max(ncol, c + 1);
    if (getenv("CAMG_DEBUG"))
      fprintf(stderr, "[camg] mcgs: %lld nodes of %d DOFs, %d colours\n", (long long)nn, bs, ncol);
    col_ptr.assign(ncol + 1, 0);
    for (int32_t c : color) col_ptr[c + 1]++;
    for (int c = 0; c < ncol; ++c) col_ptr[c + 1] += col_ptr[c];
    std::vector<int32_t> nd(nn);
    {
      std::vector<int64_t> pos(col_ptr.begin(), col_ptr.end() - 1);
      for (int64_t i = 0; i < nn; ++i) nd[pos[color[i]]++] = (int32_t)i;
    }
    nodes = DBuf<int32_t>(nn + 1);
    CAMG_CUDA(cudaMemcpy(nodes.p, nd.data(), sizeof(int32_t) * nn, cudaMemcpyHostToDevice));
    dblk = DBuf<double>(nn * bs * bs + 1);
    CAMG_CUDA(cudaMemsetAsync(dblk.p, 0, sizeof(double) * (nn * bs * bs + 1), s));
    note_launch();
    k_extract_dblk<<<grid_for(nu, 256), 256, 0, s>>>(view(K), nn, bs, dblk.p);
    col_ptr_dev = DBuf<int64_t>(ncol + 1);
    CAMG_CUDA(cudaMemcpy(col_ptr_dev.p, col_ptr.data(), sizeof(int64_t) * (ncol + 1), cudaMemcpyHostToDevice));
    // one-CTA sweeps for small square operators (CAMG_MCGS_CTA=0 disables,
    // =1 lifts the non-zero limit)
    // (CAMG_MCGS_CTA=0 disables; measured against per-colour launches)
    const char* cta_env = getenv("CAMG_MCGS_CTA");
    cta = !(cta_env && cta_env[0] == '0') && K->n_cols == nu && nu <= kMcgsCtaRows && K->nnz <= kMcgsCtaNnz;
    const char* cl_env = getenv("CAMG_MCGS_CLUSTER");
    if (bs == 1 && K->n_cols == nu && nu <= 65535 && K->nnz <= (int64_t)kMcgsCluster * 24576 &&
        !(cl_env && cl_env[0] == '0'))
      setup_cluster(K, nd, ncol);
    // colour-ordered SELL from kGsSellMinRows rows (CAMG_GS_SELL=1 forces it,
    // =0 keeps the CSR path)
    const char* env = getenv("CAMG_GS_SELL");
    // (lane-per-node SELL needs enough nodes per colour to fill the GPU;
    // below that the group-per-row CSR kernel has more parallelism)
    const bool want = env ? env[0] == '1' : (nu >= kGsSellMinRows && nn >= (int64_t)ncol * kGsSellMinNodesPerColour);
    if (!cta && want && (bs == 1 || bs == 2 || bs == 3 || bs == 6)) {
      // positions: each colour's nodes in ascending order, padded to whole slices
      std::vector<int32_t> order;
      col_slice.assign(ncol + 1, 0);
      for (int c = 0; c < ncol; ++c) {
        for (int64_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k) order.push_back(nd[k]);
        while (order.size() % 32) order.push_back(-1);
        col_slice[c + 1] = (int64_t)order.size() / 32;
      }
      sell = sell_build_ordered(K, bs, nu, nu, order, s);
      g = DBuf<double>(nu + 1);
    }
  }

  // rows of the p-th node of every colour on CTA p mod 16, compact CSR per
  // CTA (16-bit columns) and its colour ranges; enabled if the largest
  // CTA's rows plus the iterate fit in shared memory
  void setup_cluster(const Csr* K, const std::vector<int32_t>& nd, int ncol) {
    const int64_t n = nu, CS = kMcgsCluster;
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> ci(K->nnz);
    std::vector<double> va(K->nnz);
    CAMG_CUDA(cudaMemcpy(rp.data(), K->rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    if (K->nnz) {
      CAMG_CUDA(cudaMemcpy(ci.data(), K->col, sizeof(int32_t) * K->nnz, cudaMemcpyDeviceToHost));
      CAMG_CUDA(cudaMemcpy(va.data(), K->val, sizeof(double) * K->nnz, cudaMemcpyDeviceToHost));
    }
    std::vector<std::vector<int32_t>> lnd(CS), lrp(CS), lcp(CS);
    std::vector<std::vector<uint16_t>> lcol(CS);
    std::vector<std::vector<double>> lval(CS);
    for (int64_t r = 0; r < CS; ++r) lrp[r].push_back(0);
    for (int c = 0; c < ncol; ++c) {
      for (int64_t r = 0; r < CS; ++r) lcp[r].push_back((int32_t)lnd[r].size());
      for (int64_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k) {
        const int64_t r = (k - col_ptr[c]) % CS;
        const int32_t i = nd[k];
        lnd[r].push_back(i);
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
          lcol[r].push_back((uint16_t)ci[p]);
          lval[r].push_back(va[p]);
        }
        lrp[r].push_back((int32_t)lcol[r].size());
      }
    }
    for (int64_t r = 0; r < CS; ++r) lcp[r].push_back((int32_t)lnd[r].size());
    size_t need = 0;
    for (int64_t r = 0; r < CS; ++r) {
      const size_t b = 8 * (size_t)n + 10 * lval[r].size() + 4 * (2 * lnd[r].size() + 1) + 4 * (size_t)(ncol + 1) + 16;
      need = std::max(need, b);
    }
    if (need > size_t(200) * 1024) return;
    std::vector<int32_t> fnd, frp, fcp;
    std::vector<uint16_t> fcol;
    std::vector<double> fval;
    std::vector<int64_t> ond(CS + 1, 0), onz(CS + 1, 0);
    for (int64_t r = 0; r < CS; ++r) {
      ond[r + 1] = ond[r] + (int64_t)lnd[r].size();
      onz[r + 1] = onz[r] + (int64_t)lval[r].size();
      fnd.insert(fnd.end(), lnd[r].begin(), lnd[r].end());
      frp.insert(frp.end(), lrp[r].begin(), lrp[r].end());  // nloc+1 entries per CTA: offset ond[r] + r
      fcp.insert(fcp.end(), lcp[r].begin(), lcp[r].end());
      fcol.insert(fcol.end(), lcol[r].begin(), lcol[r].end());
      fval.insert(fval.end(), lval[r].begin(), lval[r].end());
    }
    auto up = [](auto& dst, const auto& src) {
      using T = typename std::decay_t<decltype(src)>::value_type;
      dst = std::decay_t<decltype(dst)>(src.size() + 1);
      if (!src.empty()) CAMG_CUDA(cudaMemcpy(dst.p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
    };
    up(cl_nd, fnd);
    up(cl_rp, frp);
    up(cl_cp, fcp);
    up(cl_col, fcol);
    up(cl_val, fval);
    up(cl_offnd, ond);
    up(cl_offnz, onz);
    cl_smem = need;
    cl_avg = n ? double(K->nnz) / n : 0.0;
    cl = true;
    cta = false;
  }

  // y = x_u (zero for x == null); the SELL path also sets g = b_u (callers
  // subtract B1 lam from g when the operator has lambda columns)
  void init(const double* x, const double* b, double* y, cudaStream_t s) {
    if (sell) {
      note_launch();
      launch_k(k_gs_init, grid_for(nu, 256), 256, 0, s, nu, x, b, y, g.p);
    } else if (!x) {
      CAMG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * nu, s));
    } else {
      note_launch();
      launch_k(k_copy, grid_for(nu, 256), 256, 0, s, nu, x, y);
    }
  }

  void pass(int c, bool fwd, bool zero, const Csr* Arows, const double* xl, const double* b, const double* dinv,
            double* y, cudaStream_t s) {
    if (sell) {
      sell_gs_launch(sell, col_slice[c], col_slice[c + 1], fwd, zero, nullptr, nu, g.p, dinv, y, s);
    } else {
      dispatch_g<LaunchMcgsNode>(Arows->avg_row, Arows, nodes.p + col_ptr[c], col_ptr[c + 1] - col_ptr[c], bs,
                                 dblk.p, xl, nu, b, dinv, y, fwd, s);
    }
  }

  // `sweeps` forward + backward colour sweeps of y_i += dinv_i (b_i - A_i [y; xl])
  // (zero: y == 0 and xl == null on entry, the first colour reads no matrix)
  void run(bool zero, const Csr* Arows, const double* xl, const double* b, const double* dinv, double* y, int sweeps,
           cudaStream_t s) {
    const int nc = colors();
    if (cl && zero && xl == nullptr && Arows->n_cols == nu) {
      dispatch_g<LaunchMcgsCl>(cl_avg, (int)nu, nc, sweeps, cl_nd.p, cl_rp.p, cl_col.p, cl_val.p, cl_offnd.p, cl_offnz.p,
                               cl_cp.p, cl_smem, b, dinv, y, s);
      return;
    }
    if (cta && Arows->n_cols == nu) {
      static double cta_avg = -1.0;  // CAMG_MCGS_CTA_G forces the lanes per row (tuning)
      if (cta_avg < 0.0) {
        const char* e = getenv("CAMG_MCGS_CTA_G");
        cta_avg = e ? atof(e) : 0.0;
      }
      dispatch_g<LaunchMcgsCta>(cta_avg > 0.0 ? cta_avg : Arows->avg_row, Arows, nodes.p, col_ptr_dev.p, nc, bs, sweeps, zero, dblk.p, b, dinv, y,
                                s);
      return;
    }
    for (int k = 0; k < sweeps; ++k) {
      for (int c = 0; c < nc; ++c) pass(c, true, zero && k == 0 && c == 0, Arows, xl, b, dinv, y, s);
      for (int c = nc - 1; c >= 0; --c) pass(c, false, false, Arows, xl, b, dinv, y, s);
    }
  }
};

// ---------------------------------------------------------------------------
// Multicolour ILU(0) corrector on S~ (GPU-only variant of the reference's
// "ilu0", smoothers.py:82-123, 167-171, 195-197): the reference ILU(0) -- no
// fill, IKJ order, unit lower factor -- of S~ with its rows and columns
// renumbered by the greedy point colouring of the MC-SGS corrector (colour
// by colour, ascending within a colour).  Rows of one colour are uncoupled,
// so on the renumbered matrix the strictly lower part of a row only reaches
// earlier colours and both triangular solves run one colour per pass.  The
// factors are kept in the original numbering (L and the strictly upper U as
// CSR over the original rows, U's diagonal apart), so the passes need no
// permuted vectors.  One sweep (smoothers.py:195-197):
//   forward  colour c = 0..C-1:  y_i = (rc_i - (S~ x)_i) - sum_{k in L(i)} l_ik y_k
//   backward colour c = C-1..0:  z_i = (y_i - sum_{j in U(i)} u_ij z_j) / u_ii,  x_i += z_i
// (x = 0 on the first sweep: no S~ product).  The oracle emulates it as the
// reference ILU(0) on the colour-permuted S~ (oracle/camg_oracle.py, Point).
template <int G, bool FWD, bool RES>
__global__ void __launch_bounds__(256) k_ilu_pass(CsrView T, CsrView A, const int32_t* __restrict__ nodes, int64_t nn,
                                                  const double* __restrict__ rc, const double* __restrict__ udiag,
                                                  double* y, double* z, double* x) {
  // the factor rows are constant: each pass loads its first entries before
  // waiting for the previous colour (PDL, as k_mcgs_node)
  pdl_launch_dependents();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  const double* v = FWD ? y : z;  // earlier colours' entries of the vector being solved for
  bool waited = false;
  for (int64_t k = tid / G; k < nn; k += stride) {
    const int64_t i = nodes[k];
    CAMG_DCHECK(i >= 0 && i < T.n_rows, "ilu pass row out of range");
    const int64_t p0 = T.rowptr[i] + lane, p1 = T.rowptr[i + 1];
    const int32_t c0 = p0 < p1 ? T.col[p0] : 0;
    CAMG_DCHECK(c0 >= 0 && c0 < T.n_cols, "ilu factor column out of range");
    const double v0 = p0 < p1 ? T.val[p0] : 0.0;
    if (!waited) {
      pdl_wait();
      waited = true;
    }
    double acc = p0 < p1 ? v0 * v[c0] : 0.0;
    for (int64_t p = p0 + G; p < p1; p += G) acc = fma(T.val[p], v[T.col[p]], acc);
    acc = group_sum<G>(acc, mask);
    double ax = 0.0;
    if (FWD && RES) {
      for (int64_t p = A.rowptr[i] + lane; p < A.rowptr[i + 1]; p += G) ax = fma(A.val[p], x[A.col[p]], ax);
      ax = group_sum<G>(ax, mask);
    }
    if (lane == 0) {
      if (FWD) {
        y[i] = (RES ? rc[i] - ax : rc[i]) - acc;
      } else {
        const double zi = (y[i] - acc) / udiag[i];
        z[i] = zi;
        x[i] = RES ? x[i] + zi : zi;
      }
    }
  }
}

template <int G>
struct LaunchIluPass {
  static void run(const Csr* T, const Csr* A, const int32_t* nodes, int64_t nn, bool fwd, bool res,
                  const double* rc, const double* udiag, double* y, double* z, double* x, cudaStream_t s) {
    if (nn <= 0) return;
    static const int64_t cap = getenv("CAMG_ILU_GRID") ? atoll(getenv("CAMG_ILU_GRID")) : int64_t(kNumSMs) * 16;
    // CTA size of the colour passes (CAMG_ILU_BLOCK, 64 / 128 / 256)
    static const int blk = getenv("CAMG_ILU_BLOCK") ? atoi(getenv("CAMG_ILU_BLOCK")) : 256;
    const unsigned grid = grid_for(nn * G, blk, cap * 256 / blk);
    note_launch();
    const CsrView tv = view(T), av = view(A);
#define CAMG_ILU_L(F, R) launch_k(k_ilu_pass<G, F, R>, grid, blk, 0, s, tv, av, nodes, nn, rc, udiag, y, z, x)
    if (fwd) { if (res) CAMG_ILU_L(true, true); else CAMG_ILU_L(true, false); }
    else { if (res) CAMG_ILU_L(false, true); else CAMG_ILU_L(false, false); }
#undef CAMG_ILU_L
  }
};

// The reference ILU(0) (smoothers.py:80-123): no fill, no pivoting, IKJ
// order on A's pattern (columns ascending), unit lower factor implicit;
// values factored in place with the product and the difference rounded
// separately, as the reference's Python loop does.  Returns the diagonal
// positions.  `name` maps a row to the number reported in errors (null:
// itself).
__attribute__((optimize("fp-contract=off"))) std::vector<int64_t> ilu0_ikj(int64_t n, const int64_t* rp,
                                                                                  const int32_t* ci, double* va,
                                                                                  const int32_t* name) {
  auto nm = [&](int64_t r) { return std::to_string(name ? (int64_t)name[r] : r); };
  std::vector<int64_t> dpos(n, -1), where(n, -1);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t q = rp[r]; q < rp[r + 1]; ++q)
      if (ci[q] == r) dpos[r] = q;
  for (int64_t r = 0; r < n; ++r)
    if (dpos[r] < 0) throw Error(CAMG_ERR_SINGULAR, "ILU(0): missing diagonal entry in row " + nm(r));
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) where[ci[q]] = q;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      const int64_t k = ci[q];
      if (k >= i) break;
      const double ukk = va[dpos[k]];
      if (ukk == 0.0) throw Error(CAMG_ERR_SINGULAR, "ILU(0): zero pivot in row " + nm(k));
      const double lik = va[q] / ukk;
      va[q] = lik;
      for (int64_t t = dpos[k] + 1; t < rp[k + 1]; ++t) {
        const int64_t w = where[ci[t]];
        if (w >= 0) {
          va[w] = va[w] - lik * va[t];  // product and difference rounded separately (fp-contract=off)
        }
      }
    }
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) where[ci[q]] = -1;
    if (va[dpos[i]] == 0.0) throw Error(CAMG_ERR_SINGULAR, "ILU(0): zero pivot in row " + nm(i));
  }
  return dpos;
}

// One zero-start MC-ILU(0) sweep of a small S~ on one 16-CTA cluster (the
// MC-SGS cluster layout, k_mcgs_cl): each CTA holds the L and U rows of the
// p-th row of every colour (p mod 16) and a replica of the vector being
// solved for; a solved entry is stored into all 16 replicas through
// distributed shared memory, colours are separated by cluster barriers, and
// y is overwritten by z in place (row i's y_i is last read by its own
// backward update, later colours' entries are z by then).
template <int G>
__global__ void __launch_bounds__(1024, 1) k_ilu_cl(int n, int ncol, const int32_t* __restrict__ nd_all,
                                                    const int32_t* __restrict__ lrp_all,
                                                    const uint16_t* __restrict__ lcol_all,
                                                    const double* __restrict__ lval_all,
                                                    const int32_t* __restrict__ urp_all,
                                                    const uint16_t* __restrict__ ucol_all,
                                                    const double* __restrict__ uval_all,
                                                    const int64_t* __restrict__ off_nd,
                                                    const int64_t* __restrict__ off_lnz,
                                                    const int64_t* __restrict__ off_unz,
                                                    const int32_t* __restrict__ cp_all, const double* __restrict__ rc,
                                                    const double* __restrict__ udiag, double* __restrict__ x) {
  CAMG_PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int64_t nloc = off_nd[r + 1] - off_nd[r];
  const int64_t lnz = off_lnz[r + 1] - off_lnz[r], unz = off_unz[r + 1] - off_unz[r];
  double* w = reinterpret_cast<double*>(smraw);
  double* lval = w + n;
  double* uval = lval + lnz;
  int32_t* lrp = reinterpret_cast<int32_t*>(uval + unz);
  int32_t* urp = lrp + nloc + 1;
  int32_t* nd = urp + nloc + 1;
  int32_t* cp = nd + nloc;
  uint16_t* lcol = reinterpret_cast<uint16_t*>(cp + ncol + 1);
  uint16_t* ucol = lcol + lnz;
  for (int64_t i = threadIdx.x; i < lnz; i += blockDim.x) {
    lval[i] = lval_all[off_lnz[r] + i];
    lcol[i] = lcol_all[off_lnz[r] + i];
  }
  for (int64_t i = threadIdx.x; i < unz; i += blockDim.x) {
    uval[i] = uval_all[off_unz[r] + i];
    ucol[i] = ucol_all[off_unz[r] + i];
  }
  for (int64_t i = threadIdx.x; i <= nloc; i += blockDim.x) {
    lrp[i] = lrp_all[off_nd[r] + r + i];
    urp[i] = urp_all[off_nd[r] + r + i];
  }
  for (int64_t i = threadIdx.x; i < nloc; i += blockDim.x) nd[i] = nd_all[off_nd[r] + i];
  for (int i = threadIdx.x; i <= ncol; i += blockDim.x) cp[i] = cp_all[(int64_t)r * (ncol + 1) + i];
  cl.sync();
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int grp = threadIdx.x / G, ngrp = blockDim.x / G;
  for (int dir = 0; dir < 2; ++dir) {
    for (int cc = 0; cc < ncol; ++cc) {
      const int c = dir == 0 ? cc : ncol - 1 - cc;
      for (int k = cp[c] + grp; k < cp[c + 1]; k += ngrp) {
        const int i = nd[k];
        double acc = 0.0;
        if (dir == 0) {
          for (int p = lrp[k] + lane; p < lrp[k + 1]; p += G) acc = fma(lval[p], w[lcol[p]], acc);
        } else {
          for (int p = urp[k] + lane; p < urp[k + 1]; p += G) acc = fma(uval[p], w[ucol[p]], acc);
        }
        acc = group_sum<G>(acc, mask);
        const double v = dir == 0 ? rc[i] - acc : (w[i] - acc) / udiag[i];
        for (int t = lane; t < kMcgsCluster; t += G) *cl.map_shared_rank(w + i, t) = v;
      }
      cl.sync();
    }
  }
  if (r == 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = w[i];
}

template <int G>
struct LaunchIluCl {
  static void run(int n, int ncol, const int32_t* nd, const int32_t* lrp, const uint16_t* lcol, const double* lval,
                  const int32_t* urp, const uint16_t* ucol, const double* uval, const int64_t* off_nd,
                  const int64_t* off_lnz, const int64_t* off_unz, const int32_t* cp, size_t smem, const double* rc,
                  const double* udiag, double* x, cudaStream_t s) {
    constexpr int GG = G < 4 ? 4 : G;
    static bool attr = false;
    if (!attr) {
      CAMG_CUDA(cudaFuncSetAttribute(k_ilu_cl<GG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      CAMG_CUDA(cudaFuncSetAttribute(k_ilu_cl<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kMcgsCluster);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kMcgsCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    note_launch();
    CAMG_CUDA(cudaLaunchKernelEx(&cfg, k_ilu_cl<GG>, n, ncol, nd, lrp, lcol, lval, urp, ucol, uval, off_nd, off_lnz,
                                 off_unz, cp, rc, udiag, x));
  }
};


// ---------------------------------------------------------------------------
// One zero-start MC-ILU(0) sweep of S~ (up to kLamIluMaxRows rows) fused with
// the lambda update on one 16-CTA cluster, without cluster barriers:
//   y = forward colour passes with L, z = backward passes with U,
//   lam'_q = lam_q + cl z_q,  dl_q = z_q (for the B1 correction kernel).
// Layout: CTA r owns the p-th row of every colour with p mod 16 == r (as
// k_ilu_cl).  Its factor rows are one contiguous byte stream in processing
// order (forward colour 0..C-1: L rows; backward C-1..0: U rows + u_ii), one
// 16-byte aligned segment per colour pass, streamed from L2 into shared
// memory by bulk copies (cp.async.bulk + mbarrier complete_tx): the whole
// stream at once when it fits, else through a ring of NB segment buffers
// refilled NB passes ahead.  The copies read only constant data and are
// issued before the programmatic-dependent-launch wait.  Every CTA keeps a
// replica of the solved vector in shared memory.  A solved entry is sent to
// all 16 replicas with st.async ... mbarrier::complete_tx (DSMEM store that
// signals the receiving CTA's barrier of that colour pass): each CTA waits
// for pass k-1's bytes (8 x rows of that colour) before computing pass k --
// no cluster barriers, no memory fences in the chain.  One barrier per pass
// (used once), so a fast CTA's stores for a later pass never count towards
// an earlier one; an entry's forward value y_i is overwritten by z_i only
// after every CTA has left the forward passes.  Per-row arithmetic equals
// k_ilu_cl<G> and k_lam_update (bit-identical results).
constexpr int kLamIluThreads = 1024;
constexpr int64_t kIluDenseMax = 2048;  // S~ rows up to which MC-ILU(0) runs through (L U)^-1 (32 MB)
constexpr int kLamIluMaxRows = 16384;

struct LamIluArgs {
  int n;                     // lambda rows (S~)
  int ncol;                  // colours
  int nb;                    // ring buffers (0: resident stream)
  int bufb;                  // ring buffer bytes
  const unsigned char* blob; // all CTAs' streams
  const int64_t* cta_off;    // [16+1] byte offsets of the CTA streams
  const int32_t* tab;        // [16][2C][3] {byte offset in stream, rows, nnz}
  const int32_t* own_off;    // [16][C+1] own rows before colour c
  const int32_t* own_nodes;  // own rows of every CTA, forward order, at own_base[r]
  const int32_t* own_base;   // [16+1]
  const int32_t* col_rows;   // [C] rows of each colour (bytes expected per pass / 8)
  int max_own;               // most rows owned by one CTA (uniform shared-memory layout)
  int* err;                  // barrier watchdog
  const double* rc;          // corrector right-hand side
  const double* xl;          // lambda (null = 0)
  double* xo_l;              // lambda out
  double* dl;                // z out
  double cl;                 // lambda update coefficient
};

__device__ __forceinline__ void lmb_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void lmb_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void lmb_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LMB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra LMB_WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// bounded wait: a barrier that never completes (a bug) sets *err and returns
// instead of hanging the GPU
__device__ __forceinline__ void lmb_wait_guard(uint64_t* bar, unsigned parity, int* err) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  for (int it = 0; it < (1 << 22); ++it) {
    unsigned ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
  }
  atomicExch(err, 1);
}
__device__ __forceinline__ void lbulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ unsigned mapa_cluster(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// DSMEM store of v to [raddr] in another CTA, completing 8 bytes of its barrier rbar
__device__ __forceinline__ void st_async_f64(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int G, int NT>
__global__ void __launch_bounds__(NT, 1) k_lam_ilu_cl(LamIluArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int C2 = 2 * a.ncol;
  // shared memory, same offsets in every CTA of the cluster (the pass
  // barriers and the replica are addressed remotely): barriers | replica |
  // own rc | tables | factor stream (resident) or ring
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* sbar = reinterpret_cast<uint64_t*>(smraw);  // stream buffers
  uint64_t* pbar = sbar + 8;                             // one per colour pass
  double* w = reinterpret_cast<double*>(pbar + ((C2 + 1) & ~1));
  const int nown = a.own_base[r + 1] - a.own_base[r];
  double* rcs = w + ((a.n + 1) & ~1);
  int32_t* tab = reinterpret_cast<int32_t*>(rcs + ((a.max_own + 1) & ~1));
  int32_t* oof = tab + ((3 * C2 + 3) & ~3);
  unsigned char* ring = reinterpret_cast<unsigned char*>(oof + ((a.ncol + 4) & ~3));
  const int64_t stream_bytes = a.cta_off[r + 1] - a.cta_off[r];
  const unsigned char* src = a.blob + a.cta_off[r];
  const int32_t* gtab = a.tab + (int64_t)r * 3 * C2;
  // constant data first: tables, barriers and the factor stream (before the PDL wait)
  for (int i = threadIdx.x; i < 3 * C2; i += blockDim.x) tab[i] = gtab[i];
  for (int i = threadIdx.x; i <= a.ncol; i += blockDim.x) oof[i] = a.own_off[(int64_t)r * (a.ncol + 1) + i];
  if (threadIdx.x == 0) {
    const int nsb = a.nb ? a.nb : 1;
    for (int i = 0; i < nsb; ++i) lmb_init(sbar + i, 1);
    for (int k = 0; k < C2; ++k) lmb_init(pbar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < C2; ++k) {  // pass k receives 8 bytes per row of its colour
      const int c = k < a.ncol ? k : C2 - 1 - k;
      lmb_expect_tx(pbar + k, 8u * (unsigned)a.col_rows[c]);
    }
    if (a.nb == 0) {
      lmb_expect_tx(sbar, (unsigned)stream_bytes);
      lbulk_g2s(ring, src, (unsigned)stream_bytes, sbar);
    } else {
      for (int k = 0; k < a.nb && k < C2; ++k) {
        const int off = gtab[3 * k];
        const int bytes = (k + 1 < C2 ? gtab[3 * (k + 1)] : (int)stream_bytes) - off;
        lmb_expect_tx(sbar + k, (unsigned)bytes);
        lbulk_g2s(ring + (int64_t)k * a.bufb, src + off, (unsigned)bytes, sbar + k);
      }
    }
  }
  pdl_launch_dependents();
  pdl_wait();
  {
    const int32_t* own = a.own_nodes + a.own_base[r];
    for (int o = threadIdx.x; o < nown; o += blockDim.x) rcs[o] = a.rc[own[o]];
  }
  __syncthreads();
  cluster_barrier();  // every CTA runs and its barriers are armed: stores may start
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int grp = threadIdx.x / G, ngrp = blockDim.x / G;
  const unsigned w_s = (unsigned)__cvta_generic_to_shared(w);
  const unsigned pbar_s = (unsigned)__cvta_generic_to_shared(pbar);
  // lanes t < 16 of a row group send to CTA t: cluster addresses of its replica and barriers
  const unsigned w_t = lane < kMcgsCluster ? mapa_cluster(w_s, lane) : 0u;
  const unsigned pbar_t = lane < kMcgsCluster ? mapa_cluster(pbar_s, lane) : 0u;
  for (int k = 0; k < C2; ++k) {
    const bool fwd = k < a.ncol;
    const int c = fwd ? k : C2 - 1 - k;
    const unsigned char* seg;
    if (a.nb == 0) {
      if (k == 0) lmb_wait_guard(sbar, 0, a.err);
      seg = ring + tab[3 * k];
    } else {
      lmb_wait_guard(sbar + (k % a.nb), (unsigned)((k / a.nb) & 1), a.err);
      seg = ring + (int64_t)(k % a.nb) * a.bufb;
    }
    if (k > 0) lmb_wait_guard(pbar + (k - 1), 0, a.err);  // every entry of the previous colour pass has arrived
    const int nrows = tab[3 * k + 1], nnz = tab[3 * k + 2];
    const double* val = reinterpret_cast<const double*>(seg);
    const double* ud = val + nnz;
    const int32_t* rp = reinterpret_cast<const int32_t*>(ud + (fwd ? 0 : nrows));
    const int32_t* node = rp + nrows + 1;
    const uint16_t* col = reinterpret_cast<const uint16_t*>(node + nrows);
    CAMG_DCHECK(tab[3 * k] + 8ll * nnz + 4ll * (nrows + 1) <= stream_bytes, "lam_ilu segment beyond its stream");
    for (int q = grp; q < nrows; q += ngrp) {
      double acc = 0.0;
      for (int p = rp[q] + lane; p < rp[q + 1]; p += G) {
        CAMG_DCHECK(p < nnz && col[p] < a.n, "lam_ilu entry out of range");
        acc = fma(val[p], w[col[p]], acc);
      }
      acc = group_sum<G>(acc, mask);
      const int i = node[q];
      CAMG_DCHECK(i >= 0 && i < a.n, "lam_ilu row out of range");
      const double v = fwd ? rcs[oof[c] + q] - acc : (w[i] - acc) / ud[q];
      for (int t = lane; t < kMcgsCluster; t += G) {
        const unsigned wt = G >= kMcgsCluster ? w_t : mapa_cluster(w_s, t);
        const unsigned bt = G >= kMcgsCluster ? pbar_t : mapa_cluster(pbar_s, t);
        st_async_f64(wt + 8u * (unsigned)i, v, bt + 8u * (unsigned)k);
      }
      if (!fwd && lane == 0) {
        a.xo_l[i] = (a.xl ? a.xl[i] : 0.0) + a.cl * v;
        a.dl[i] = v;
      }
    }
    if (a.nb && k + a.nb < C2) {  // refill this stream buffer NB passes ahead
      __syncthreads();
      if (threadIdx.x == 0) {
        const int kk = k + a.nb;
        const int off = tab[3 * kk];
        const int bytes = (kk + 1 < C2 ? tab[3 * (kk + 1)] : (int)stream_bytes) - off;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        lmb_expect_tx(sbar + (k % a.nb), (unsigned)bytes);
        lbulk_g2s(ring + (int64_t)(k % a.nb) * a.bufb, src + off, (unsigned)bytes, sbar + (k % a.nb));
      }
    }
  }
  lmb_wait_guard(pbar + (C2 - 1), 0, a.err);  // no store into this CTA's memory is still in flight when it exits
}

template <int G, int NT>
static void launch_lam_ilu_nt(const LamIluArgs& a, size_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    CAMG_CUDA(cudaFuncSetAttribute(k_lam_ilu_cl<G, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CAMG_CUDA(cudaFuncSetAttribute(k_lam_ilu_cl<G, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kMcgsCluster);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kMcgsCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl() ? 2 : 1;
  note_launch();
  CAMG_CUDA(cudaLaunchKernelEx(&cfg, k_lam_ilu_cl<G, NT>, a));
}

template <int G>
static void launch_lam_ilu(const LamIluArgs& a, size_t smem, cudaStream_t s) {
  static const int nt = getenv("CAMG_LAMILU_NT") ? atoi(getenv("CAMG_LAMILU_NT")) : kLamIluThreads;
  if (nt == 256) launch_lam_ilu_nt<G, 256>(a, smem, s);
  else if (nt == 512) launch_lam_ilu_nt<G, 512>(a, smem, s);
  else launch_lam_ilu_nt<G, 1024>(a, smem, s);
}

// ---------------------------------------------------------------------------
// The whole lambda side of one smoother step in ONE sync-free launch
// (k_lam_engine): every warp takes tickets in dependency order --
//   [0, n)            forward MC-ILU(0) rows in colour order, rc computed inline:
//                     y_i = ((A_bot [u_half; lam])_i - b_lam,i) - sum_{L(i)} l_ik y_k
//   [n, 2n)           backward rows in reverse colour order:
//                     z_i = (y_i - sum_{U(i)} u_ij z_j) / u_ii,  lam'_i = lam_i + cl z_i
//   [2n, 2n + n_b1)   interface rows: u'_r = u_half,r - mult ainv_r (B1 z)_r
// -- and reads an entry only after its producer's completion flag (acquire /
// release, as the sync-free triangular solve): a row waits for exactly the
// rows it reads instead of for whole colour passes, so the critical path is
// one flag hand-off per dependency level rather than one kernel boundary per
// colour, and the 35 launches of a step (k_lam_rhs, 2 x 16-17 colour passes,
// k_lam_update, k_b1_correct) become one.  Tickets are handed out in order,
// so every row a warp waits on is held by a running warp: deadlock-free for
// any grid.  Flags hold the launch epoch + 1 (zeroed buffers are "not done");
// the last warp to finish resets the ticket and advances the epoch, so the
// launch replays from a CUDA graph without memset nodes.  Bounded waits set
// the watchdog flag instead of hanging.  Same operations per row as the
// colour-pass path up to the summation order inside a row.
struct LamEngineArgs {
  CsrView A;                    // merged operator (lambda rows)
  CsrView L, U;                 // MC-ILU(0) factors, original numbering
  const double* udiag;
  const int32_t* nd;            // rows in colour order
  int64_t nu, n, n_b1;
  const double* uh;             // u_half
  const double* xl;             // lambda (null = 0)
  const double* bl;             // b_lam
  double* y;                    // forward values
  double* z;                    // backward values (dl)
  double* xo;                   // merged output
  double cl, mult;
  CsrView B1;
  const int64_t* b1_rows;
  const double* ainv;
  unsigned long long* ticket;   // sync block: ticket, done, epoch, flags
  unsigned* done;
  unsigned* epoch;
  unsigned* fy;
  unsigned* fz;
  int* err;
};

__device__ __forceinline__ unsigned eng_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double eng_ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void eng_st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// wait until flag == want (bounded)
__device__ __forceinline__ void eng_wait(const unsigned* f, unsigned want, int* err) {
  if (eng_ld_acquire(f) == want) return;
  for (int it = 0; it < (1 << 22); ++it) {
    __nanosleep(32);
    if (eng_ld_acquire(f) == want) return;
  }
  atomicExch(err, 1);
}

__global__ void __launch_bounds__(256) k_lam_engine(LamEngineArgs a) {
  CAMG_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const unsigned want = *a.epoch + 1u;  // read before any warp can finish
  const int64_t total = 2 * a.n + a.n_b1;
  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1ull);
    tk = __shfl_sync(0xffffffffu, tk, 0);
    if ((int64_t)tk >= total) break;
    const int64_t t = (int64_t)tk;
    if (t < a.n) {  // forward
      const int64_t i = a.nd[t];
      double r = 0.0;
      for (int64_t p = a.A.rowptr[a.nu + i] + lane; p < a.A.rowptr[a.nu + i + 1]; p += 32) {
        const int32_t c = a.A.col[p];
        CAMG_DCHECK(c >= 0 && c < a.A.n_cols, "engine: A column out of range");
        const double xv = c < a.nu ? a.uh[c] : (a.xl ? a.xl[c - a.nu] : 0.0);
        r = fma(a.A.val[p], xv, r);
      }
      double acc = 0.0;
      for (int64_t p = a.L.rowptr[i] + lane; p < a.L.rowptr[i + 1]; p += 32) {
        const int32_t k = a.L.col[p];
        CAMG_DCHECK(k >= 0 && k < a.n, "engine: L column out of range");
        eng_wait(a.fy + k, want, a.err);
        acc = fma(a.L.val[p], eng_ld_relaxed(a.y + k), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(0xffffffffu, r, o);
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
      }
      if (lane == 0) {
        a.y[i] = (r - a.bl[i]) - acc;
        eng_st_release(a.fy + i, want);
      }
    } else if (t < 2 * a.n) {  // backward
      const int64_t i = a.nd[2 * a.n - 1 - t];
      double acc = 0.0;
      for (int64_t p = a.U.rowptr[i] + lane; p < a.U.rowptr[i + 1]; p += 32) {
        const int32_t j = a.U.col[p];
        CAMG_DCHECK(j >= 0 && j < a.n, "engine: U column out of range");
        eng_wait(a.fz + j, want, a.err);
        acc = fma(a.U.val[p], eng_ld_relaxed(a.z + j), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        eng_wait(a.fy + i, want, a.err);
        const double zi = (eng_ld_relaxed(a.y + i) - acc) / a.udiag[i];
        a.z[i] = zi;
        a.xo[a.nu + i] = (a.xl ? a.xl[i] : 0.0) + a.cl * zi;
        eng_st_release(a.fz + i, want);
      }
    } else {  // interface row of B1
      const int64_t r = a.b1_rows[t - 2 * a.n];
      double acc = 0.0;
      for (int64_t p = a.B1.rowptr[r] + lane; p < a.B1.rowptr[r + 1]; p += 32) {
        const int32_t j = a.B1.col[p];
        CAMG_DCHECK(j >= 0 && j < a.n, "engine: B1 column out of range");
        eng_wait(a.fz + j, want, a.err);
        acc = fma(a.B1.val[p], eng_ld_relaxed(a.z + j), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) a.xo[r] = a.xo[r] - a.mult * (a.ainv[r] * acc);
    }
    __syncwarp();
  }
  // the last warp out resets the ticket and advances the epoch
  if (lane == 0) {
    __threadfence();
    const unsigned nw = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(a.done, 1u) == nw - 1) {
      *a.ticket = 0ull;
      *a.done = 0u;
      __threadfence();
      *a.epoch = want;
    }
  }
}

struct McIlu {
  int64_t n = 0;
  std::vector<int64_t> col_ptr;
  DBuf<int32_t> nodes;
  std::unique_ptr<Csr> L, U;  // strictly lower / upper factor rows, original numbering
  DBuf<double> udiag, y, z;
  // small S~: zero-start sweeps on one 16-CTA cluster (k_ilu_cl)
  bool cl = false;
  size_t cl_smem = 0;
  double cl_avg = 0.0;
  DBuf<int32_t> cl_nd, cl_lrp, cl_urp, cl_cp;
  DBuf<uint16_t> cl_lcol, cl_ucol;
  DBuf<double> cl_lval, cl_uval;
  DBuf<int64_t> cl_offnd, cl_offl, cl_offu;
  // fused lambda step (k_lam_ilu_cl)
  bool fused = false;
  int fz_nb = 0, fz_bufb = 0, fz_g = 4, fz_max_own = 0;
  size_t fz_smem = 0;
  DBuf<unsigned char> fz_blob;
  DBuf<int64_t> fz_cta_off;
  DBuf<int32_t> fz_tab, fz_own_off, fz_own_nodes, fz_own_base, fz_col_rows;
  DBuf<int> fz_err;
  // explicit inverse of the factors (small S~): one GEMV per zero-start sweep
  DBuf<double> dense_inv;
  // sync block of the one-launch lambda engine (k_lam_engine): ticket, done,
  // epoch, forward / backward flags (per workspace)
  DBuf<double> eng_sync;
  DBuf<int> eng_err;

  int colors() const { return (int)col_ptr.size() - 1; }

  void setup(const Csr* S, cudaStream_t s) {
    n = S->n_rows;
    CAMG_CHECK(S->n_cols == n, CAMG_ERR_DIMENSION, "ILU(0) needs a square operator");
    std::vector<int32_t> color = node_colors(S, n, 1);
    int ncol = 0;
    for (int32_t c : color) ncol = std::max(ncol, c + 1);
    col_ptr.assign(ncol + 1, 0);
    for (int32_t c : color) col_ptr[c + 1]++;
    for (int c = 0; c < ncol; ++c) col_ptr[c + 1] += col_ptr[c];
    std::vector<int32_t> nd(n), pos(n);  // nd[new] = old, pos[old] = new
    {
      std::vector<int64_t> at(col_ptr.begin(), col_ptr.end() - 1);
      for (int64_t i = 0; i < n; ++i) nd[at[color[i]]++] = (int32_t)i;
    }
    for (int64_t r = 0; r < n; ++r) pos[nd[r]] = (int32_t)r;
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> ci(S->nnz);
    std::vector<double> va(S->nnz);
    CAMG_CUDA(cudaMemcpy(rp.data(), S->rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    if (S->nnz) {
      CAMG_CUDA(cudaMemcpy(ci.data(), S->col, sizeof(int32_t) * S->nnz, cudaMemcpyDeviceToHost));
      CAMG_CUDA(cudaMemcpy(va.data(), S->val, sizeof(double) * S->nnz, cudaMemcpyDeviceToHost));
    }
    // renumbered matrix: row r = old row nd[r], columns renumbered and sorted
    std::vector<int64_t> prp(n + 1, 0);
    std::vector<int32_t> pci(S->nnz);
    std::vector<double> pva(S->nnz);
    {
      std::vector<std::pair<int32_t, double>> row;
      for (int64_t r = 0; r < n; ++r) {
        const int32_t o = nd[r];
        row.clear();
        for (int64_t q = rp[o]; q < rp[o + 1]; ++q) row.emplace_back(pos[ci[q]], va[q]);
        std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        prp[r + 1] = prp[r] + (int64_t)row.size();
        for (size_t t = 0; t < row.size(); ++t) {
          pci[prp[r] + t] = row[t].first;
          pva[prp[r] + t] = row[t].second;
        }
      }
    }
    // reference ILU(0) (smoothers.py:80-123) on the renumbered matrix
    std::vector<int64_t> dpos = ilu0_ikj(n, prp.data(), pci.data(), pva.data(), nd.data());
    // factors in the original numbering
    std::vector<int64_t> lrp(n + 1, 0), urp(n + 1, 0);
    for (int64_t r = 0; r < n; ++r) {
      lrp[nd[r] + 1] = dpos[r] - prp[r];
      urp[nd[r] + 1] = prp[r + 1] - dpos[r] - 1;
    }
    for (int64_t o = 0; o < n; ++o) {
      lrp[o + 1] += lrp[o];
      urp[o + 1] += urp[o];
    }
    std::vector<int32_t> lci(lrp[n]), uci(urp[n]);
    std::vector<double> lva(lrp[n]), uva(urp[n]), ud(n);
    for (int64_t r = 0; r < n; ++r) {
      const int32_t o = nd[r];
      int64_t a = lrp[o], b = urp[o];
      for (int64_t q = prp[r]; q < dpos[r]; ++q, ++a) { lci[a] = nd[pci[q]]; lva[a] = pva[q]; }
      for (int64_t q = dpos[r] + 1; q < prp[r + 1]; ++q, ++b) { uci[b] = nd[pci[q]]; uva[b] = pva[q]; }
      ud[o] = pva[dpos[r]];
    }
    auto upload = [&](const std::vector<int64_t>& tr, const std::vector<int32_t>& tc, const std::vector<double>& tv) {
      Csr* T = csr_alloc(n, n, tr[n]);
      CAMG_CUDA(cudaMemcpy(T->rowptr, tr.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
      if (tr[n]) {
        CAMG_CUDA(cudaMemcpy(T->col, tc.data(), sizeof(int32_t) * tr[n], cudaMemcpyHostToDevice));
        CAMG_CUDA(cudaMemcpy(T->val, tv.data(), sizeof(double) * tr[n], cudaMemcpyHostToDevice));
      }
      return T;
    };
    L.reset(upload(lrp, lci, lva));
    U.reset(upload(urp, uci, uva));
    udiag = DBuf<double>(n + 1);
    CAMG_CUDA(cudaMemcpy(udiag.p, ud.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    nodes = DBuf<int32_t>(n + 1);
    CAMG_CUDA(cudaMemcpy(nodes.p, nd.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    y = DBuf<double>(n + 1);
    z = DBuf<double>(n + 1);
    const char* cl_env = getenv("CAMG_MCGS_CLUSTER");
    if (n <= 65535 && !(cl_env && cl_env[0] == '0')) setup_cluster(nd, lrp, lci, lva, urp, uci, uva);
    const char* fz_env = getenv("CAMG_LAM_FUSED");
    if (n <= kLamIluMaxRows && !(fz_env && fz_env[0] == '0')) setup_fused(nd, lrp, lci, lva, urp, uci, uva, ud);
    eng_sync = DBuf<double>(2 + (n + 1));  // 16 B header + 2 x 4 B flags per row
    CAMG_CUDA(cudaMemset(eng_sync.p, 0, sizeof(double) * (2 + (n + 1))));
    eng_err = DBuf<int>(1);
    CAMG_CUDA(cudaMemset(eng_err.p, 0, sizeof(int)));
    const char* dn_env = getenv("CAMG_ILU_DENSE_MAX");
    const int64_t dense_max = dn_env ? atoll(dn_env) : kIluDenseMax;
    if (n >= 1 && n <= dense_max) {
      // (L U)^-1 in the original numbering, on the device
      dense_inv = DBuf<double>((size_t)n * n + 1);
      note_launch();
      k_ilu_inverse<<<(unsigned)((n + 127) / 128), 128>>>((int)n, nodes.p, view(L.get()), view(U.get()), udiag.p,
                                                         dense_inv.p);
      CAMG_LAUNCH_CHECK();
      CAMG_CUDA(cudaDeviceSynchronize());
    }
  }

  // the whole lambda side of a step in one sync-free launch (k_lam_engine)
  void run_engine(const Csr* A, int64_t nu, const double* uh, const double* xl, const double* bl, double* xo,
                  double* dl, double cl, const Csr* B1, const int64_t* b1_rows, int64_t n_b1, const double* ainv,
                  double mult, cudaStream_t s) {
    LamEngineArgs a;
    a.A = view(A);
    a.L = view(L.get());
    a.U = view(U.get());
    a.udiag = udiag.p;
    a.nd = nodes.p;
    a.nu = nu;
    a.n = n;
    a.n_b1 = n_b1;
    a.uh = uh;
    a.xl = xl;
    a.bl = bl;
    a.y = y.p;
    a.z = dl;
    a.xo = xo;
    a.cl = cl;
    a.mult = mult;
    a.B1 = view(B1);
    a.b1_rows = b1_rows;
    a.ainv = ainv;
    unsigned char* sb = reinterpret_cast<unsigned char*>(eng_sync.p);
    a.ticket = reinterpret_cast<unsigned long long*>(sb);
    a.done = reinterpret_cast<unsigned*>(sb + 8);
    a.epoch = reinterpret_cast<unsigned*>(sb + 12);
    a.fy = reinterpret_cast<unsigned*>(sb + 16);
    a.fz = a.fy + n;
    a.err = eng_err.p;
    const int64_t total = 2 * n + n_b1;
    static const int64_t cap = getenv("CAMG_ENGINE_CTAS") ? atoll(getenv("CAMG_ENGINE_CTAS")) : int64_t(kNumSMs) * 8;
    note_launch();
    launch_k(k_lam_engine, grid_for(total * 32, 256, cap), 256, 0, s, a);
  }

  // one zero-start sweep through the explicit inverse fused with the lambda
  // update: dl = (L U)^-1 rc, xo_l = xl + cl dl
  void run_dense(const double* rc, const double* xl, double* xo_l, double* dl, double cl, cudaStream_t s,
                 const double* M2 = nullptr, const int64_t* b1_rows = nullptr, int64_t n_b1 = 0,
                 double* xo_u = nullptr) {
    static bool attr = false;
    if (!attr) {
      CAMG_CUDA(cudaFuncSetAttribute(k_dense_gemv_lam, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * kCoarseInvMax)));
      attr = true;
    }
    note_launch();
    launch_k(k_dense_gemv_lam, grid_for((n + (M2 ? n_b1 : 0)) * 32, 256, int64_t(kNumSMs) * 4), 256,
             sizeof(double) * n, s, (int)n, (const double*)dense_inv.p, rc, xl, cl, dl, xo_l, M2, b1_rows,
             (int)(M2 ? n_b1 : 0), xo_u);
  }

  // per-CTA factor streams of k_lam_ilu_cl (see there)
  void setup_fused(const std::vector<int32_t>& nd, const std::vector<int64_t>& lrp, const std::vector<int32_t>& lci,
                   const std::vector<double>& lva, const std::vector<int64_t>& urp, const std::vector<int32_t>& uci,
                   const std::vector<double>& uva, const std::vector<double>& ud) {
    const int CS = kMcgsCluster;
    const int C = colors();
    const int C2 = 2 * C;
    std::vector<std::vector<unsigned char>> stream(CS);
    std::vector<int32_t> tab((size_t)CS * C2 * 3), oof((size_t)CS * (C + 1)), own_nodes, own_base(CS + 1, 0);
    std::vector<std::vector<int32_t>> own(CS);
    auto put = [](std::vector<unsigned char>& st, const void* p, size_t b) {
      const unsigned char* q = static_cast<const unsigned char*>(p);
      st.insert(st.end(), q, q + b);
    };
    int64_t max_seg = 0;
    for (int r = 0; r < CS; ++r) {
      for (int c = 0; c < C; ++c) {
        oof[(size_t)r * (C + 1) + c] = (int32_t)own[r].size();
        for (int64_t k = col_ptr[c] + r; k < col_ptr[c + 1]; k += CS) own[r].push_back(nd[k]);
      }
      oof[(size_t)r * (C + 1) + C] = (int32_t)own[r].size();
      for (int k = 0; k < C2; ++k) {
        const bool fwd = k < C;
        const int c = fwd ? k : C2 - 1 - k;
        std::vector<int32_t> rows;
        for (int64_t q = col_ptr[c] + r; q < col_ptr[c + 1]; q += CS) rows.push_back(nd[q]);
        const std::vector<int64_t>& rp = fwd ? lrp : urp;
        const std::vector<int32_t>& ci = fwd ? lci : uci;
        const std::vector<double>& va = fwd ? lva : uva;
        std::vector<int32_t> lrp2(1, 0);
        std::vector<double> vals, dg;
        std::vector<uint16_t> cols;
        for (int32_t i : rows) {
          for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            vals.push_back(va[p]);
            cols.push_back((uint16_t)ci[p]);
          }
          lrp2.push_back((int32_t)vals.size());
          if (!fwd) dg.push_back(ud[i]);
        }
        std::vector<unsigned char>& st = stream[r];
        const size_t start = st.size();
        tab[((size_t)r * C2 + k) * 3 + 0] = (int32_t)start;
        tab[((size_t)r * C2 + k) * 3 + 1] = (int32_t)rows.size();
        tab[((size_t)r * C2 + k) * 3 + 2] = (int32_t)vals.size();
        put(st, vals.data(), 8 * vals.size());
        put(st, dg.data(), 8 * dg.size());
        put(st, lrp2.data(), 4 * lrp2.size());
        put(st, rows.data(), 4 * rows.size());
        put(st, cols.data(), 2 * cols.size());
        st.resize((st.size() + 15) & ~size_t(15), 0);
        max_seg = std::max<int64_t>(max_seg, (int64_t)(st.size() - start));
      }
      own_base[r + 1] = own_base[r] + (int32_t)own[r].size();
      own_nodes.insert(own_nodes.end(), own[r].begin(), own[r].end());
    }
    // shared memory: replica + own rc + stream (resident) or ring + tables + barriers
    size_t max_stream = 0, max_own = 0;
    for (int r = 0; r < CS; ++r) {
      max_stream = std::max(max_stream, stream[r].size());
      max_own = std::max(max_own, own[r].size());
    }
    const size_t fixed = 8 * (8 + (size_t)((C2 + 1) & ~1)) + 8 * (size_t)((n + 1) & ~1) +
                         8 * ((max_own + 1) & ~size_t(1)) + 4 * (size_t)((3 * C2 + 3) & ~3) + 4 * (size_t)((C + 4) & ~3) + 16;
    const size_t cap = 227 * 1024;
    if (fixed + 16 > cap) return;
    int nb = 0;
    size_t ring = max_stream;
    // CAMG_LAM_RING=1 streams through a 2-buffer ring even when the whole
    // stream fits (tests exercise the refill path on small systems)
    const char* re = getenv("CAMG_LAM_RING");
    if (re && re[0] == '1' && C2 > 2 && fixed + 2 * (size_t)max_seg <= cap) {
      nb = 2;
      ring = 2 * (size_t)max_seg;
    } else if (fixed + max_stream > cap) {
      nb = (int)std::min<int64_t>((cap - fixed) / max_seg, 8);
      if (nb < 2) return;
      ring = (size_t)nb * max_seg;
    }
    std::vector<int64_t> cta_off(CS + 1, 0);
    std::vector<unsigned char> blob;
    for (int r = 0; r < CS; ++r) {
      blob.insert(blob.end(), stream[r].begin(), stream[r].end());
      cta_off[r + 1] = (int64_t)blob.size();
    }
    auto up = [](auto& dst, const auto& src) {
      using T = typename std::decay_t<decltype(src)>::value_type;
      dst = std::decay_t<decltype(dst)>(src.size() + 1);
      if (!src.empty()) CAMG_CUDA(cudaMemcpy(dst.p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
    };
    up(fz_blob, blob);
    up(fz_cta_off, cta_off);
    up(fz_tab, tab);
    up(fz_own_off, oof);
    up(fz_own_nodes, own_nodes);
    up(fz_own_base, own_base);
    std::vector<int32_t> crows(C);
    for (int c = 0; c < C; ++c) crows[c] = (int32_t)(col_ptr[c + 1] - col_ptr[c]);
    up(fz_col_rows, crows);
    fz_nb = nb;
    fz_max_own = (int)max_own;
    fz_err = DBuf<int>(1);
    CAMG_CUDA(cudaMemset(fz_err.p, 0, sizeof(int)));
    fz_bufb = (int)max_seg;
    fz_smem = fixed + ring;
    const double avg = n ? double(lrp[n] + urp[n]) / (2.0 * n) : 0.0;
    fz_g = std::max(4, group_for(avg));
    fused = true;
  }

  // one zero-start sweep fused with the lambda update (k_lam_ilu_cl):
  // xo_l = xl + cl z, dl = z for rc
  void run_fused(const double* rc, const double* xl, double* xo_l, double* dl, double cl, cudaStream_t s) {
    LamIluArgs a;
    a.n = (int)n;
    a.ncol = colors();
    a.nb = fz_nb;
    a.bufb = fz_bufb;
    a.blob = fz_blob.p;
    a.cta_off = fz_cta_off.p;
    a.tab = fz_tab.p;
    a.own_off = fz_own_off.p;
    a.own_nodes = fz_own_nodes.p;
    a.own_base = fz_own_base.p;
    a.col_rows = fz_col_rows.p;
    a.max_own = fz_max_own;
    a.err = fz_err.p;
    a.rc = rc;
    a.xl = xl;
    a.xo_l = xo_l;
    a.dl = dl;
    a.cl = cl;
    switch (fz_g) {
      case 4: launch_lam_ilu<4>(a, fz_smem, s); break;
      case 8: launch_lam_ilu<8>(a, fz_smem, s); break;
      case 16: launch_lam_ilu<16>(a, fz_smem, s); break;
      default: launch_lam_ilu<32>(a, fz_smem, s); break;
    }
  }

  // the p-th row of every colour on CTA p mod 16 (k_mcgs_cl layout); enabled
  // if the largest CTA's rows plus the vector replica fit in shared memory
  void setup_cluster(const std::vector<int32_t>& nd, const std::vector<int64_t>& lrp, const std::vector<int32_t>& lci,
                     const std::vector<double>& lva, const std::vector<int64_t>& urp,
                     const std::vector<int32_t>& uci, const std::vector<double>& uva) {
    const int64_t CS = kMcgsCluster;
    const int ncol = colors();
    std::vector<std::vector<int32_t>> lnd(CS), llrp(CS), lurp(CS), lcp(CS);
    std::vector<std::vector<uint16_t>> llcol(CS), lucol(CS);
    std::vector<std::vector<double>> llval(CS), luval(CS);
    for (int64_t r = 0; r < CS; ++r) {
      llrp[r].push_back(0);
      lurp[r].push_back(0);
    }
    for (int c = 0; c < ncol; ++c) {
      for (int64_t r = 0; r < CS; ++r) lcp[r].push_back((int32_t)lnd[r].size());
      for (int64_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k) {
        const int64_t r = (k - col_ptr[c]) % CS;
        const int32_t i = nd[k];
        lnd[r].push_back(i);
        for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) {
          llcol[r].push_back((uint16_t)lci[p]);
          llval[r].push_back(lva[p]);
        }
        for (int64_t p = urp[i]; p < urp[i + 1]; ++p) {
          lucol[r].push_back((uint16_t)uci[p]);
          luval[r].push_back(uva[p]);
        }
        llrp[r].push_back((int32_t)llcol[r].size());
        lurp[r].push_back((int32_t)lucol[r].size());
      }
    }
    for (int64_t r = 0; r < CS; ++r) lcp[r].push_back((int32_t)lnd[r].size());
    size_t need = 0;
    for (int64_t r = 0; r < CS; ++r) {
      const size_t b = 8 * (size_t)n + 10 * (llval[r].size() + luval[r].size()) + 4 * (3 * lnd[r].size() + 2) +
                       4 * (size_t)(ncol + 1) + 32;
      need = std::max(need, b);
    }
    if (need > size_t(200) * 1024) return;
    std::vector<int32_t> fnd, flrp, furp, fcp;
    std::vector<uint16_t> flcol, fucol;
    std::vector<double> flval, fuval;
    std::vector<int64_t> ond(CS + 1, 0), ol(CS + 1, 0), ou(CS + 1, 0);
    for (int64_t r = 0; r < CS; ++r) {
      ond[r + 1] = ond[r] + (int64_t)lnd[r].size();
      ol[r + 1] = ol[r] + (int64_t)llval[r].size();
      ou[r + 1] = ou[r] + (int64_t)luval[r].size();
      fnd.insert(fnd.end(), lnd[r].begin(), lnd[r].end());
      flrp.insert(flrp.end(), llrp[r].begin(), llrp[r].end());  // nloc+1 entries per CTA: offset ond[r] + r
      furp.insert(furp.end(), lurp[r].begin(), lurp[r].end());
      fcp.insert(fcp.end(), lcp[r].begin(), lcp[r].end());
      flcol.insert(flcol.end(), llcol[r].begin(), llcol[r].end());
      fucol.insert(fucol.end(), lucol[r].begin(), lucol[r].end());
      flval.insert(flval.end(), llval[r].begin(), llval[r].end());
      fuval.insert(fuval.end(), luval[r].begin(), luval[r].end());
    }
    auto up = [](auto& dst, const auto& src) {
      using T = typename std::decay_t<decltype(src)>::value_type;
      dst = std::decay_t<decltype(dst)>(src.size() + 1);
      if (!src.empty()) CAMG_CUDA(cudaMemcpy(dst.p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
    };
    up(cl_nd, fnd);
    up(cl_lrp, flrp);
    up(cl_urp, furp);
    up(cl_cp, fcp);
    up(cl_lcol, flcol);
    up(cl_ucol, fucol);
    up(cl_lval, flval);
    up(cl_uval, fuval);
    up(cl_offnd, ond);
    up(cl_offl, ol);
    up(cl_offu, ou);
    cl_smem = need;
    cl_avg = n ? double(lrp[n] + urp[n]) / (2.0 * n) : 0.0;
    cl = true;
  }

  // x = `sweeps` ILU(0) sweeps on S x = rc from zero
  void run(const Csr* S, const double* rc, double* x, int sweeps, cudaStream_t s) {
    const int nc = colors();
    if (cl && sweeps == 1) {
      dispatch_g<LaunchIluCl>(cl_avg, (int)n, nc, cl_nd.p, cl_lrp.p, cl_lcol.p, cl_lval.p, cl_urp.p, cl_ucol.p,
                              cl_uval.p, cl_offnd.p, cl_offl.p, cl_offu.p, cl_cp.p, cl_smem, rc, udiag.p, x, s);
      return;
    }
    for (int k = 0; k < sweeps; ++k) {
      const bool res = k > 0;
      for (int c = 0; c < nc; ++c)
        dispatch_g<LaunchIluPass>(std::max(L->avg_row, res ? S->avg_row : 0.0), L.get(), S, nodes.p + col_ptr[c],
                                  col_ptr[c + 1] - col_ptr[c], true, res, rc, udiag.p, y.p, z.p, x, s);
      for (int c = nc - 1; c >= 0; --c)
        dispatch_g<LaunchIluPass>(U->avg_row, U.get(), S, nodes.p + col_ptr[c], col_ptr[c + 1] - col_ptr[c], false,
                                  res, rc, udiag.p, y.p, z.p, x, s);
    }
  }
};

// pred_update: out = x + alpha du (and, when uh != null, uh = x + du)
__global__ void k_pred_update(int64_t n, const double* __restrict__ x, const double* __restrict__ du, double alpha,
                              double* __restrict__ uh, double* __restrict__ out) {
  CAMG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x ? x[i] : 0.0;
    if (uh) uh[i] = xi + du[i];
    out[i] = uh ? xi + alpha * du[i] : xi + du[i];
  }
}

struct ScalarHier;
const double* scalar_run(ScalarHier* H, const double* b, cudaStream_t s);
void scalar_work_slots(ScalarHier* H, std::vector<DBuf<double>*>& v);

// ---------------------------------------------------------------------------
// level

struct Level {
  int64_t nu = 0, nl = 0, n = 0;
  camg_smoother_cfg cfg{};
  int pre = 1, post = 1;
  Csr* A = nullptr;    // merged [[K,B1],[B2,-Cz]]
  bool owns_A = true;
  camg_csr op_handle{nullptr};  // borrowed view handed out by camg_level_operator
  Csr* B1 = nullptr;   // copy (interface rows)
  Csr* S = nullptr;    // S~
  DBuf<int64_t> b1_rows;
  int64_t n_b1_rows = 0;
  DBuf<double> dinv_p, ainv, dinv_c;
  // multicolour Gauss-Seidel corrector on S~ (point colouring)
  McgsK cgs;
  // multicolour ILU(0) corrector on S~
  McIlu cilu;
  // multicolour Gauss-Seidel predictor on K
  McgsK gs;
  // external predictor solver (nested preconditioner: scalar AMG V-cycle on
  // K, hierarchy.py:364-371 via smoothers.py:277-278); borrowed
  ScalarHier* inner = nullptr;
  // Overlap of a step's lambda side (latency-bound: B2/Cz rows, the S~
  // corrector, lambda update, interface-row B1 correction) with the next
  // bandwidth-bound [K | B1] pass: that chain runs on `side`, and the next
  // pass first streams the SELL slices whose rows read no interface row and
  // no multiplier (sl_indep), then waits for the chain and streams the rest
  // (sl_dep).  Same arithmetic per row, so results are bit-identical.
  bool overlap = false;
  bool pending = false;  // a lambda-side chain runs on `side`
  DBuf<int32_t> sl_indep, sl_dep;
  int64_t n_indep = 0, n_dep = 0;
  // the same lists as work items of the passes with x != 0 (sell_compact_list: group followers dropped)
  DBuf<int32_t> wi_indep, wi_dep;
  DBuf<uint8_t> wm_indep, wm_dep;
  DBuf<int32_t> wd_indep, wd_dep;
  int64_t nw_indep = 0, nw_dep = 0;
  void pass_lists(bool zero, bool dep, const int32_t*& list, int64_t& n, const uint8_t*& lmode,
                  const int32_t*& ldist) const {
    const bool wi = !zero && (dep ? wi_dep.p : wi_indep.p) != nullptr;
    list = wi ? (dep ? wi_dep.p : wi_indep.p) : (dep ? sl_dep.p : sl_indep.p);
    n = wi ? (dep ? nw_dep : nw_indep) : (dep ? n_dep : n_indep);
    lmode = wi ? (dep ? wm_dep.p : wm_indep.p) : nullptr;
    ldist = wi ? (dep ? wd_dep.p : wd_indep.p) : nullptr;
  }
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // Chebyshev predictor: d_k = c1[k] d_{k-1} + c2[k] D^-1 r_k, y_{k+1} = y_k + d_k
  double cheb_lmax = 0.0;
  std::vector<double> cheb_c1, cheb_c2;
  DBuf<double> w_cd[2];
  // direct corrector
  DBuf<double> corr_lu;
  DBuf<int32_t> corr_piv;
  // reference-semantics inner solves: lexicographic sgs / ilu0 predictor on
  // K (pps, on the level's own copy of K) and corrector on S~ (cps)
  PointSolver pps, cps;
  std::unique_ptr<Csr> K_own;
  // dense LU of K: the `direct` predictor and the exact A^-1 of a_hat_mode
  // "exact" (smoothers.py:182-183, 272-273; factors from the host)
  DBuf<double> k_lu;
  DBuf<int32_t> k_piv;
  bool exact = false;
  // dense path: mult diag(ainv) B1 (L U)^-1 on the interface rows (n_b1 x nl),
  // so the B1 correction is part of the corrector GEMV
  DBuf<double> dense_b1;
  // transfer (merged block-diagonal)
  Csr* P = nullptr;
  Csr* R = nullptr;
  int64_t nc = 0;
  int64_t nnz_top = 0;  // entries of the [K | B1] rows
  // work vectors
  DBuf<double> w_du, w_du2, w_ru, w_rc, w_dl, w_dl2, w_rl, w_tmp;
  Sell* alt_sell = nullptr;  // streaming-layout mirror of A's rows (camg_level_fine_pass mode | 0x100)
  ~Level() {
    delete alt_sell;
    if (owns_A) delete A;
    delete B1; delete S; delete P; delete R;
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }

  // order stream s after the pending lambda-side chain
  void join(cudaStream_t s) {
    if (!pending) return;
    CAMG_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    pending = false;
  }

  // fused pass over the [K | B1] rows reading x = [xu; xl]: with a pending
  // lambda-side chain, the independent slices go first
  void top_pass(const RowEpi& e, const double* xu, const double* xl, bool zero, cudaStream_t s) {
    if (!pending || !ovl()) {
      join(s);
      resid_rows(A, int64_t(0), nu, xu, xl, nu, e, zero, s);
      return;
    }
    const SellEpi se = sell_epi(e);
    const int32_t *li, *ld;
    const uint8_t* lm;
    int64_t ln;
    pass_lists(zero, false, li, ln, lm, ld);
    sell_launch(A->sell, 1, zero, xu, xl, nu, se, s, li, ln, lm, ld);
    join(s);
    pass_lists(zero, true, li, ln, lm, ld);
    sell_launch(A->sell, 1, zero, xu, xl, nu, se, s, li, ln, lm, ld);
  }

  void alloc_work() {
    w_du = DBuf<double>(n);
    w_du2 = DBuf<double>(n);
    w_ru = DBuf<double>(nu + 1);
    w_rc = DBuf<double>(nl + 1);
    w_dl = DBuf<double>(nl + 1);
    w_dl2 = DBuf<double>(nl + 1);
    w_rl = DBuf<double>(nl + 1);
    w_tmp = DBuf<double>(n);
  }

  // corrector: dl = C^-1 rc (jacobi sweeps from zero or dense LU)
  double* corrector(const double* rc, cudaStream_t s) {
    if (nl == 0) return w_dl.p;
    if (cfg.corr_kind == CAMG_PT_DIRECT) {
      CAMG_CHECK(corr_lu.p != nullptr, CAMG_ERR_SETUP, "direct corrector factors were not set");
      lu_solve((int)nl, corr_lu.p, corr_piv.p, rc, w_dl.p, s);
      return w_dl.p;
    }
    if (cfg.corr_kind == CAMG_PT_MCGS) {
      // reference SSOR (smoothers.py:155-164, 189-191) on the node-colour
      // permuted S~, from zero
      cgs.init(nullptr, rc, w_dl.p, s);
      cgs.run(true, S, nullptr, rc, dinv_c.p, w_dl.p, cfg.corr_sweeps, s);
      return w_dl.p;
    }
    if (cfg.corr_kind == CAMG_PT_MCILU0) {
      // reference ILU(0) sweeps (smoothers.py:195-197) on the colour-permuted S~, from zero
      cilu.run(S, rc, w_dl.p, cfg.corr_sweeps, s);
      return w_dl.p;
    }
    if (cfg.corr_kind == CAMG_PT_SGS || cfg.corr_kind == CAMG_PT_ILU0) {
      // the reference's lexicographic sweeps on S~ from zero (smoothers.py:197-199)
      cps.smooth(nullptr, rc, w_dl.p, s);
      return w_dl.p;
    }
    double* cur = w_dl.p;
    double* nxt = w_dl2.p;
    dispatch_g<LaunchCorr>(S->avg_row, S, rc, dinv_c.p, nullptr, cur, true, s);
    for (int k = 1; k < cfg.corr_sweeps; ++k) {
      dispatch_g<LaunchCorr>(S->avg_row, S, rc, dinv_c.p, cur, nxt, false, s);
      std::swap(cur, nxt);
    }
    return cur;
  }

  int pred_colors() const { return gs.colors(); }
  // CAMG_LAM_FUSED: 0 no fused cluster kernel (k_lam_ilu_cl), 1 (the
  // default) on levels without the overlapped lambda stream, 2 on all
  // levels, 3 on all levels with the overlap turned off where it would run
  static int lam_mode() {
    const char* e = getenv("CAMG_LAM_FUSED");
    return e ? atoi(e) : 1;
  }
  bool mcilu_once() const { return cfg.corr_kind == CAMG_PT_MCILU0 && cfg.corr_sweeps == 1 && !exact; }
  // the lambda-side chain runs on the second stream, overlapping the next pass
  bool ovl() const {
    return overlap && !(lam_mode() == 3 && mcilu_once() && (cilu.fused || cilu.dense_inv.p != nullptr));
  }
  // small S~: the zero-start MC-ILU(0) sweep as one GEMV with (L U)^-1
  bool lam_dense() const { return mcilu_once() && cilu.dense_inv.p != nullptr && !ovl(); }
  // the one-launch sync-free lambda engine (CAMG_LAM_ENGINE: 0 off -- the
  // default: measured slower, C5 19.0 -> 21.8 ms, C3 1.51 -> 2.41 ms, the
  // flag hand-offs per dependency level cost more than the PDL-chained
  // colour passes --, 1 on the levels that would run colour passes, 2
  // everywhere)
  bool lam_engine() const {
    if (!mcilu_once() || !cilu.eng_sync.p) return false;
    const char* e = getenv("CAMG_LAM_ENGINE");
    const int m = e ? atoi(e) : 0;
    if (m == 0) return false;
    if (m == 2) return true;
    return !lam_dense() && !lam_fused();
  }
  // the one-cluster ILU(0) sweep
  bool lam_fused() const {
    if (!mcilu_once() || !cilu.fused) return false;
    const int m = lam_mode();
    return m == 2 || m == 3 || (m == 1 && !ovl());
  }
  bool pred_generic() const {
    return cfg.kind != CAMG_BRAESS_SARAZIN &&
           (cfg.pred_kind == CAMG_PT_DIRECT || cfg.pred_kind == CAMG_PT_SGS || cfg.pred_kind == CAMG_PT_ILU0);
  }

  // MC-SGS predictor in iterate form: y_0 = u, then pred_sweeps forward +
  // backward colour sweeps of Gauss-Seidel on K y = b_u - B1 lam -- the
  // reference's zero-start SSOR correction on r_u (smoothers.py:186-199) with
  // u added back, on the colour-permuted K
  void gs_predict(const double* x, const double* b, double* y, int sweeps, cudaStream_t s) {
    const double* xl = x ? x + nu : nullptr;
    gs.init(x, b, y, s);
    if (gs.sell && xl && n_b1_rows) {
      note_launch();
      launch_k(k_b1_sub, grid_for(n_b1_rows * 8, 256), 256, 0, s, view(B1), b1_rows.p, n_b1_rows, xl, gs.g.p);
    }
    gs.run(x == nullptr, A, xl, b, dinv_p.p, y, sweeps, s);
  }

  // one algorithmic smoother step: xo = step(x, b); x == nullptr means zero
  void step(const double* x, const double* b, double* xo, cudaStream_t s) {
    const bool zero = (x == nullptr);
    const double* xu = x;
    const double* xl = x ? x + nu : nullptr;
    const int kind = cfg.kind;
    const int sp = cfg.pred_sweeps;
    const double alpha = cfg.alpha;
    // u-half: the predicted displacement the lambda side is coupled to
    const double* uh = xo;
    if (kind == CAMG_BRAESS_SARAZIN) {
      // u_half = u + (A^-1 r_u) / alpha   (smoothers.py:296)
      RowEpi e{b, x, nullptr, ainv.p, nullptr, xo, 1.0 / alpha};
      top_pass(e, xu, xl, zero, s);
    } else if (inner || pred_generic()) {
      join(s);
      // du = predictor.apply(r_u), r_u = b_u - K u - B1 lam (smoothers.py:285-314):
      // the nested preconditioner's inner AMG (predictor_solver), a dense LU
      // of K (direct) or lexicographic sgs / ilu0 sweeps on K from zero;
      // SIMPLE: u_half = u + du; Uzawa: u + alpha du
      RowEpi e{b, x, w_ru.p, nullptr, nullptr, nullptr, 0.0};
      resid_rows(A, int64_t(0), nu, xu, xl, nu, e, zero, s);
      const double* du = w_du.p;
      if (inner) {
        du = scalar_run(inner, w_ru.p, s);
      } else if (cfg.pred_kind == CAMG_PT_DIRECT) {
        CAMG_CHECK(k_lu.p != nullptr, CAMG_ERR_SETUP, "direct predictor factors were not set");
        lu_solve((int)nu, k_lu.p, k_piv.p, w_ru.p, w_du.p, s);
      } else {
        pps.smooth(nullptr, w_ru.p, w_du.p, s);
      }
      note_launch();
      if (kind == CAMG_UZAWA) {
        launch_k(k_pred_update, grid_for(nu, 256), 256, 0, s, nu, xu, du, alpha, w_du2.p, xo);
        uh = w_du2.p;
      } else {
        launch_k(k_pred_update, grid_for(nu, 256), 256, 0, s, nu, xu, du, 1.0, nullptr, xo);
      }
    } else if (cfg.pred_kind == CAMG_PT_MCGS) {
      // Uzawa keeps y for the lambda side and relaxes u_new = u + alpha (y - u)
      join(s);
      double* y = (kind == CAMG_UZAWA) ? w_du.p : xo;
      gs_predict(x, b, y, sp, s);
      if (kind == CAMG_UZAWA) {
        note_launch();
        launch_k(k_relax, grid_for(nu, 256), 256, 0, s, nu, xu, y, alpha, xo);
        uh = y;
      }
    } else {
      // Jacobi predictor in iterate form: y_0 = u, y_k = y_{k-1} + w D^-1
      // (b_u - K y_{k-1} - B1 lam) -- the reference's zero-start correction
      // sweeps on r_u (smoothers.py:186-199, 285-314) with u added back, so
      // no residual / increment vectors are stored.  Uzawa keeps y_sp for the
      // lambda side and relaxes u_new = u + alpha (y_sp - u).
      // Chebyshev: the same pass with d_k = c1 d_{k-1} + c2 D^-1 r_k kept
      // between steps (w_cd ping-pong)
      const bool cheb = cfg.pred_kind == CAMG_PT_CHEBYSHEV;
      const double* y = x;
      double* bufs[2] = {w_du.p, w_du2.p};
      for (int k = 0; k < sp; ++k) {
        const bool last = (k == sp - 1);
        double* dst = bufs[k & 1];
        RowEpi e{b, y, nullptr, dinv_p.p, nullptr, nullptr, 1.0};
        if (cheb) {
          e.c1 = cheb_c1[k];
          e.c2 = cheb_c2[k];
          e.dprev = k ? w_cd[(k - 1) & 1].p : nullptr;
          if (!last) e.out_d = w_cd[k & 1].p;
        }
        if (!last) {
          e.out_x = dst;
        } else if (kind == CAMG_UZAWA) {
          e.out_y = dst;
          e.out_x = xo;
          e.x0 = x;
          e.xmode = 1;
          e.coef = alpha;
          uh = dst;
        } else {
          e.out_x = xo;
        }
        if (k == 0) top_pass(e, y, xl, y == nullptr, s);
        else resid_rows(A, int64_t(0), nu, y, xl, nu, e, false, s);
        y = dst;
      }
    }
    if (nl == 0) return;
    CAMG_CHECK(S != nullptr, CAMG_ERR_SETUP, "S~ was not set (a_hat_mode exact: camg_level_set_schur)");
    join(s);
    cudaStream_t ls = s;
    if (ovl()) {  // fork the lambda side onto `side`
      CAMG_CUDA(cudaEventRecord(ev_fork, s));
      CAMG_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
      ls = side;
    }
    // lambda side: rc = B2 u_half - Cz lam - b_lam = -(b_lam + Cz lam - B2 u_half)
    const double cl = (kind == CAMG_BRAESS_SARAZIN) ? 1.0 : alpha;
    const double mult = (kind == CAMG_BRAESS_SARAZIN) ? 1.0 / alpha : alpha;
    if (lam_engine()) {
      cilu.run_engine(A, nu, uh, xl, b + nu, xo, w_dl.p, cl, B1, b1_rows.p, kind != CAMG_UZAWA ? n_b1_rows : 0,
                      ainv.p, mult, ls);
    } else if (lam_dense() || lam_fused()) {
      // rc (wide kernel), then the ILU(0) sweep + lambda update (one GEMV
      // with the explicit inverse, or one cluster), then the interface-row
      // B1 correction (wide kernel)
      dispatch_g<LaunchLamRhs>(A->avg_row, A, nu, nl, uh, xl, b + nu, w_rc.p, ls);
      const bool b1_fused = lam_dense() && kind != CAMG_UZAWA && n_b1_rows && dense_b1.p;
      if (lam_dense())
        cilu.run_dense(w_rc.p, xl, xo + nu, w_dl.p, cl, ls, b1_fused ? dense_b1.p : nullptr, b1_rows.p, n_b1_rows, xo);
      else cilu.run_fused(w_rc.p, xl, xo + nu, w_dl.p, cl, ls);
      if (kind != CAMG_UZAWA && n_b1_rows && !b1_fused) {
        note_launch();
        launch_k(k_b1_correct, grid_for(n_b1_rows * 8, 256), 256, 0, ls, view(B1), b1_rows.p, n_b1_rows, ainv.p,
                 (const double*)w_dl.p, mult, xo);
      }
    } else {
      dispatch_g<LaunchLamRhs>(A->avg_row, A, nu, nl, uh, xl, b + nu, w_rc.p, ls);
      double* dl = corrector(w_rc.p, ls);
      note_launch();
      launch_k(k_lam_update, grid_for(nl, 256), 256, 0, ls, nl, xl, dl, cl, xo + nu);
      if (kind != CAMG_UZAWA && n_b1_rows && exact) {
        // u_new = u_half - alpha K^-1 B1 dlam (a_hat_mode "exact", smoothers.py:313)
        CAMG_CHECK(k_lu.p != nullptr, CAMG_ERR_SETUP, "exact a_hat mode needs the LU factors of K");
        spmv(B1, 1.0, dl, 0.0, w_ru.p, ls);
        lu_solve((int)nu, k_lu.p, k_piv.p, w_ru.p, w_du.p, ls);
        vec_axpy(nu, -alpha, w_du.p, xo, ls);
      } else if (kind != CAMG_UZAWA && n_b1_rows) {
        // u_new = u_half - c A^-1 B1 dlam on the interface rows
        note_launch();
        launch_k(k_b1_correct, grid_for(n_b1_rows * 8, 256), 256, 0, ls, view(B1), b1_rows.p, n_b1_rows, ainv.p, dl,
                 mult, xo);
      }
    }
    if (ovl()) {
      CAMG_CUDA(cudaEventRecord(ev_join, side));
      pending = true;
    }
  }

  // BlockSmoother.sweep: outer steps from x (null = zero) into out; out != x
  void sweep(const double* x, const double* b, double* out, cudaStream_t s) {
    const int outer = cfg.outer_sweeps;
    const double* cur = x;
    for (int k = 0; k < outer; ++k) {
      double* dst = ((outer - 1 - k) % 2 == 0) ? out : w_tmp.p;
      step(cur, b, dst, s);
      cur = dst;
    }
  }

  // r = b - A x over all rows (independent slices first while a lambda-side
  // chain is pending)
  void residual(const double* x, const double* b, double* r, cudaStream_t s) {
    RowEpi e{b, nullptr, r, nullptr, nullptr, nullptr, 0.0};
    if (pending && ovl() && x) {
      const SellEpi se = sell_epi(e);
      const int32_t *li, *ld;
      const uint8_t* lm;
      int64_t ln;
      pass_lists(false, false, li, ln, lm, ld);
      sell_launch(A->sell, 1, false, x, nullptr, -1, se, s, li, ln, lm, ld);
      join(s);
      pass_lists(false, true, li, ln, lm, ld);
      sell_launch(A->sell, 1, false, x, nullptr, -1, se, s, li, ln, lm, ld);
      const int64_t done = A->sell->rows();
      if (n > done) dispatch_g<LaunchResid>(A->avg_row, A, done, n - done, x, (const double*)nullptr, n, e, false, s);
      return;
    }
    join(s);
    resid_rows(A, int64_t(0), n, x, (const double*)nullptr, n, e, x == nullptr, s);
  }
};

// ---------------------------------------------------------------------------

static void check_no_zero(const double* d, int64_t n, const char* what) {
  if (n <= 0) return;
  DBuf<unsigned long long> first(1);
  unsigned long long init = ~0ull;
  CAMG_CUDA(cudaMemcpy(first.p, &init, sizeof(init), cudaMemcpyHostToDevice));
  note_launch();
  k_first_zero<<<grid_for(n, 256), 256>>>(n, d, first.p);
  unsigned long long h = 0;
  CAMG_CUDA(cudaMemcpy(&h, first.p, sizeof(h), cudaMemcpyDeviceToHost));
  if (h != ~0ull) throw Error(CAMG_ERR_SINGULAR, std::string(what) + ": zero diagonal in row " + std::to_string(h));
}



double lambda_max_dinv(const Csr* A, const double* d, int iters, cudaStream_t s);

// Chebyshev polynomial of D^-1 K (degree = predictor sweeps) on
// [lmax/kChebRatio, kChebBoost*lmax], lmax by 10 power steps (the
// smoothed-aggregation estimate, transfer.py:148-161):
//   theta = (b+a)/2, delta = (b-a)/2, sigma = theta/delta, rho_0 = 1/sigma
//   d_0 = D^-1 r_0 / theta; d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k/delta) D^-1 r_k,
//   rho_k = 1/(2 sigma - rho_{k-1})
static void cheb_coefficients(double lmax, int degree, std::vector<double>& c1, std::vector<double>& c2) {
  const double beta = kChebBoost * lmax, alpha = beta / kChebRatio;
  const double theta = 0.5 * (beta + alpha), delta = 0.5 * (beta - alpha), sigma = theta / delta;
  c1.assign(degree, 0.0);
  c2.assign(degree, 0.0);
  double rho = 1.0 / sigma;
  c2[0] = 1.0 / theta;
  for (int k = 1; k < degree; ++k) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    c1[k] = rn * rho;
    c2[k] = 2.0 * rn / delta;
    rho = rn;
  }
}

static void setup_chebyshev(Level* L, const Csr* K, const double* dK, int degree, cudaStream_t s) {
  L->cheb_lmax = lambda_max_dinv(K, dK, 10, s);
  cheb_coefficients(L->cheb_lmax, degree, L->cheb_c1, L->cheb_c2);
  if (degree > 1) {
    L->w_cd[0] = DBuf<double>(L->nu + 1);
    L->w_cd[1] = DBuf<double>(L->nu + 1);
  }
}

// rows r < nu with a multiplier column (B1 part of the merged rows)
__global__ void k_iface_rows(CsrView A, int64_t nu, int8_t* __restrict__ iface) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nu; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = A.rowptr[r], e = A.rowptr[r + 1];
    iface[r] = (e > b && A.col[e - 1] >= nu) ? 1 : 0;
  }
}

// rows that read an interface row or a multiplier
__global__ void k_dep_rows(CsrView A, int64_t nu, const int8_t* __restrict__ iface, int8_t* __restrict__ dep) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nu; r += (int64_t)gridDim.x * blockDim.x) {
    int8_t d = iface[r];
    for (int64_t p = A.rowptr[r]; p < A.rowptr[r + 1] && !d; ++p) {
      const int32_t c = A.col[p];
      if (c < nu && iface[c]) d = 1;
    }
    dep[r] = d;
  }
}

__global__ void k_dep_slices(const int8_t* __restrict__ dep, int64_t nu, int64_t rows_per_slice, int64_t nslices,
                             int8_t* __restrict__ ds) {
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nslices; sl += (int64_t)gridDim.x * blockDim.x) {
    int8_t d = 0;
    const int64_t r1 = min(nu, (sl + 1) * rows_per_slice);
    for (int64_t r = sl * rows_per_slice; r < r1 && !d; ++r) d = dep[r];
    ds[sl] = d;
  }
}

static void setup_overlap(Level* L) {
  const Sell* S = L->A->sell;
  const char* env = getenv("CAMG_OVERLAP");
  if ((env && env[0] == '0') || !S || L->nl == 0 || S->rows() != L->nu || L->cfg.kind == CAMG_UZAWA) return;
  const int64_t nu = L->nu;
  DBuf<int8_t> iface(nu + 1), dep(nu + 1), ds(S->nslices + 1);
  note_launch(3);
  k_iface_rows<<<grid_for(nu, 256), 256>>>(view(L->A), nu, iface.p);
  k_dep_rows<<<grid_for(nu, 256), 256>>>(view(L->A), nu, iface.p, dep.p);
  k_dep_slices<<<grid_for(S->nslices, 256), 256>>>(dep.p, nu, 32 * (int64_t)S->br, S->nslices, ds.p);
  CAMG_LAUNCH_CHECK();
  std::vector<int8_t> h(S->nslices);
  CAMG_CUDA(cudaMemcpy(h.data(), ds.p, S->nslices, cudaMemcpyDeviceToHost));
  std::vector<int32_t> ind, dp;
  for (int64_t i = 0; i < S->nslices; ++i) (h[i] ? dp : ind).push_back((int32_t)i);
  L->n_indep = (int64_t)ind.size();
  L->n_dep = (int64_t)dp.size();
  L->sl_indep = DBuf<int32_t>(ind.size() + 1);
  L->sl_dep = DBuf<int32_t>(dp.size() + 1);
  if (!ind.empty()) CAMG_CUDA(cudaMemcpy(L->sl_indep.p, ind.data(), sizeof(int32_t) * ind.size(), cudaMemcpyHostToDevice));
  if (!dp.empty()) CAMG_CUDA(cudaMemcpy(L->sl_dep.p, dp.data(), sizeof(int32_t) * dp.size(), cudaMemcpyHostToDevice));
  if (S->witems) {
    // work items of the passes with x != 0: the followers of the uniform-slice groups leave the lists
    auto items = [&](std::vector<int32_t>& list, DBuf<int32_t>& wi, DBuf<uint8_t>& wm, DBuf<int32_t>& wd,
                     int64_t& nw) {
      std::vector<uint8_t> mode;
      std::vector<int32_t> dist;
      sell_compact_list(S, list, mode, dist);
      nw = (int64_t)list.size();
      wi = DBuf<int32_t>(list.size() + 1);
      wm = DBuf<uint8_t>(list.size() + 1);
      wd = DBuf<int32_t>(list.size() + 1);
      if (!list.empty()) {
        CAMG_CUDA(cudaMemcpy(wi.p, list.data(), sizeof(int32_t) * list.size(), cudaMemcpyHostToDevice));
        CAMG_CUDA(cudaMemcpy(wm.p, mode.data(), list.size(), cudaMemcpyHostToDevice));
        CAMG_CUDA(cudaMemcpy(wd.p, dist.data(), sizeof(int32_t) * list.size(), cudaMemcpyHostToDevice));
      }
    };
    items(ind, L->wi_indep, L->wm_indep, L->wd_indep, L->nw_indep);
    items(dp, L->wi_dep, L->wm_dep, L->wd_dep, L->nw_dep);
  }
  {
    // the lambda-side stream at the greatest priority (graph nodes keep it:
    // cudaGraphInstantiateFlagUseNodePriority): its short chain kernels take
    // the CTA slots the concurrent pass frees first (C5 19.19 -> 18.98 ms,
    // C3 1.565 -> 1.507 ms); CAMG_SIDE_PRIO=0 restores equal priority
    const char* pe = getenv("CAMG_SIDE_PRIO");
    int lo = 0, hi = 0;
    CAMG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CAMG_CUDA(cudaStreamCreateWithPriority(&L->side, cudaStreamNonBlocking, (pe && pe[0] == '0') ? lo : hi));
  }
  CAMG_CUDA(cudaEventCreateWithFlags(&L->ev_fork, cudaEventDisableTiming));
  CAMG_CUDA(cudaEventCreateWithFlags(&L->ev_join, cudaEventDisableTiming));
  L->overlap = true;
  if (getenv("CAMG_DEBUG"))
    fprintf(stderr, "[camg] overlap: %lld independent / %lld dependent slices\n", (long long)L->n_indep,
            (long long)L->n_dep);
}

// corrector structures on S~ (colourings, factors, inverse diagonal)
static void setup_corrector(Level* L) {
  const camg_smoother_cfg& cfg = L->cfg;
  const int64_t nl = L->nl;
  cudaStream_t s = 0;
  if (nl == 0) return;
  // point colouring of S~: the multiplier-node graph needs as many colours
  // (16 on C5) and the per-node kernels measured slower
  if (cfg.corr_kind == CAMG_PT_MCGS) L->cgs.setup(L->S, 1, s);
  if (cfg.corr_kind == CAMG_PT_MCILU0) L->cilu.setup(L->S, s);
  if (cfg.corr_kind == CAMG_PT_SGS || cfg.corr_kind == CAMG_PT_ILU0)
    L->cps.setup(L->S, cfg.corr_kind, cfg.corr_sweeps, cfg.corr_damping);
  if (cfg.corr_kind == CAMG_PT_JACOBI || cfg.corr_kind == CAMG_PT_MCGS) {
    DBuf<double> dS(nl + 1);
    csr_diagonal(L->S, 0, dS.p, s);
    CAMG_CUDA(cudaDeviceSynchronize());
    check_no_zero(dS.p, nl, "jacobi");
    L->dinv_c = DBuf<double>(nl + 1);
    note_launch();
    k_scaled_recip<<<grid_for(nl, 256), 256>>>(nl, dS.p, cfg.corr_damping, 1.0, L->dinv_c.p);
  }
  CAMG_CUDA(cudaDeviceSynchronize());
}

Level* level_create(const Csr* K, const Csr* B1, const Csr* B2, const Csr* Cz, const camg_smoother_cfg& cfg, int pre,
                    int post, Csr* A_shared) {
  CAMG_CHECK(cfg.kind >= CAMG_UZAWA && cfg.kind <= CAMG_SIMPLEC, CAMG_ERR_CONFIG, "unknown block smoother kind");
  CAMG_CHECK(cfg.alpha > 0.0, CAMG_ERR_CONFIG, "alpha must be positive");
  CAMG_CHECK(cfg.outer_sweeps >= 1, CAMG_ERR_CONFIG, "outer_sweeps must be >= 1");
  CAMG_CHECK(cfg.kind == CAMG_BRAESS_SARAZIN || (cfg.pred_kind >= CAMG_PT_JACOBI && cfg.pred_kind <= CAMG_PT_MCGS),
             CAMG_ERR_CONFIG, "GPU predictor supports jacobi, sgs, ilu0, direct, chebyshev and mcgs");
  CAMG_CHECK(cfg.pred_sweeps >= 1, CAMG_ERR_CONFIG, "predictor sweeps must be >= 1");
  CAMG_CHECK(cfg.corr_kind >= CAMG_PT_JACOBI && cfg.corr_kind <= CAMG_PT_MCILU0 && cfg.corr_kind != CAMG_PT_CHEBYSHEV,
             CAMG_ERR_CONFIG, "GPU corrector supports jacobi, sgs, ilu0, direct, mcgs and mcilu0");
  CAMG_CHECK(cfg.a_hat_mode >= CAMG_AHAT_PLAIN && cfg.a_hat_mode <= CAMG_AHAT_EXACT, CAMG_ERR_CONFIG,
             "unknown a_hat mode");
  cudaStream_t s = 0;
  std::unique_ptr<Level> L(new Level());
  L->cfg = cfg;
  L->pre = pre;
  L->post = post;
  L->nu = K->n_rows;
  L->nl = Cz->n_rows;
  L->n = L->nu + L->nl;
  if (A_shared) {
    CAMG_CHECK(A_shared->n_rows == K->n_rows + Cz->n_rows && A_shared->n_cols == A_shared->n_rows,
               CAMG_ERR_DIMENSION, "merged operator does not match the blocks");
    L->A = A_shared;
    L->owns_A = false;
  } else {
    L->A = csr_saddle_merge(K, B1, B2, Cz, s);
  }
  L->B1 = csr_copy(B1, s);
  L->nnz_top = read_i64(L->A->rowptr + L->nu);
  const int64_t nu = L->nu, nl = L->nl;
  // diagonals
  DBuf<double> dK(nu + 1);
  csr_diagonal(K, 0, dK.p, s);
  const int mode = (cfg.kind == CAMG_SIMPLEC) ? CAMG_AHAT_ABS_ROWSUM
                   : (cfg.kind == CAMG_BRAESS_SARAZIN) ? CAMG_AHAT_PLAIN
                                                       : cfg.a_hat_mode;
  L->exact = mode == CAMG_AHAT_EXACT;
  DBuf<double> ahat(nu + 1);
  if (L->exact) {
    // A^ = K: A^-1 applications are LU solves, S~ comes from camg_level_set_schur
    note_launch();
    k_copy<<<grid_for(nu, 256), 256>>>(nu, dK.p, ahat.p);
  } else if (mode == CAMG_AHAT_ABS_ROWSUM) {
    csr_diagonal(K, 1, ahat.p, s);
    CAMG_CUDA(cudaDeviceSynchronize());
    check_no_zero(ahat.p, nu, "abs_rowsum lumping");
  } else {
    CAMG_CUDA(cudaMemcpy(ahat.p, dK.p, sizeof(double) * nu, cudaMemcpyDeviceToDevice));
    check_no_zero(ahat.p, nu, "a_hat");
  }
  L->ainv = DBuf<double>(nu + 1);
  note_launch();
  k_scaled_recip<<<grid_for(nu, 256), 256>>>(nu, ahat.p, 1.0, 1.0, L->ainv.p);
  if (cfg.kind != CAMG_BRAESS_SARAZIN) {
    check_no_zero(dK.p, nu, "jacobi");
    L->dinv_p = DBuf<double>(nu + 1);
    const bool cheb = cfg.pred_kind == CAMG_PT_CHEBYSHEV;
    note_launch();
    k_scaled_recip<<<grid_for(nu, 256), 256>>>(nu, dK.p, cheb ? 1.0 : cfg.pred_damping, 1.0, L->dinv_p.p);
    if (cheb) setup_chebyshev(L.get(), K, dK.p, cfg.pred_sweeps, s);
  }
  // Schur approximation (smoothers.py:255-267); exact: set later
  if (!L->exact) {
    DBuf<double> ainv_s(nu + 1);
    double scale = 1.0;
    if (cfg.kind == CAMG_BRAESS_SARAZIN) {
      note_launch();
      k_scaled_recip<<<grid_for(nu, 256), 256>>>(nu, ahat.p, 1.0, cfg.alpha, ainv_s.p);
    } else {
      CAMG_CUDA(cudaMemcpy(ainv_s.p, L->ainv.p, sizeof(double) * nu, cudaMemcpyDeviceToDevice));
      if (cfg.kind == CAMG_SIMPLE || cfg.kind == CAMG_SIMPLEC) scale = cfg.alpha;
    }
    L->S = schur(B2, Cz, B1, ainv_s.p, scale, s);
  }
  if (cfg.kind != CAMG_BRAESS_SARAZIN && cfg.pred_kind == CAMG_PT_MCGS) L->gs.setup(K, cfg.node_block, s);
  if (L->pred_generic() && cfg.pred_kind != CAMG_PT_DIRECT) {
    L->K_own.reset(csr_copy(K, s));
    L->pps.setup(L->K_own.get(), cfg.pred_kind, cfg.pred_sweeps, cfg.pred_damping);
  }
  if (L->S) setup_corrector(L.get());
  // nonempty rows of B1
  {
    DBuf<int32_t> flags(nu + 1);
    note_launch();
    k_nonempty_flags<<<grid_for(nu, 256), 256>>>(L->B1->rowptr, nu, flags.p);
    DBuf<int64_t> idx(nu + 1), out(nu + 1), nsel(1);
    note_launch();
    auto it = cub::CountingInputIterator<int64_t>(0);
    size_t tmp = 0;
    CAMG_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags.p, out.p, nsel.p, nu));
    DBuf<char> t(tmp);
    CAMG_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, it, flags.p, out.p, nsel.p, nu));
    L->n_b1_rows = read_i64(nsel.p);
    L->b1_rows = std::move(out);
  }
  if (!L->exact) setup_overlap(L.get());
  const char* db_env = getenv("CAMG_DENSE_B1");
  if (L->cilu.dense_inv.p && cfg.kind != CAMG_UZAWA && L->n_b1_rows && !L->exact && !(db_env && db_env[0] == '0') &&
      L->n_b1_rows * nl <= (int64_t(1) << 25)) {
    const double mult = (cfg.kind == CAMG_BRAESS_SARAZIN) ? 1.0 / cfg.alpha : cfg.alpha;
    L->dense_b1 = DBuf<double>((size_t)L->n_b1_rows * nl + 1);
    note_launch();
    k_b1_dense<<<grid_for(L->n_b1_rows * nl, 256), 256>>>((int)nl, L->n_b1_rows, L->b1_rows.p, view(L->B1),
                                                          L->ainv.p, mult, L->cilu.dense_inv.p, L->dense_b1.p);
    CAMG_LAUNCH_CHECK();
  }
  L->alloc_work();
  CAMG_CUDA(cudaDeviceSynchronize());
  return L.release();
}

void shift_copy(const int64_t* rp, int64_t n, int64_t add, int64_t* out, const int32_t* col, int64_t nnz, int32_t cadd,
                int32_t* cout, cudaStream_t s);

Csr* block_diag(const Csr* Pu, const Csr* Pl, cudaStream_t s) {
  // [[Pu, 0], [0, Pl]]: reuse the saddle merge with empty off-diagonal blocks
  // is not possible (square check); do it directly.
  const int64_t nu = Pu->n_rows, nl = Pl->n_rows, cu = Pu->n_cols, cl = Pl->n_cols;
  Csr* C = csr_alloc(nu + nl, cu + cl, Pu->nnz + Pl->nnz);
  CAMG_CUDA(cudaMemcpyAsync(C->rowptr, Pu->rowptr, sizeof(int64_t) * (nu + 1), cudaMemcpyDeviceToDevice, s));
  CAMG_CUDA(cudaMemcpyAsync(C->col, Pu->col, sizeof(int32_t) * Pu->nnz, cudaMemcpyDeviceToDevice, s));
  CAMG_CUDA(cudaMemcpyAsync(C->val, Pu->val, sizeof(double) * Pu->nnz, cudaMemcpyDeviceToDevice, s));
  CAMG_CUDA(cudaMemcpyAsync(C->val + Pu->nnz, Pl->val, sizeof(double) * Pl->nnz, cudaMemcpyDeviceToDevice, s));
  shift_copy(Pl->rowptr + 1, nl, Pu->nnz, C->rowptr + nu + 1, Pl->col, Pl->nnz, (int32_t)cu, C->col + Pu->nnz, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  return C;
}

__global__ void k_shift_copy(const int64_t* __restrict__ rp, int64_t n, int64_t add, int64_t* __restrict__ out,
                             const int32_t* __restrict__ col, int64_t nnz, int32_t cadd, int32_t* __restrict__ cout) {
  const int64_t m = n > nnz ? n : nnz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) out[i] = rp[i] + add;
    if (i < nnz) cout[i] = col[i] + cadd;
  }
}

void shift_copy(const int64_t* rp, int64_t n, int64_t add, int64_t* out, const int32_t* col, int64_t nnz, int32_t cadd,
                int32_t* cout, cudaStream_t s) {
  note_launch();
  k_shift_copy<<<grid_for(std::max(n, nnz), 256), 256, 0, s>>>(rp, n, add, out, col, nnz, cadd, cout);
  CAMG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// hierarchy

// A V-cycle workspace: the work vectors of one caller plus the CUDA graph
// recorded over them.  A built hierarchy "may be applied concurrently to
// independent right-hand sides, each application owning its work vectors"
// (SPEC.md:526): every workspace owns a private copy of every vector the
// cycle writes (per-level rhs / iterates / residuals, the smoother's step
// vectors, the multicolour and ILU(0) solve vectors, an inner scalar
// hierarchy's vectors) and its own graph, stream and events, so cycles on
// different workspaces may run at the same time on different streams.  The
// operators, factors and colourings are shared and read-only.  The graph is
// recorded with the workspace's vectors bound in place of the hierarchy's
// own (swapped in under a process-wide lock for the capture only).
struct VcycleWs {
  std::vector<DBuf<double>> bufs;  // one per Hierarchy::work_slots() entry (owned == true)
  bool owned = false;              // false: the hierarchy's own vectors (default workspace)
  DBuf<double> in, out;            // level-0 rhs / result bound into the graph
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaGraphExec_t graph = nullptr;
  int64_t kernels = 0;
  ~VcycleWs() {
    if (graph) cudaGraphExecDestroy(graph);
    if (stream) cudaStreamDestroy(stream);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
};

static std::mutex g_capture_mu;

struct Hierarchy {
  std::vector<Level*> levels;
  int coarse_solver = CAMG_COARSE_MERGED_LU;
  DBuf<double> lu;
  DBuf<int32_t> piv;
  int64_t n_coarse = 0;
  // blocked multi-CTA coarse solve (k_lu_solve_blk): composed row
  // permutation, forward-solve vector, hand-off flags (per workspace)
  bool lu_blk = false;
  DBuf<int32_t> lu_perm;
  DBuf<double> lu_y, lu_flags;
  // explicit inverse of the coarsest operator (k_dense_gemv path) and its
  // refinement vectors (per workspace)
  DBuf<double> cinv, c_x0, c_r;
  // per-level vectors: b (rhs), x[2]
  std::vector<DBuf<double>> vb, vx0, vx1, vr;
  bool use_graph = true;
  VcycleWs def;  // workspace of camg_vcycle (the hierarchy's own vectors)

  // every device vector a V-cycle writes (the per-call state of a workspace)
  std::vector<DBuf<double>*> work_slots() {
    std::vector<DBuf<double>*> v;
    for (size_t l = 0; l < levels.size(); ++l) {
      Level* L = levels[l];
      for (DBuf<double>* b : {&vb[l], &vx0[l], &vx1[l], &vr[l], &L->w_du, &L->w_du2, &L->w_ru, &L->w_rc, &L->w_dl,
                              &L->w_dl2, &L->w_rl, &L->w_tmp, &L->w_cd[0], &L->w_cd[1], &L->gs.g, &L->cgs.g,
                              &L->cilu.y, &L->cilu.z, &L->cilu.eng_sync})
        v.push_back(b);
      if (L->inner) scalar_work_slots(L->inner, v);
      L->pps.work_slots(v);
      L->cps.work_slots(v);
    }
    v.push_back(&lu_y);
    v.push_back(&lu_flags);
    v.push_back(&c_x0);
    v.push_back(&c_r);
    return v;
  }

  void set_coarse_lu(int64_t n, const double* lu_h, const int32_t* piv_h) {
    n_coarse = n;
    lu = DBuf<double>(n * n + 1);
    piv = DBuf<int32_t>(n + 1);
    CAMG_CUDA(cudaMemcpy(lu.p, lu_h, sizeof(double) * n * n, cudaMemcpyHostToDevice));
    CAMG_CUDA(cudaMemcpy(piv.p, piv_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    const int64_t nb = (n + kLuB - 1) / kLuB;
    const char* e = getenv("CAMG_LU_BLOCKED");  // 0: always the one-CTA solve
    const size_t smem_need = sizeof(double) * ((size_t)n * n + 2 * (size_t)n);
    lu_blk = !(e && e[0] == '0') && (n >= kLuBlkMin || (e && e[0] == '1')) && nb <= kLuBlkMaxBlocks &&
             !(smem_need <= size_t(220) * 1024 && !(e && e[0] == '1'));
    if (lu_blk) {
      // x = P b with LAPACK's sequential row swaps composed into one gather
      std::vector<int32_t> idx(n);
      for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
      for (int64_t i = 0; i < n; ++i) std::swap(idx[i], idx[piv_h[i]]);
      lu_perm = DBuf<int32_t>(n + 1);
      CAMG_CUDA(cudaMemcpy(lu_perm.p, idx.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
      lu_y = DBuf<double>(n + 1);
      lu_flags = DBuf<double>(nb + 2);  // 2 nb + 1 unsigned flags
      CAMG_CUDA(cudaMemset(lu_flags.p, 0, sizeof(double) * (nb + 2)));
    }
  }

  void set_coarse_inverse(int64_t n, const double* inv_rowmajor) {
    CAMG_CHECK(n == n_coarse, CAMG_ERR_DIMENSION, "coarse inverse does not match the LU factors");
    CAMG_CHECK(n <= kCoarseInvMax, CAMG_ERR_DIMENSION, "coarse inverse larger than 4096 rows");
    cinv = DBuf<double>(n * n + 1);
    CAMG_CUDA(cudaMemcpy(cinv.p, inv_rowmajor, sizeof(double) * n * n, cudaMemcpyHostToDevice));
    c_x0 = DBuf<double>(n + 1);
    c_r = DBuf<double>(n + 1);
  }

  // LU (and, up to kCoarseInvMax rows, the inverse) of the coarsest merged
  // operator computed on the device (no host LAPACK)
  void coarse_factor(bool inverse) {
    const Csr* A = levels.back()->A;
    const int n = (int)A->n_rows;
    CAMG_CHECK(n >= 1 && n < 46341, CAMG_ERR_DIMENSION, "coarse operator too large for a dense factorization");
    DBuf<double> D((size_t)n * n + 1), lk(n + 1);
    DBuf<int32_t> pv(n + 1);
    CAMG_CUDA(cudaMemset(D.p, 0, sizeof(double) * (size_t)n * n));
    note_launch(2);
    k_csr_to_dense_colmajor<<<grid_for(n, 256), 256>>>(view(A), D.p);
    CAMG_LAUNCH_CHECK();
    int per_sm = 0;
    CAMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_lu, 256, 0));
    const int64_t want = ((int64_t)n * n + 255) / 256;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)kNumSMs * std::max(1, per_sm)));
    int nn = n;
    double* dp = D.p;
    int32_t* pp = pv.p;
    double* lp = lk.p;
    void* args[] = {&nn, &dp, &pp, &lp};
    CAMG_CUDA(cudaLaunchCooperativeKernel((void*)k_dense_lu, blocks, 256, args, 0, 0));
    CAMG_CUDA(cudaDeviceSynchronize());
    std::vector<double> lu_h((size_t)n * n);
    std::vector<int32_t> piv_h(n);
    CAMG_CUDA(cudaMemcpy(lu_h.data(), D.p, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToHost));
    CAMG_CUDA(cudaMemcpy(piv_h.data(), pv.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    set_coarse_lu(n, lu_h.data(), piv_h.data());
    if (inverse && n <= kCoarseInvMax) {
      cinv = DBuf<double>((size_t)n * n + 1);
      DBuf<int32_t> perm(n + 1);
      int pb = 0;
      CAMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pb, k_lu_inverse_coop, 256, 0));
      const int ib = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)n * n + 255) / 256,
                                                                 (int64_t)kNumSMs * std::max(1, pb)));
      const double* lup = lu.p;
      const int32_t* pvp = piv.p;
      double* xp = cinv.p;
      int32_t* prp = perm.p;
      void* iargs[] = {&nn, &lup, &pvp, &xp, &prp};
      CAMG_CUDA(cudaLaunchCooperativeKernel((void*)k_lu_inverse_coop, ib, 256, iargs, 0, 0));
      CAMG_CUDA(cudaDeviceSynchronize());
      c_x0 = DBuf<double>(n + 1);
      c_r = DBuf<double>(n + 1);
    }
  }

  void coarse_solve(const double* b, double* x, cudaStream_t s) {
    Level* L = levels.back();
    if (coarse_solver == CAMG_COARSE_MERGED_LU) {
      CAMG_CHECK(lu.p != nullptr, CAMG_ERR_SETUP, "coarse LU factors were not set");
      if (cinv.p) {
        const int n = (int)n_coarse;
        dense_gemv(n, cinv.p, b, nullptr, c_x0.p, s);
        RowEpi e{b, nullptr, c_r.p, nullptr, nullptr, nullptr, 0.0};
        resid_rows(L->A, int64_t(0), n, c_x0.p, (const double*)nullptr, n, e, false, s);
        dense_gemv(n, cinv.p, c_r.p, c_x0.p, x, s);
        return;
      }
      if (lu_blk) {
        const int nb = (int)((n_coarse + kLuB - 1) / kLuB);
        note_launch();
        launch_k(k_lu_solve_blk, nb, 256, 0, s, (int)n_coarse, (const double*)lu.p, (const int32_t*)lu_perm.p, b,
                 lu_y.p, x, reinterpret_cast<unsigned*>(lu_flags.p));
        return;
      }
      lu_solve((int)n_coarse, lu.p, piv.p, b, x, s);
    } else {
      L->sweep(nullptr, b, x, s);
      L->join(s);
    }
  }

  // V-cycle at level l from zero with rhs b; result in x (returns pointer)
  double* vcycle(int l, const double* b, cudaStream_t s) {
    Level* L = levels[l];
    double* X[2] = {vx0[l].p, vx1[l].p};
    int cur = 0;
    if (l == (int)levels.size() - 1) {
      coarse_solve(b, X[0], s);
      return X[0];
    }
    const double* x = nullptr;  // zero
    for (int k = 0; k < L->pre; ++k) {
      double* dst = X[cur];
      L->sweep(x, b, dst, s);
      x = dst;
      cur ^= 1;
    }
    L->residual(x, b, vr[l].p, s);
    spmv(L->R, 1.0, vr[l].p, 0.0, vb[l + 1].p, s);
    const double* xc = vcycle(l + 1, vb[l + 1].p, s);
    double* xx;
    if (x == nullptr) {  // no pre-smoothing: x = P xc
      xx = X[cur];
      spmv(L->P, 1.0, xc, 0.0, xx, s);
      cur ^= 1;
    } else {
      xx = const_cast<double*>(x);
      spmv(L->P, 1.0, xc, 1.0, xx, s);
    }
    const double* xs = xx;
    for (int k = 0; k < L->post; ++k) {
      double* dst = (xs == X[0]) ? X[1] : X[0];
      L->sweep(xs, b, dst, s);
      xs = dst;
    }
    L->join(s);
    return const_cast<double*>(xs);
  }

  void run(const double* r, double* z, cudaStream_t s) {
    const int64_t n = levels[0]->n;
    double* res = vcycle(0, r, s);
    CAMG_CUDA(cudaMemcpyAsync(z, res, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }

  // a fresh workspace with private copies of every work vector
  VcycleWs* make_ws() {
    std::unique_ptr<VcycleWs> w(new VcycleWs());
    w->owned = true;
    for (DBuf<double>* b : work_slots()) {
      w->bufs.emplace_back(b->p ? DBuf<double>(b->n) : DBuf<double>());
      if (b->p) CAMG_CUDA(cudaMemset(w->bufs.back().p, 0, sizeof(double) * b->n));  // (hand-off flags start at 0)
    }
    return w.release();
  }

  // record the cycle over w's vectors into w's graph
  void capture(VcycleWs& w) {
    const int64_t n = levels[0]->n;
    if (!w.stream) {
      CAMG_CUDA(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
      CAMG_CUDA(cudaEventCreateWithFlags(&w.ev0, cudaEventDisableTiming));
      CAMG_CUDA(cudaEventCreateWithFlags(&w.ev1, cudaEventDisableTiming));
      w.in = DBuf<double>(n);
      w.out = DBuf<double>(n);
    }
    std::lock_guard<std::mutex> lk(g_capture_mu);
    std::vector<DBuf<double>*> slots;
    if (w.owned) {
      slots = work_slots();
      CAMG_CHECK(slots.size() == w.bufs.size(), CAMG_ERR_NATIVE, "workspace does not match the hierarchy");
    }
    struct Swap {  // bind w's vectors for the capture, restore on every exit
      std::vector<DBuf<double>*>& s;
      std::vector<DBuf<double>>& b;
      Swap(std::vector<DBuf<double>*>& s_, std::vector<DBuf<double>>& b_) : s(s_), b(b_) { flip(); }
      ~Swap() { flip(); }
      void flip() { for (size_t i = 0; i < s.size(); ++i) std::swap(*s[i], b[i]); }
    } bind(slots, w.bufs);
    cudaGraph_t g;
    CAMG_CUDA(cudaStreamBeginCapture(w.stream, cudaStreamCaptureModeThreadLocal));
    const int64_t before = g_thread_launches;
    try {
      run(w.in.p, w.out.p, w.stream);
    } catch (...) {
      cudaStreamEndCapture(w.stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    w.kernels = g_thread_launches - before;
    g_launches.fetch_sub(w.kernels);
    g_thread_launches -= w.kernels;
    CAMG_CUDA(cudaStreamEndCapture(w.stream, &g));
    const char* pe = getenv("CAMG_SIDE_PRIO");
    CAMG_CUDA(cudaGraphInstantiate(&w.graph, g, (pe && pe[0] == '0') ? 0 : cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
  }

  void apply_ws(VcycleWs& w, const double* r, double* z, cudaStream_t caller) {
    const int64_t n = levels[0]->n;
    if (!w.graph) capture(w);
    CAMG_CUDA(cudaMemcpyAsync(w.in.p, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, caller));
    CAMG_CUDA(cudaEventRecord(w.ev0, caller));
    CAMG_CUDA(cudaStreamWaitEvent(w.stream, w.ev0, 0));
    note_launch((int)w.kernels);
    CAMG_CUDA(cudaGraphLaunch(w.graph, w.stream));
    CAMG_CUDA(cudaEventRecord(w.ev1, w.stream));
    CAMG_CUDA(cudaStreamWaitEvent(caller, w.ev1, 0));
    CAMG_CUDA(cudaMemcpyAsync(z, w.out.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, caller));
  }

  void apply(const double* r, double* z, cudaStream_t caller) {
    if (!use_graph) {  // eager launches over the hierarchy's own vectors (not re-entrant)
      std::lock_guard<std::mutex> lk(g_capture_mu);
      run(r, z, caller);
      CAMG_LAUNCH_CHECK();
      return;
    }
    apply_ws(def, r, z, caller);
  }
};

Hierarchy* hierarchy_create(Level** lv, int nlev, int coarse_solver) {
  CAMG_CHECK(nlev >= 1, CAMG_ERR_ARG, "need at least one level");
  std::unique_ptr<Hierarchy> H(new Hierarchy());
  H->levels.assign(lv, lv + nlev);
  H->coarse_solver = coarse_solver;
  for (int l = 0; l < nlev; ++l) {
    Level* L = H->levels[l];
    if (l < nlev - 1) {
      CAMG_CHECK(L->P != nullptr, CAMG_ERR_SETUP, "level transfer was not set");
      CAMG_CHECK(L->P->n_cols == H->levels[l + 1]->n, CAMG_ERR_DIMENSION, "transfer does not match the next level");
    }
    H->vb.emplace_back(L->n + 1);
    H->vx0.emplace_back(L->n + 1);
    H->vx1.emplace_back(L->n + 1);
    H->vr.emplace_back(L->n + 1);
  }
  return H.release();
}

void hierarchy_apply(Hierarchy* H, const double* r, double* z, cudaStream_t s) { H->apply(r, z, s); }
void hierarchy_apply_ws(Hierarchy* H, VcycleWs* w, const double* r, double* z, cudaStream_t s) {
  if (w) H->apply_ws(*w, r, z, s);
  else H->apply(r, z, s);
}
int64_t hierarchy_rows(const Hierarchy* H) { return H->levels[0]->n; }
// one BlockSmoother sweep from zero (the nested preconditioner's apply,
// hierarchy.py:366-376): out = sweep(0, b)
void level_precond(Level* L, const double* b, double* out, cudaStream_t s) {
  L->sweep(nullptr, b, out, s);
  L->join(s);
}
int64_t level_rows(const Level* L) { return L->n; }

// ---------------------------------------------------------------------------
// scalar smoothed-aggregation hierarchy on K (ScalarHierarchy,
// hierarchy.py:293-320): V(1,1) with one point-smoother call before and after
// the coarse correction, dense LU on the coarsest level

struct ScalarLevel {
  const Csr* A = nullptr;  // borrowed
  Csr* P = nullptr;        // owned copy
  Csr* R = nullptr;        // P^T (owned)
  int64_t n = 0;
  int kind = CAMG_PT_JACOBI, sweeps = 1;
  DBuf<double> dinv;
  McgsK gs;
  std::vector<double> c1, c2;  // Chebyshev coefficients
  DBuf<double> cd[2];
  DBuf<double> b, x0, x1, r, t;
  ~ScalarLevel() { delete P; delete R; }
};

struct ScalarHier {
  std::vector<std::unique_ptr<ScalarLevel>> levels;
  DBuf<double> lu;
  DBuf<int32_t> piv;
  int64_t n_coarse = 0;

  // PointSmoother.smooth (smoothers.py:186-199): `sweeps` sweeps from x
  // (null = zero) into out
  void smooth(ScalarLevel& L, const double* x, const double* b, double* out, cudaStream_t s) {
    if (L.kind == CAMG_PT_MCGS) {
      L.gs.init(x, b, out, s);
      L.gs.run(x == nullptr, L.A, nullptr, b, L.dinv.p, out, L.sweeps, s);
      return;
    }
    const bool cheb = L.kind == CAMG_PT_CHEBYSHEV;
    const double* cur = x;
    for (int k = 0; k < L.sweeps; ++k) {
      const bool last = k == L.sweeps - 1;
      double* dst = ((L.sweeps - 1 - k) % 2 == 0) ? out : L.t.p;
      RowEpi e{b, cur, nullptr, L.dinv.p, nullptr, dst, 1.0};
      if (cheb) {
        e.c1 = L.c1[k];
        e.c2 = L.c2[k];
        e.dprev = k ? L.cd[(k - 1) & 1].p : nullptr;
        if (!last) e.out_d = L.cd[k & 1].p;
      }
      resid_rows(L.A, int64_t(0), L.n, cur, (const double*)nullptr, L.n, e, cur == nullptr, s);
      cur = dst;
    }
  }

  // ScalarHierarchy.vcycle from zero (hierarchy.py:305-315)
  const double* vcycle(int l, const double* b, cudaStream_t s) {
    ScalarLevel& L = *levels[l];
    if (l == (int)levels.size() - 1) {
      CAMG_CHECK(lu.p != nullptr, CAMG_ERR_SETUP, "scalar coarse LU factors were not set");
      lu_solve((int)n_coarse, lu.p, piv.p, b, L.x0.p, s);
      return L.x0.p;
    }
    smooth(L, nullptr, b, L.x0.p, s);
    RowEpi e{b, nullptr, L.r.p, nullptr, nullptr, nullptr, 0.0};
    resid_rows(L.A, int64_t(0), L.n, L.x0.p, (const double*)nullptr, L.n, e, false, s);
    ScalarLevel& C = *levels[l + 1];
    spmv(L.R, 1.0, L.r.p, 0.0, C.b.p, s);
    const double* xc = vcycle(l + 1, C.b.p, s);
    spmv(L.P, 1.0, xc, 1.0, L.x0.p, s);
    smooth(L, L.x0.p, b, L.x1.p, s);
    return L.x1.p;
  }
};

const double* scalar_run(ScalarHier* H, const double* b, cudaStream_t s) { return H->vcycle(0, b, s); }

void scalar_work_slots(ScalarHier* H, std::vector<DBuf<double>*>& v) {
  for (auto& L : H->levels)
    for (DBuf<double>* b : {&L->b, &L->x0, &L->x1, &L->r, &L->t, &L->cd[0], &L->cd[1], &L->gs.g}) v.push_back(b);
}

static ScalarHier* scalar_hierarchy_create(int nlev, const Csr* const* A, const Csr* const* P, const int* node_block,
                                           int kind, int sweeps, double damping) {
  CAMG_CHECK(nlev >= 1, CAMG_ERR_ARG, "need at least one level");
  CAMG_CHECK(kind == CAMG_PT_JACOBI || kind == CAMG_PT_MCGS || kind == CAMG_PT_CHEBYSHEV, CAMG_ERR_CONFIG,
             "GPU scalar smoother supports jacobi, mcgs and chebyshev");
  CAMG_CHECK(sweeps >= 1, CAMG_ERR_CONFIG, "point smoother sweeps must be >= 1");
  cudaStream_t s = 0;
  std::unique_ptr<ScalarHier> H(new ScalarHier());
  for (int l = 0; l < nlev; ++l) {
    std::unique_ptr<ScalarLevel> L(new ScalarLevel());
    L->A = A[l];
    L->n = A[l]->n_rows;
    CAMG_CHECK(A[l]->n_cols == L->n, CAMG_ERR_DIMENSION, "scalar level operator must be square");
    L->kind = kind;
    L->sweeps = sweeps;
    const int64_t n = L->n;
    L->b = DBuf<double>(n + 1);
    L->x0 = DBuf<double>(n + 1);
    if (l < nlev - 1) {
      CAMG_CHECK(P[l]->n_rows == n && P[l]->n_cols == A[l + 1]->n_rows, CAMG_ERR_DIMENSION,
                 "scalar transfer does not match the levels");
      L->P = csr_copy(P[l], s);
      L->R = csr_transpose(L->P, s);
      L->x1 = DBuf<double>(n + 1);
      L->r = DBuf<double>(n + 1);
      L->t = DBuf<double>(n + 1);
      DBuf<double> d(n + 1);
      csr_diagonal(L->A, 0, d.p, s);
      CAMG_CUDA(cudaDeviceSynchronize());
      check_no_zero(d.p, n, kind == CAMG_PT_MCGS ? "sgs" : "jacobi");
      L->dinv = DBuf<double>(n + 1);
      note_launch();
      k_scaled_recip<<<grid_for(n, 256), 256>>>(n, d.p, kind == CAMG_PT_CHEBYSHEV ? 1.0 : damping, 1.0, L->dinv.p);
      if (kind == CAMG_PT_MCGS) L->gs.setup(L->A, node_block ? node_block[l] : 1, s);
      if (kind == CAMG_PT_CHEBYSHEV) {
        cheb_coefficients(lambda_max_dinv(L->A, d.p, 10, s), sweeps, L->c1, L->c2);
        if (sweeps > 1) {
          L->cd[0] = DBuf<double>(n + 1);
          L->cd[1] = DBuf<double>(n + 1);
        }
      }
    }
    H->levels.push_back(std::move(L));
  }
  CAMG_CUDA(cudaDeviceSynchronize());
  return H.release();
}

}  // namespace camg

using namespace camg;


extern "C" {

int camg_level_create(const camg_csr* K, const camg_csr* B1, const camg_csr* B2, const camg_csr* Cz,
                      const camg_smoother_cfg* cfg, int pre_sweeps, int post_sweeps, camg_level** out) {
  return guarded([&] { *out = new camg_level{level_create(K->m, B1->m, B2->m, Cz->m, *cfg, pre_sweeps, post_sweeps, nullptr)}; });
}

int camg_level_create_shared(camg_csr* A, const camg_csr* K, const camg_csr* B1, const camg_csr* B2,
                             const camg_csr* Cz, const camg_smoother_cfg* cfg, int pre_sweeps, int post_sweeps,
                             camg_level** out) {
  return guarded([&] {
    *out = new camg_level{level_create(K->m, B1->m, B2->m, Cz->m, *cfg, pre_sweeps, post_sweeps, A->m)};
  });
}

int camg_level_destroy(camg_level* L) {
  return guarded([&] {
    if (L) { delete L->L; delete L; }
  });
}

int camg_level_schur(const camg_level* L, camg_csr** out) {
  return guarded([&] {
    CAMG_CHECK(L->L->S != nullptr, CAMG_ERR_SETUP, "S~ was not set");
    *out = new camg_csr{csr_copy(L->L->S, 0)};
  });
}

int camg_level_operator(const camg_level* L, const camg_csr** out) {
  return guarded([&] {
    L->L->op_handle.m = L->L->A;
    *out = &L->L->op_handle;
  });
}

int camg_level_set_corrector_lu(camg_level* L, int64_t n, const double* lu, const int32_t* piv) {
  return guarded([&] {
    CAMG_CHECK(n == L->L->nl, CAMG_ERR_DIMENSION, "corrector LU size does not match n_lam");
    L->L->corr_lu = DBuf<double>(n * n + 1);
    L->L->corr_piv = DBuf<int32_t>(n + 1);
    CAMG_CUDA(cudaMemcpy(L->L->corr_lu.p, lu, sizeof(double) * n * n, cudaMemcpyHostToDevice));
    CAMG_CUDA(cudaMemcpy(L->L->corr_piv.p, piv, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  });
}

int camg_level_set_k_lu(camg_level* L, int64_t n, const double* lu, const int32_t* piv) {
  return guarded([&] {
    CAMG_CHECK(n == L->L->nu, CAMG_ERR_DIMENSION, "K LU size does not match n_u");
    L->L->k_lu = DBuf<double>(n * n + 1);
    L->L->k_piv = DBuf<int32_t>(n + 1);
    CAMG_CUDA(cudaMemcpy(L->L->k_lu.p, lu, sizeof(double) * n * n, cudaMemcpyHostToDevice));
    CAMG_CUDA(cudaMemcpy(L->L->k_piv.p, piv, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  });
}

int camg_level_set_schur(camg_level* L, const camg_csr* S) {
  return guarded([&] {
    Level* lv = L->L;
    CAMG_CHECK(lv->exact, CAMG_ERR_CONFIG, "S~ is supplied only for a_hat_mode exact");
    CAMG_CHECK(lv->S == nullptr, CAMG_ERR_SETUP, "S~ was already set");
    CAMG_CHECK(S->m->n_rows == lv->nl && S->m->n_cols == lv->nl, CAMG_ERR_DIMENSION, "S~ must be n_lam x n_lam");
    lv->S = csr_copy(S->m, 0);
    setup_corrector(lv);
  });
}

int camg_level_set_transfer(camg_level* L, const camg_csr* P_u, const camg_csr* P_lam) {
  return guarded([&] {
    Level* lv = L->L;
    CAMG_CHECK(P_u->m->n_rows == lv->nu && P_lam->m->n_rows == lv->nl, CAMG_ERR_DIMENSION,
               "transfer dimensions do not match the operator");
    delete lv->P;
    delete lv->R;
    lv->P = block_diag(P_u->m, P_lam->m, 0);
    lv->R = csr_transpose(lv->P, 0);
    lv->nc = lv->P->n_cols;
  });
}

int camg_level_block_transfer(camg_level* L, int bs_fine, int bs_coarse, int64_t ncoarse_u) {
  return guarded([&] {
    Level* lv = L->L;
    CAMG_CHECK(lv->P != nullptr, CAMG_ERR_SETUP, "transfer not set");
    delete lv->P->sell;
    lv->P->sell = sell_build(lv->P, bs_fine, bs_coarse, lv->nu, ncoarse_u, 0);
    delete lv->R->sell;
    lv->R->sell = nullptr;
    // R has few, long rows: one lane per block row only pays when there are
    // enough block rows to fill the GPU; otherwise the warp-per-row CSR wins
    // (CAMG_SELL_MIN_BLOCK_ROWS overrides the threshold: tests force the
    // block SELL restriction on small hierarchies)
    const char* e = getenv("CAMG_SELL_MIN_BLOCK_ROWS");
    const int64_t min_rows = e ? atoll(e) : kSellMinBlockRows;
    if (ncoarse_u / bs_coarse >= min_rows)
      lv->R->sell = sell_build(lv->R, bs_coarse, bs_fine, ncoarse_u, lv->nu, 0);
  });
}

// one fine-level pass of the dominant smoother kernel (timing / profiling):
// mode 1 = fused residual + first Jacobi sweep, mode 2 = extra Jacobi sweep
int camg_level_fine_pass(camg_level* L, int mode, const double* x, const double* b, void* stream,
                         double* bytes_csr_model, double* bytes_format) {
  return guarded([&] {
    Level* lv = L->L;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nu = lv->nu;
    // mode | 0x100: the same pass through a second mirror of the rows in the
    // streaming layout (no shared value groups), built on first use, so one
    // run times both layouts; 0x200 alone releases that mirror
    if (mode == 0x200) {
      delete lv->alt_sell;
      lv->alt_sell = nullptr;
      return;
    }
    struct Swap {
      Csr* A; Sell* keep; bool on;
      ~Swap() { if (on) A->sell = keep; }
    } swap{lv->A, lv->A->sell, false};
    if (mode & 0x100) {
      mode &= 0xff;
      const Sell* S = lv->A->sell;
      CAMG_CHECK(S && S->br == S->bc && S->rows() == nu, CAMG_ERR_CONFIG, "level has no block mirror of its rows");
      if (!lv->alt_sell) {
        sell_share_override(0);
        try {
          lv->alt_sell = sell_build(lv->A, S->br, S->bc, nu, lv->A->n_cols - lv->A->n_cols % S->bc, 0, S->masked);
        } catch (...) {
          sell_share_override(-1);
          throw;
        }
        sell_share_override(-1);
      }
      lv->A->sell = lv->alt_sell;
      swap.on = true;
    }
    // the smoother's predictor sweep: y_new = y + w D^-1 (b - [K B1][y; lam]),
    // or Braess-Sarazin's u_half = u + A^-1 r / alpha (no Jacobi predictor)
    const bool bs = lv->dinv_p.p == nullptr;
    CAMG_CHECK(mode == 1 || !bs, CAMG_ERR_CONFIG, "level has no Jacobi predictor");
    CAMG_CHECK(mode != 3 || lv->pred_colors() > 0, CAMG_ERR_CONFIG, "level has no multicolour predictor");
    if (mode == 3) {
      lv->gs_predict(x, b, lv->w_tmp.p, 1, s);
      CAMG_LAUNCH_CHECK();
      // two passes over K: matrix + x read + y written + b, D^-1 read; the
      // init pass reads x_u, b_u and writes y, g; lambda via B1 is < 0.1%
      const double nnzK = (double)(lv->nnz_top - lv->B1->nnz);
      const double vec = 4.0 * 8.0 * nu;
      const double pass = 12.0 * nnzK + 4.0 * (nu + 1) + vec;
      if (bytes_csr_model) *bytes_csr_model = 2.0 * pass + 32.0 * nu;
      if (bytes_format) {
        if (lv->gs.sell) {
          const int br = lv->gs.sell->br;
          *bytes_format = 2.0 * (sell_pass_bytes(lv->gs.sell) + vec + 4.0 * lv->gs.sell->nbr +
                                 8.0 * (br * (br - 1) / 2) * (double)(nu / br)) + 32.0 * nu;
        } else {
          *bytes_format = 2.0 * (12.0 * (double)lv->nnz_top + 8.0 * (nu + 1) + vec) + 16.0 * nu;
        }
      }
      return;
    }
    if (mode == 1) {
      RowEpi e{b, x, nullptr, bs ? lv->ainv.p : lv->dinv_p.p, nullptr, lv->w_tmp.p,
               bs ? 1.0 / lv->cfg.alpha : 1.0};
      resid_rows(lv->A, int64_t(0), nu, x, x + nu, nu, e, false, s);
    } else {
      jacobi_rows(lv->A, nu, x, b, lv->dinv_p.p, lv->w_du2.p, x, lv->w_tmp.p, 1.0, s);
    }
    CAMG_LAUNCH_CHECK();
    // §8(d): 12 B per non-zero of the [K | B1] rows + int32 offsets + x read
    // + 3 (mode 1: b, dinv, y out) or 6 (mode 2) vector streams
    const double nv = mode == 1 ? 3.0 : 6.0;
    const double vec = 8.0 * (double)lv->n + nv * 8.0 * (double)nu;
    if (bytes_csr_model) *bytes_csr_model = 12.0 * (double)lv->nnz_top + 4.0 * (nu + 1) + vec;
    if (bytes_format) {
      if (lv->A->sell && lv->A->sell->rows() == nu)
        *bytes_format = sell_pass_bytes(lv->A->sell) + vec;
      else
        *bytes_format = 12.0 * (double)lv->nnz_top + 8.0 * (nu + 1) + vec;
    }
  });
}

int camg_level_sweep(camg_level* L, const double* x, const double* b, double* out, void* stream) {
  return guarded([&] {
    L->L->sweep(x, b, out, (cudaStream_t)stream);
    L->L->join((cudaStream_t)stream);
    CAMG_LAUNCH_CHECK();
  });
}

int camg_hierarchy_create(camg_level** levels, int num_levels, int coarse_solver, camg_hierarchy** out) {
  return guarded([&] {
    std::vector<Level*> lv(num_levels);
    for (int i = 0; i < num_levels; ++i) lv[i] = levels[i]->L;
    *out = new camg_hierarchy{hierarchy_create(lv.data(), num_levels, coarse_solver)};
  });
}

int camg_hierarchy_set_coarse_lu(camg_hierarchy* H, int64_t n, const double* lu, const int32_t* piv) {
  return guarded([&] {
    CAMG_CHECK(n == H->H->levels.back()->n, CAMG_ERR_DIMENSION, "coarse LU size mismatch");
    CAMG_CHECK(n < (1 << 30), CAMG_ERR_DIMENSION, "coarse LU too large");
    CAMG_CHECK(!H->H->def.graph, CAMG_ERR_SETUP, "coarse LU must be set before the first V-cycle");
    H->H->set_coarse_lu(n, lu, piv);
  });
}

int camg_hierarchy_set_coarse_inverse(camg_hierarchy* H, int64_t n, const double* inv) {
  return guarded([&] {
    CAMG_CHECK(!H->H->def.graph, CAMG_ERR_SETUP, "coarse inverse must be set before the first V-cycle");
    H->H->set_coarse_inverse(n, inv);
  });
}

int camg_hierarchy_coarse_factor(camg_hierarchy* H, int inverse) {
  return guarded([&] {
    CAMG_CHECK(!H->H->def.graph, CAMG_ERR_SETUP, "coarse factors must be set before the first V-cycle");
    CAMG_CHECK(H->H->coarse_solver == CAMG_COARSE_MERGED_LU, CAMG_ERR_CONFIG, "coarse solver is not merged_lu");
    H->H->coarse_factor(inverse != 0);
  });
}

int camg_hierarchy_coarse_solve(camg_hierarchy* H, const double* b, double* x, void* stream) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_capture_mu);  // the hierarchy's own work vectors
    H->H->coarse_solve(b, x, (cudaStream_t)stream);
    H->H->levels.back()->join((cudaStream_t)stream);
    CAMG_LAUNCH_CHECK();
  });
}

int camg_hierarchy_destroy(camg_hierarchy* H) {
  return guarded([&] {
    if (H) { delete H->H; delete H; }
  });
}

int camg_vcycle(camg_hierarchy* H, const double* r, double* z, void* stream) {
  return guarded([&] { H->H->apply(r, z, (cudaStream_t)stream); });
}

int camg_scalar_hierarchy_create(int num_levels, const camg_csr* const* A, const camg_csr* const* P,
                                 const int* node_block, int kind, int sweeps, double damping,
                                 camg_scalar_hierarchy** out) {
  return guarded([&] {
    std::vector<const Csr*> a(num_levels), p(num_levels);
    for (int i = 0; i < num_levels; ++i) {
      a[i] = A[i]->m;
      p[i] = (i < num_levels - 1) ? P[i]->m : nullptr;
    }
    *out = new camg_scalar_hierarchy{scalar_hierarchy_create(num_levels, a.data(), p.data(), node_block, kind, sweeps,
                                                             damping)};
  });
}

int camg_scalar_hierarchy_set_coarse_lu(camg_scalar_hierarchy* H, int64_t n, const double* lu, const int32_t* piv) {
  return guarded([&] {
    CAMG_CHECK(n == H->H->levels.back()->n, CAMG_ERR_DIMENSION, "coarse LU size mismatch");
    CAMG_CHECK(n < (1 << 30), CAMG_ERR_DIMENSION, "coarse LU too large");
    H->H->n_coarse = n;
    H->H->lu = DBuf<double>(n * n + 1);
    H->H->piv = DBuf<int32_t>(n + 1);
    CAMG_CUDA(cudaMemcpy(H->H->lu.p, lu, sizeof(double) * n * n, cudaMemcpyHostToDevice));
    CAMG_CUDA(cudaMemcpy(H->H->piv.p, piv, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  });
}

int camg_scalar_hierarchy_apply(camg_scalar_hierarchy* H, const double* b, double* x, void* stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    const double* res = H->H->vcycle(0, b, s);
    CAMG_CUDA(cudaMemcpyAsync(x, res, sizeof(double) * H->H->levels[0]->n, cudaMemcpyDeviceToDevice, s));
    CAMG_LAUNCH_CHECK();
  });
}

int camg_scalar_hierarchy_destroy(camg_scalar_hierarchy* H) {
  return guarded([&] {
    if (H) { delete H->H; delete H; }
  });
}

int camg_level_set_predictor_solver(camg_level* L, camg_scalar_hierarchy* inner) {
  return guarded([&] {
    Level* lv = L->L;
    if (inner) {
      CAMG_CHECK(inner->H->levels[0]->n == lv->nu, CAMG_ERR_DIMENSION, "predictor solver size does not match n_u");
      CAMG_CHECK(lv->cfg.kind != CAMG_BRAESS_SARAZIN, CAMG_ERR_CONFIG, "braess_sarazin has no predictor");
    }
    lv->inner = inner ? inner->H : nullptr;
  });
}

int camg_vcycle_workspace_create(camg_hierarchy* H, camg_vcycle_workspace** out) {
  return guarded([&] { *out = new camg_vcycle_workspace{H->H->make_ws(), H->H}; });
}

int camg_vcycle_workspace_destroy(camg_vcycle_workspace* W) {
  return guarded([&] {
    if (W) { delete W->W; delete W; }
  });
}

int camg_vcycle_ws(camg_hierarchy* H, camg_vcycle_workspace* W, const double* r, double* z, void* stream) {
  return guarded([&] {
    CAMG_CHECK(!W || W->H == H->H, CAMG_ERR_ARG, "workspace belongs to another hierarchy");
    hierarchy_apply_ws(H->H, W ? W->W : nullptr, r, z, (cudaStream_t)stream);
  });
}

int camg_hierarchy_kernels_per_cycle(camg_hierarchy* H, int64_t* kernels) {
  return guarded([&] { *kernels = H->H->def.graph ? H->H->def.kernels : -1; });
}

int camg_level_get_info(const camg_level* Lh, camg_level_info* info) {
  return guarded([&] {
    const Level* L = Lh->L;
    camg_level_info o{};
    o.n_u = L->nu;
    o.n_lam = L->nl;
    o.nnz = L->A->nnz;
    const Sell* S = L->A->sell;
    if (S) {
      o.sell_block = S->br;
      o.sell_rows = S->rows();
      o.sell_masked = S->masked ? 1 : 0;
      o.sell_lanes = sell_lanes(S);
      o.sell_slices = S->nslices;
      o.sell_shared_values = S->dedup ? 1 : 0;
      o.sell_value_groups = S->ngroups;
      o.sell_value_groups_full = S->dedup ? S->ngroups_full : S->ngroups;
    }
    o.overlap = L->overlap ? 1 : 0;
    o.overlap_indep_slices = L->n_indep;
    o.overlap_dep_slices = L->n_dep;
    const camg_smoother_cfg& c = L->cfg;
    auto mc_path = [](const McgsK& g) {
      return g.cl ? CAMG_PATH_CLUSTER : g.cta ? CAMG_PATH_CTA : g.sell ? CAMG_PATH_COLOUR_SELL : CAMG_PATH_COLOUR_CSR;
    };
    if (L->nl == 0) o.corr_path = CAMG_PATH_NONE;
    else if (c.corr_kind == CAMG_PT_DIRECT) o.corr_path = CAMG_PATH_DENSE_LU;
    else if (c.corr_kind == CAMG_PT_MCGS) { o.corr_path = mc_path(L->cgs); o.corr_colors = L->cgs.colors(); }
    else if (c.corr_kind == CAMG_PT_SGS || c.corr_kind == CAMG_PT_ILU0) o.corr_path = CAMG_PATH_LEX_TRSV;
    else if (c.corr_kind == CAMG_PT_MCILU0) {
      o.corr_path = L->lam_engine() ? CAMG_PATH_LAM_ENGINE
                    : L->lam_dense() ? CAMG_PATH_DENSE_INV
                    : L->lam_fused() ? CAMG_PATH_LAM_FUSED
                    : (L->cilu.cl && c.corr_sweeps == 1) ? CAMG_PATH_CLUSTER : CAMG_PATH_COLOUR_CSR;
      o.corr_colors = L->cilu.colors();
    } else o.corr_path = CAMG_PATH_FUSED;
    if (L->inner) o.pred_path = CAMG_PATH_INNER_AMG;
    else if (L->pred_generic()) o.pred_path = c.pred_kind == CAMG_PT_DIRECT ? CAMG_PATH_DENSE_LU : CAMG_PATH_LEX_TRSV;
    else if (c.kind != CAMG_BRAESS_SARAZIN && c.pred_kind == CAMG_PT_MCGS) {
      o.pred_path = mc_path(L->gs);
      o.pred_colors = L->gs.colors();
    } else o.pred_path = CAMG_PATH_FUSED;
    for (const DBuf<int>* e : {&L->cilu.fz_err, &L->cilu.eng_err}) {
      if (!e->p) continue;
      int h = 0;
      CAMG_CUDA(cudaMemcpy(&h, e->p, sizeof(int), cudaMemcpyDeviceToHost));
      o.watchdog |= h;
    }
    if (L->P) {
      o.transfer_block_rows = L->P->sell ? L->P->sell->br : 0;
      o.restrict_block_rows = L->R->sell ? L->R->sell->br : 0;
    }
    *info = o;
  });
}

int camg_hierarchy_use_graph(camg_hierarchy* H, int enable) {
  return guarded([&] { H->H->use_graph = enable != 0; });
}

int camg_hierarchy_vcycle_bytes(const camg_hierarchy* Hh, double* bytes_csr, double* bytes_fmt) {
  return guarded([&] {
    // 12 B/nnz + 4(m+1) + 8 n + 8 m per sparse application,
    // zero-vector products skipped, fused epilogue vectors counted.  The
    // format count replaces the matrix term by what the stored format must
    // stream: the block SELL mirror for the rows it covers (values + one
    // int32 per block, none for linear slots, masked slots only their union
    // pattern), int32-CSR with int64 offsets for the rest.
    const Hierarchy* H = Hh->H;
    for (int pass = 0; pass < 2; ++pass) {
      const bool F = pass == 1;
      auto mat = [&](const Csr* A, int64_t rows, double nnz) {
        if (!F) return 12.0 * nnz + 4.0 * (rows + 1);
        double b = 0.0;
        int64_t r0 = 0;
        if (A->sell && A->sell->rows() <= rows) {
          b += sell_pass_bytes(A->sell);
          r0 = A->sell->rows();
        }
        const double tail = (double)(read_i64(A->rowptr + rows) - read_i64(A->rowptr + r0));
        return b + 12.0 * tail + 8.0 * (rows - r0 + 1);
      };
      auto spm = [&](const Csr* A, int64_t rows, double nnz) {
        return mat(A, rows, nnz) + 8.0 * A->n_cols + 8.0 * rows;
      };
      double total = 0.0;
      const int nl = (int)H->levels.size();
      for (int l = 0; l < nl; ++l) {
        const Level* L = H->levels[l];
        const double nnzA = (double)L->A->nnz;
        const double top = (double)L->nnz_top;
        const camg_smoother_cfg& c = L->cfg;
        const int sp = (c.kind == CAMG_BRAESS_SARAZIN) ? 1 : c.pred_sweeps;
        // one predictor sweep over [K | B1]: matrix + x read + (b, D^-1, y out);
        // a multicolour SGS sweep is two such passes (forward, backward) plus
        // the per-step init of y (and g) from x, b
        const bool gs = c.kind != CAMG_BRAESS_SARAZIN && c.pred_kind == CAMG_PT_MCGS;
        const double top_pass = (gs && F && L->gs.sell) ? sell_pass_bytes(L->gs.sell) + 8.0 * L->n + 8.0 * L->nu
                                                        : spm(L->A, L->nu, top);
        const double sweep = gs ? 2.0 * (top_pass + 8.0 * 2 * L->nu) : top_pass + 8.0 * 2 * L->nu;
        // lambda side: B2/Cz rows, corrector sweeps over S~ (MCGS: forward +
        // backward), interface-row B1 correction, a few lambda vectors
        // (MC-ILU(0): forward + backward factor passes, plus an S~ product from the second sweep)
        const int corr_passes = c.corr_kind == CAMG_PT_MCGS ? 2 * c.corr_sweeps
                                : c.corr_kind == CAMG_PT_MCILU0 ? c.corr_sweeps + std::max(0, c.corr_sweeps - 1)
                                                                : std::max(0, c.corr_sweeps - 1);
        const double lam = 8.0 * 6 * L->nl + (nnzA - top) * 12.0 + 12.0 * (L->S ? L->S->nnz : 0) * corr_passes +
                           (c.kind != CAMG_UZAWA ? 12.0 * L->B1->nnz : 0.0);
        // Chebyshev keeps d_k between its steps: + write / read of one vector
        const double cheb = (!gs && c.kind != CAMG_BRAESS_SARAZIN && c.pred_kind == CAMG_PT_CHEBYSHEV)
                                ? 16.0 * L->nu * std::max(0, sp - 1) : 0.0;
        const double step = sp * sweep + lam + cheb +
                            (gs ? 32.0 * L->nu + (c.kind == CAMG_UZAWA ? 24.0 * L->nu : 0.0) : 0.0);
        // zero start: the first sweep reads no matrix / x (MC-SGS: only its
        // first colour is skipped)
        const double mat_top = top_pass - 8.0 * L->n - 8.0 * L->nu;
        const double step0 = gs ? step - (mat_top + 8.0 * L->n) / std::max(1, L->pred_colors())
                                : step - mat_top - 8.0 * L->n;
        int nsteps_pre = L->pre * c.outer_sweeps, nsteps_post = L->post * c.outer_sweeps;
        if (l == nl - 1) {
          if (H->coarse_solver == CAMG_COARSE_MERGED_LU) total += 8.0 * H->n_coarse * H->n_coarse + 16.0 * H->n_coarse;
          else total += step0 + (c.outer_sweeps - 1) * step;
          continue;
        }
        total += (nsteps_pre > 0 ? step0 + (nsteps_pre - 1) * step : 0.0) + nsteps_post * step;
        total += spm(L->A, L->n, nnzA) + 8.0 * L->n;          // residual (+ b read)
        total += spm(L->R, L->R->n_rows, (double)L->R->nnz);    // restriction
        total += spm(L->P, L->P->n_rows, (double)L->P->nnz) + 8.0 * L->n;  // prolong-add
      }
      (F ? *bytes_fmt : *bytes_csr) = total;
    }
  });
}

}  // extern "C"

// reference ilu0_factor (smoothers.py:80-106) on host CSR arrays, in place
extern "C" int camg_ilu0_factor(int64_t n, const int64_t* rowptr, const int32_t* col, double* val) {
  return guarded([&] {
    CAMG_CHECK(n >= 0 && (n == 0 || (rowptr && col && val)), CAMG_ERR_ARG, "ilu0_factor: bad arguments");
    for (int64_t r = 0; r < n; ++r)
      for (int64_t q = rowptr[r] + 1; q < rowptr[r + 1]; ++q)
        CAMG_CHECK(col[q - 1] < col[q], CAMG_ERR_ARG, "ilu0_factor: columns must be strictly increasing");
    ilu0_ikj(n, rowptr, col, val, nullptr);
  });
}

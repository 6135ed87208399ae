// Tentative prolongator on the device (transfer.py:86-145):
// one warp per aggregate runs LAPACK's column-pivoted Householder QR on the
// aggregate's near-kernel block in shared memory -- the unblocked path
// dgeqp3 takes for these k <= 16 column blocks (dlaqp2: pivot = first column
// of largest partial norm, reflector by dlarfg, dlarf update, the dlaqp2
// norm downdate with its recomputation guard) followed by dorg2r for the
// economic Q -- then the rank test |r_ii| > tol |r_00|, the coarse null space
// rows R P^T and the scatter of Q's kept columns into the CSR of P.
//
// Same algorithm, pivot rule, reflector signs and rank test as LAPACK; the
// inner sums run in warp-tree order instead of OpenBLAS's SIMD order, so the
// factors agree with scipy.linalg.qr to rounding (1e-15) whenever the pivot
// order is decided by more than rounding.  It often is not: the rotation
// modes of a symmetric aggregate have mathematically EQUAL partial norms
// (measured: 1,610 of the 4,913 level-0 aggregates of C5/4), and which of
// them LAPACK takes first is decided by the last bits of OpenBLAS's own dnrm2
// / dgemv kernels.  On those aggregates this kernel may order (and sign) the
// tied columns differently: the same coarse space and the same projector
// P P^T, another basis of it.  So this path is a GPU VARIANT in the
// north star's sense -- compared with the reference through the spanned space
// (P P^T, P B_c = B, ranks) and by convergence -- and the bit-identical path
// (camg_tentative: scipy's own LAPACK on host threads) stays the default; this
// one is selected with CAMG_TENTATIVE=gpu (transfer.py).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace camg {

struct PtGroup {
  int64_t G, M, kk, dof_off, q_off, agg_off;
};

Csr* tentative_assemble_dev(int64_t n_dofs, int64_t ncoarse, int64_t ngroups, const int64_t* meta,
                            const int64_t* d_dofs, const double* d_q, const int64_t* d_rank, const int64_t* d_col0);

namespace {

constexpr int kMaxK = 16;

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;  // identical in every lane (the butterfly adds the same pairs)
}

// dlapy2: sqrt(x^2 + y^2) without unnecessary overflow
__device__ __forceinline__ double lapy2(double x, double y) {
  const double xa = fabs(x), ya = fabs(y);
  const double w = fmax(xa, ya), z = fmin(xa, ya);
  if (z == 0.0) return w;
  const double q = z / w;
  return w * sqrt(1.0 + q * q);
}

// 2-norm of rows [r0, M) of column c (column-major A, leading dimension M)
__device__ __forceinline__ double col_norm(const double* A, int M, int c, int r0, int lane) {
  double s = 0.0;
  for (int r = r0 + lane; r < M; r += 32) {
    const double a = A[c * M + r];
    s = fma(a, a, s);
  }
  return sqrt(wsum(s));
}

// One warp per aggregate of the size group gp (M rows, k columns, kk = min(M, k)).
// Shared memory per warp: A (M x k, column-major) + vn1, vn2, tau (kMaxK each) + jpvt.
__global__ void __launch_bounds__(128) k_agg_qr(PtGroup gp, int k, const int64_t* __restrict__ dofs,
                                                const double* __restrict__ vecs, double rank_tol,
                                                double* __restrict__ Q, double* __restrict__ Rf,
                                                int64_t* __restrict__ rank, int* __restrict__ err) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int M = (int)gp.M, kk = (int)gp.kk;
  const int per_warp = M * k + 4 * kMaxK;
  double* A = sm + (size_t)wib * per_warp;
  double* vn1 = A + M * k;
  double* vn2 = vn1 + kMaxK;
  double* tau = vn2 + kMaxK;
  int* jp = reinterpret_cast<int*>(tau + kMaxK);
  const double tol3z = 1.0536712127723509e-08;  // sqrt(dlamch('Epsilon')) = sqrt(2^-53)
  for (int64_t g = blockIdx.x * (int64_t)wpb + wib; g < gp.G; g += (int64_t)gridDim.x * wpb) {
    const int64_t* d = dofs + gp.dof_off + g * M;
    for (int r = lane; r < M; r += 32) {
      const int64_t dof = d[r];
      for (int j = 0; j < k; ++j) A[j * M + r] = vecs[dof * k + j];
    }
    __syncwarp();
    for (int j = 0; j < k; ++j) {
      const double nr = col_norm(A, M, j, 0, lane);
      if (lane == 0) { vn1[j] = nr; vn2[j] = nr; jp[j] = j; }
    }
    __syncwarp();
    // ---- dlaqp2
    for (int i = 0; i < kk; ++i) {
      int pvt = i;
      double best = vn1[i];
      for (int j = i + 1; j < k; ++j)
        if (vn1[j] > best) { best = vn1[j]; pvt = j; }  // idamax: first of the largest
      __syncwarp();
      if (pvt != i) {
        for (int r = lane; r < M; r += 32) {
          const double t = A[pvt * M + r];
          A[pvt * M + r] = A[i * M + r];
          A[i * M + r] = t;
        }
        if (lane == 0) {
          const int t = jp[pvt]; jp[pvt] = jp[i]; jp[i] = t;
          vn1[pvt] = vn1[i];
          vn2[pvt] = vn2[i];
        }
      }
      __syncwarp();
      // dlarfg on rows i..M-1 of column i
      const double alpha = A[i * M + i];
      const double xnorm = col_norm(A, M, i, i + 1, lane);
      double t_i = 0.0;
      if (xnorm != 0.0) {
        const double beta = -copysign(lapy2(alpha, xnorm), alpha);
        t_i = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        for (int r = i + 1 + lane; r < M; r += 32) A[i * M + r] *= sc;
        __syncwarp();
        if (lane == 0) A[i * M + i] = beta;
      }
      if (lane == 0) tau[i] = t_i;
      __syncwarp();
      // dlarf: H(i) applied from the left to columns i+1..k-1 (v_i = 1)
      if (t_i != 0.0) {
        for (int j = i + 1; j < k; ++j) {
          double s = 0.0;
          for (int r = i + 1 + lane; r < M; r += 32) s = fma(A[i * M + r], A[j * M + r], s);
          const double w = A[j * M + i] + wsum(s);
          const double t = -t_i * w;
          for (int r = i + 1 + lane; r < M; r += 32) A[j * M + r] = fma(A[i * M + r], t, A[j * M + r]);
          __syncwarp();
          if (lane == 0) A[j * M + i] += t;
        }
      }
      __syncwarp();
      // partial column norm downdate (dlaqp2)
      for (int j = i + 1; j < k; ++j) {
        const double v1 = vn1[j];
        if (v1 != 0.0) {
          double temp = fabs(A[j * M + i]) / v1;
          temp = fmax(0.0, 1.0 - temp * temp);
          const double q = v1 / vn2[j];
          const double temp2 = temp * (q * q);
          if (temp2 <= tol3z) {
            double nv = 0.0;
            if (i + 1 < M) nv = col_norm(A, M, j, i + 1, lane);
            __syncwarp();
            if (lane == 0) { vn1[j] = nv; vn2[j] = nv; }
          } else {
            __syncwarp();
            if (lane == 0) vn1[j] = v1 * sqrt(temp);
          }
        }
      }
      __syncwarp();
    }
    // ---- R P^T rows and the rank
    const int64_t ga = gp.agg_off + g;
    const double d0 = fabs(A[0]);
    int r = 0;
    for (int i = 0; i < kk; ++i) r += fabs(A[i * M + i]) > rank_tol * d0;
    if (lane == 0) {
      rank[ga] = r;
      if (!(d0 > 0.0)) atomicCAS(err, 0, 1);
    }
    double* Rg = Rf + ga * (int64_t)k * k;
    for (int t = lane; t < kk * k; t += 32) {
      const int i = t / k, j = t % k;
      Rg[i * k + jp[j]] = j >= i ? A[j * M + i] : 0.0;
    }
    __syncwarp();
    // ---- dorg2r: the first kk columns of Q = H(0) ... H(kk-1)
    for (int i = kk - 1; i >= 0; --i) {
      const double t_i = tau[i];
      if (i < kk - 1 && t_i != 0.0) {
        for (int j = i + 1; j < kk; ++j) {
          double s = 0.0;
          for (int rr = i + 1 + lane; rr < M; rr += 32) s = fma(A[i * M + rr], A[j * M + rr], s);
          const double w = A[j * M + i] + wsum(s);
          const double t = -t_i * w;
          for (int rr = i + 1 + lane; rr < M; rr += 32) A[j * M + rr] = fma(A[i * M + rr], t, A[j * M + rr]);
          __syncwarp();
          if (lane == 0) A[j * M + i] += t;
        }
      }
      __syncwarp();
      for (int rr = i + 1 + lane; rr < M; rr += 32) A[i * M + rr] *= -t_i;
      for (int rr = lane; rr < i; rr += 32) A[i * M + rr] = 0.0;
      if (lane == 0) A[i * M + i] = 1.0 - t_i;
      __syncwarp();
      // rows above the diagonal of the columns to the right were zeroed when
      // those columns were formed, so A[j*M + i] (j > i) started from 0 above
    }
    double* Qg = Q + gp.q_off + g * (int64_t)M * kk;
    for (int t = lane; t < M * kk; t += 32) {
      const int rr = t / kk, c = t % kk;
      Qg[t] = A[c * M + rr];
    }
    __syncwarp();
  }
}

}  // namespace
}  // namespace camg

using namespace camg;

// The whole tentative prolongator with the QR on the device.  Same inputs and
// outputs as camg_tentative (hostqr.cu) without the LAPACK library.
extern "C" int camg_tentative_device(int64_t n_dofs, int k, const double* vecs, const int64_t* dof_node,
                                     const int64_t* node_to_agg, int64_t num_nodes, int64_t na, double rank_tol,
                                     camg_csr** P_out, int64_t* rank_out, double* coarse_ns, int64_t* ncoarse) {
  return guarded([&] {
    CAMG_CHECK(n_dofs >= 1 && k >= 1 && na >= 1, CAMG_ERR_ARG, "tentative: bad sizes");
    CAMG_CHECK(k <= kMaxK, CAMG_ERR_ARG, "tentative (device QR): more than 16 near-kernel vectors");
    // DOFs by aggregate (ascending within), aggregates by size (ids ascending within): as camg_tentative
    std::vector<int64_t> agg_of(n_dofs), cnt(na + 1, 0);
    for (int64_t i = 0; i < n_dofs; ++i) {
      const int64_t nd = dof_node[i];
      CAMG_CHECK(nd >= 0 && nd < num_nodes, CAMG_ERR_DIMENSION, "tentative: DOF node out of range");
      const int64_t a = node_to_agg[nd];
      CAMG_CHECK(a >= 0 && a < na, CAMG_ERR_SETUP, "tentative prolongator requires a complete aggregation");
      agg_of[i] = a;
      cnt[a + 1]++;
    }
    for (int64_t a = 0; a < na; ++a)
      if (cnt[a + 1] == 0) throw Error(CAMG_ERR_SETUP, "aggregate " + std::to_string(a) + " owns no DOFs");
    std::vector<int64_t> start(na + 1, 0);
    for (int64_t a = 0; a < na; ++a) start[a + 1] = start[a] + cnt[a + 1];
    std::vector<int64_t> order(n_dofs), at(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < n_dofs; ++i) order[at[agg_of[i]]++] = i;
    std::vector<std::pair<int64_t, int64_t>> bysize(na);
    for (int64_t a = 0; a < na; ++a) bysize[a] = {cnt[a + 1], a};
    std::sort(bysize.begin(), bysize.end());
    std::vector<int64_t> meta, dofs_f(n_dofs), agg_f(na);
    int64_t dof_off = 0, q_off = 0, agg_off = 0;
    for (int64_t g0 = 0; g0 < na;) {
      const int64_t M = bysize[g0].first;
      int64_t g1 = g0;
      while (g1 < na && bysize[g1].first == M) ++g1;
      const int64_t G = g1 - g0, kk = std::min<int64_t>(M, k);
      for (int64_t g = 0; g < G; ++g) {
        const int64_t a = bysize[g0 + g].second;
        agg_f[agg_off + g] = a;
        for (int64_t i = 0; i < M; ++i) dofs_f[dof_off + g * M + i] = order[start[a] + i];
      }
      meta.insert(meta.end(), {G, M, kk, dof_off, q_off, agg_off});
      dof_off += G * M;
      q_off += G * M * kk;
      agg_off += G;
      g0 = g1;
    }
    const int64_t ngroups = (int64_t)meta.size() / 6;
    cudaStream_t s = 0;
    DBuf<double> d_vecs((size_t)n_dofs * k), d_q((size_t)q_off + 1), d_Rf((size_t)na * k * k);
    DBuf<int64_t> d_dofs(n_dofs), d_rank(na), d_col0(na);
    DBuf<int> d_err(1);
    CAMG_CUDA(cudaMemcpyAsync(d_vecs.p, vecs, sizeof(double) * (size_t)n_dofs * k, cudaMemcpyHostToDevice, s));
    CAMG_CUDA(cudaMemcpyAsync(d_dofs.p, dofs_f.data(), sizeof(int64_t) * n_dofs, cudaMemcpyHostToDevice, s));
    CAMG_CUDA(cudaMemsetAsync(d_err.p, 0, sizeof(int), s));
    CAMG_CUDA(cudaMemsetAsync(d_Rf.p, 0, sizeof(double) * (size_t)na * k * k, s));
    for (int64_t gi = 0; gi < ngroups; ++gi) {
      const int64_t* m = meta.data() + 6 * gi;
      PtGroup gp{m[0], m[1], m[2], m[3], m[4], m[5]};
      const size_t per_warp = sizeof(double) * ((size_t)gp.M * k + 4 * kMaxK);
      CAMG_CHECK(per_warp <= 200 * 1024, CAMG_ERR_SETUP,
                 "tentative (device QR): an aggregate block exceeds shared memory; use the host path");
      int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, (96 * 1024) / per_warp));
      const size_t smem = per_warp * wpb;
      if (smem > 48 * 1024)
        CAMG_CUDA(cudaFuncSetAttribute(k_agg_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      note_launch();
      k_agg_qr<<<grid_for(gp.G, wpb, int64_t(kNumSMs) * 32), 32 * wpb, smem, s>>>(gp, k, d_dofs.p, d_vecs.p, rank_tol,
                                                                                 d_q.p, d_Rf.p, d_rank.p, d_err.p);
      CAMG_LAUNCH_CHECK();
    }
    std::vector<int64_t> rank_f(na);
    std::vector<double> Rf((size_t)na * k * k);
    int h_err = 0;
    CAMG_CUDA(cudaMemcpyAsync(rank_f.data(), d_rank.p, sizeof(int64_t) * na, cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaMemcpyAsync(Rf.data(), d_Rf.p, sizeof(double) * (size_t)na * k * k, cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaMemcpyAsync(&h_err, d_err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    if (h_err) {
      // |r_00| = 0 (rank 0): name the aggregate of smallest id, as the host path's loop does per size group
      int64_t bad = -1;
      for (int64_t g = 0; g < na; ++g)
        if (rank_f[g] == 0 && (bad < 0 || agg_f[g] < bad)) bad = agg_f[g];
      throw Error(CAMG_ERR_SETUP, "aggregate " + std::to_string(bad) + ": near-kernel block is identically zero");
    }
    // ranks and coarse null space in aggregate order, column offsets in group order
    std::vector<int64_t> r_all(na), col0(na + 1, 0), col0_f(na), pos_of(na);
    for (int64_t g = 0; g < na; ++g) { r_all[agg_f[g]] = rank_f[g]; pos_of[agg_f[g]] = g; }
    for (int64_t a = 0; a < na; ++a) col0[a + 1] = col0[a] + r_all[a];
    for (int64_t a = 0; a < na; ++a) {
      rank_out[a] = r_all[a];
      const double* Rg = Rf.data() + (size_t)pos_of[a] * k * k;
      for (int64_t i = 0; i < r_all[a]; ++i)
        for (int j = 0; j < k; ++j) coarse_ns[(size_t)(col0[a] + i) * k + j] = Rg[i * k + j];
    }
    for (int64_t g = 0; g < na; ++g) col0_f[g] = col0[agg_f[g]];
    *ncoarse = col0[na];
    CAMG_CUDA(cudaMemcpy(d_col0.p, col0_f.data(), sizeof(int64_t) * na, cudaMemcpyHostToDevice));
    *P_out = new camg_csr{tentative_assemble_dev(n_dofs, col0[na], ngroups, meta.data(), d_dofs.p, d_q.p, d_rank.p,
                                                 d_col0.p)};
  });
}

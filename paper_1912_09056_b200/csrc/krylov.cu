// Right-preconditioned restarted GMRES on device (krylov.py:45-129).
//
// Same outer logic as the reference (x0 = 0, Givens recurrence on the host,
// happy-breakdown test 1e-14*max(1,|H_jj|), true residual at every restart),
// but classical Gram-Schmidt applied twice (CGS2) instead of MGS + one
// re-orthogonalisation pass: both are two projection passes, CGS2 turns each
// into one streaming multi-vector kernel.  Three passes over the Krylov basis
// per iteration:  h1 = V^T w ;  w -= V h1 fused with h2 = V^T w ;
// w -= V h2 fused with ||w||^2.  One host synchronisation per iteration.
//
// The preconditioned vectors z_j = M^-1 v_j each iteration computes anyway
// are kept (Z, n x m, when the device has room), so a restart cycle ends
// with x += Z y instead of x += M^-1 (V y): one V-cycle less per cycle.  The
// V-cycle is linear, so the iterates are the reference's up to rounding.
#include <cmath>
#include <cstdlib>
#include <memory>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace camg {

struct Hierarchy;
void hierarchy_apply(Hierarchy* H, const double* r, double* z, cudaStream_t s);

namespace {

constexpr int kBlk = 256;
constexpr int kWarps = kBlk / 32;
constexpr int kPer = 8;                 // elements per lane per chunk
constexpr int kChunk = 32 * kPer;       // elements per warp chunk
constexpr int kGrid = 592;              // 4 x 148

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// MODE 0: part_i = V_i . w
// MODE 1: w -= V h ; part_i = V_i . w
// MODE 2: w -= V h ; part_0 = w . w
template <int MODE>
__global__ void __launch_bounds__(kBlk) k_ortho(const double* __restrict__ V, int64_t ld, int k, int64_t n,
                                                const double* __restrict__ h, double* __restrict__ w,
                                                double* __restrict__ part) {
  extern __shared__ double sh[];
  const int nacc = (MODE == 2) ? 1 : k;
  double* sacc = sh;                 // kWarps x nacc
  double* sh_h = sh + kWarps * nacc; // k
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * nacc; i += kBlk) sacc[i] = 0.0;
  if (MODE != 0)
    for (int i = threadIdx.x; i < k; i += kBlk) sh_h[i] = h[i];
  __syncthreads();
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  for (int64_t c = (int64_t)blockIdx.x * kWarps + warp; c < nchunks; c += (int64_t)gridDim.x * kWarps) {
    const int64_t base = c * kChunk + lane;
    double wv[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int64_t e = base + 32 * t;
      wv[t] = e < n ? w[e] : 0.0;
    }
    if (MODE != 0) {
      for (int i = 0; i < k; ++i) {
        const double hi = sh_h[i];
        const double* Vi = V + (int64_t)i * ld;
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
          const int64_t e = base + 32 * t;
          if (e < n) wv[t] = fma(-hi, Vi[e], wv[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int64_t e = base + 32 * t;
        if (e < n) w[e] = wv[t];
      }
    }
    if (MODE == 2) {
      double a = 0.0;
#pragma unroll
      for (int t = 0; t < kPer; ++t) a = fma(wv[t], wv[t], a);
      a = warp_sum(a);
      if (lane == 0) sacc[warp] += a;
    } else {
      for (int i = 0; i < k; ++i) {
        const double* Vi = V + (int64_t)i * ld;
        double a = 0.0;
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
          const int64_t e = base + 32 * t;
          if (e < n) a = fma(Vi[e], wv[t], a);
        }
        a = warp_sum(a);
        if (lane == 0) sacc[warp * k + i] += a;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nacc; i += kBlk) {
    double a = 0.0;
    for (int q = 0; q < kWarps; ++q) a += sacc[q * nacc + i];
    part[(int64_t)blockIdx.x * nacc + i] = a;
  }
}

// out[i] = sum_b part[b*k + i]   (fixed order, deterministic)
__global__ void k_reduce_cols(const double* __restrict__ part, int nb, int k, double* __restrict__ out) {
  for (int i = blockIdx.x; i < k; i += gridDim.x) {
    double a = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[(int64_t)b * k + i];
    a = block_sum(a);
    if (threadIdx.x == 0) out[i] = a;
    __syncthreads();
  }
}

// u = sum_i y_i V_i
__global__ void k_lincomb(const double* __restrict__ V, int64_t ld, int k, int64_t n, const double* __restrict__ y,
                          double* __restrict__ u) {
  extern __shared__ double sy[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) sy[i] = y[i];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a = fma(sy[i], V[(int64_t)i * ld + e], a);
    u[e] = a;
  }
}

__global__ void k_scale_into(int64_t n, const double* __restrict__ w, double inv, double* __restrict__ v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    v[e] = w[e] / inv;
}

__global__ void k_add(int64_t n, const double* __restrict__ a, double* __restrict__ x) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] += a[e];
}

}  // namespace

struct Gmres {
  int64_t n;
  int m;
  DBuf<double> V, Z, w, z, r, u, part, hdev;
  double* hhost = nullptr;
  Gmres(int64_t n_, int m_) : n(n_), m(m_) {
    V = DBuf<double>((size_t)n * (m + 1));
    {
      // Z only with 4 GB to spare (CAMG_GMRES_STORE_Z=0 disables)
      const char* e = getenv("CAMG_GMRES_STORE_Z");
      size_t fr = 0, tot = 0;
      CAMG_CUDA(cudaMemGetInfo(&fr, &tot));
      const size_t need = sizeof(double) * (size_t)n * m;
      if (!(e && e[0] == '0') && fr > need + (size_t(4) << 30)) Z = DBuf<double>((size_t)n * m);
    }
    w = DBuf<double>(n);
    z = DBuf<double>(n);
    r = DBuf<double>(n);
    u = DBuf<double>(n);
    part = DBuf<double>((size_t)kGrid * (m + 2));
    hdev = DBuf<double>(3 * (m + 2) + 8);
    CAMG_CUDA(cudaMallocHost(&hhost, sizeof(double) * (3 * (m + 2) + 8)));
  }
  ~Gmres() { if (hhost) cudaFreeHost(hhost); }

  double norm(const double* v, cudaStream_t s) {
    dot_device(n, v, v, hdev.p, part.p, s);
    CAMG_CUDA(cudaMemcpyAsync(hhost, hdev.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    return std::sqrt(hhost[0]);
  }

  void precond(Hierarchy* H, const double* v, double* out, cudaStream_t s) {
    if (H) hierarchy_apply(H, v, out, s);
    else CAMG_CUDA(cudaMemcpyAsync(out, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }

  void residual(const Csr* A, const double* b, const double* x, double* r_, cudaStream_t s) {
    CAMG_CUDA(cudaMemcpyAsync(r_, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    spmv(A, -1.0, x, 1.0, r_, s);
  }

  template <int MODE>
  void ortho(int k, const double* h, double* out, cudaStream_t s) {
    const int nacc = MODE == 2 ? 1 : k;
    size_t sh = sizeof(double) * (kWarps * nacc + k);
    note_launch(2);
    k_ortho<MODE><<<kGrid, kBlk, sh, s>>>(V.p, n, k, n, h, w.p, part.p);
    k_reduce_cols<<<std::min(nacc, 1024), 256, 0, s>>>(part.p, kGrid, nacc, out);
  }
};

void gmres_run(const Csr* A, Hierarchy* H, const double* b, double* x, double rtol, int max_iters, int restart,
               int* iterations, double* hist, int* converged, cudaStream_t s) {
  CAMG_CHECK(A->n_rows == A->n_cols, CAMG_ERR_DIMENSION, "gmres: operator must be square");
  CAMG_CHECK(rtol > 0.0 && rtol < 1.0, CAMG_ERR_CONFIG, "rel_tol must lie in (0, 1)");
  CAMG_CHECK(restart >= 1 && max_iters >= 1, CAMG_ERR_CONFIG, "restart and max_iters must be >= 1");
  const int64_t n = A->n_rows;
  const int mmax = std::min(restart, max_iters);
  // the Krylov basis (n x (m+1), 19 GB at C5) is allocated once and reused
  // by later solves of the same size on this thread
  static thread_local std::unique_ptr<Gmres> cache;
  if (!cache || cache->n != n || cache->m != mmax) {
    cache.reset();
    cache.reset(new Gmres(n, mmax));
  }
  Gmres& G = *cache;
  CAMG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  const double norm_b = G.norm(b, s);
  hist[0] = norm_b;
  int total = 0;
  bool conv = false;
  if (norm_b == 0.0) {
    *iterations = 0;
    *converged = 1;
    return;
  }
  const double target = rtol * norm_b;
  std::vector<double> Hm, cs, sn, g, y;
  bool first = true;
  while (total < max_iters && !conv) {
    // x0 = 0: the first residual is b and its norm is known
    double beta = norm_b;
    if (first) {
      CAMG_CUDA(cudaMemcpyAsync(G.r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    } else {
      G.residual(A, b, x, G.r.p, s);
      beta = G.norm(G.r.p, s);
    }
    first = false;
    if (beta <= target) { conv = true; break; }
    const int m = std::min(restart, max_iters - total);
    Hm.assign((size_t)(m + 1) * m, 0.0);
    cs.assign(m, 0.0);
    sn.assign(m, 0.0);
    g.assign(m + 1, 0.0);
    g[0] = beta;
    auto Hij = [&](int i, int j) -> double& { return Hm[(size_t)i * m + j]; };
    note_launch();
    k_scale_into<<<grid_for(n, 256), 256, 0, s>>>(n, G.r.p, beta, G.V.p);
    int used = 0;
    const bool keep_z = H && G.Z.p;
    for (int j = 0; j < m; ++j) {
      const double* vj = G.V.p + (int64_t)j * n;
      double* zj = keep_z ? G.Z.p + (int64_t)j * n : G.z.p;
      G.precond(H, vj, zj, s);
      spmv(A, 1.0, zj, 0.0, G.w.p, s);
      const int k = j + 1;
      double* h1 = G.hdev.p;
      double* h2 = G.hdev.p + (m + 2);
      double* nr = G.hdev.p + 2 * (m + 2);
      G.ortho<0>(k, nullptr, h1, s);
      G.ortho<1>(k, h1, h2, s);
      G.ortho<2>(k, h2, nr, s);
      CAMG_CUDA(cudaMemcpyAsync(G.hhost, G.hdev.p, sizeof(double) * (2 * (m + 2) + 1), cudaMemcpyDeviceToHost, s));
      CAMG_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i <= j; ++i) Hij(i, j) = G.hhost[i] + G.hhost[(m + 2) + i];
      Hij(j + 1, j) = std::sqrt(G.hhost[2 * (m + 2)]);
      const bool happy = Hij(j + 1, j) <= 1e-14 * std::max(1.0, std::fabs(Hij(j, j)));
      if (!happy) {
        note_launch();
        k_scale_into<<<grid_for(n, 256), 256, 0, s>>>(n, G.w.p, Hij(j + 1, j), G.V.p + (int64_t)(j + 1) * n);
      }
      for (int i = 0; i < j; ++i) {
        const double h0 = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = h0;
      }
      const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = Hij(j, j) / den;
      sn[j] = Hij(j + 1, j) / den;
      Hij(j, j) = den;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      used = j + 1;
      const double est = std::fabs(g[j + 1]);
      hist[total] = est;
      if (happy || est <= target || total >= max_iters) break;
    }
    y.assign(used, 0.0);
    for (int i = used - 1; i >= 0; --i) {
      double acc = g[i];
      for (int q = i + 1; q < used; ++q) acc -= Hij(i, q) * y[q];
      y[i] = acc / Hij(i, i);
    }
    CAMG_CUDA(cudaMemcpyAsync(G.hdev.p, y.data(), sizeof(double) * used, cudaMemcpyHostToDevice, s));
    note_launch();
    if (keep_z) {
      // x += Z y
      k_lincomb<<<grid_for(n, 256), 256, sizeof(double) * used, s>>>(G.Z.p, n, used, n, G.hdev.p, G.z.p);
    } else {
      // x += M^-1 (V y)
      k_lincomb<<<grid_for(n, 256), 256, sizeof(double) * used, s>>>(G.V.p, n, used, n, G.hdev.p, G.u.p);
      G.precond(H, G.u.p, G.z.p, s);
    }
    note_launch();
    k_add<<<grid_for(n, 256), 256, 0, s>>>(n, G.z.p, x);
    G.residual(A, b, x, G.r.p, s);
    const double tr = G.norm(G.r.p, s);
    if (tr <= target) conv = true;
  }
  CAMG_LAUNCH_CHECK();
  *iterations = total;
  *converged = conv ? 1 : 0;
}

}  // namespace camg

using namespace camg;

extern "C" int camg_gmres(const camg_csr* A, camg_hierarchy* H, const double* b, double* x, double rel_tol,
                          int max_iters, int restart, int* iterations, double* history, int* converged,
                          void* stream) {
  return guarded([&] {
    gmres_run(A->m, H ? H->H : nullptr, b, x, rel_tol, max_iters, restart, iterations, history, converged,
              (cudaStream_t)stream);
  });
}

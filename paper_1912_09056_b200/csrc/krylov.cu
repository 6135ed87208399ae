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
struct Level;
struct VcycleWs;
void hierarchy_apply_ws(Hierarchy* H, VcycleWs* w, const double* r, double* z, cudaStream_t s);
int64_t hierarchy_rows(const Hierarchy* H);
void level_precond(Level* L, const double* b, double* out, cudaStream_t s);
int64_t level_rows(const Level* L);

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

__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    c[e] = a[e] - b[e];
}

__global__ void k_add(int64_t n, const double* __restrict__ a, double* __restrict__ x) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] += a[e];
}

}  // namespace

constexpr int kMaxOrthoK = 2048;  // basis vectors per k_ortho launch (shared memory: 72 B per vector)

static void call_back(camg_apply_fn f, void* user, const double* x, double* y, cudaStream_t s) {
  const int rc = f(user, x, y, (void*)s);
  CAMG_CHECK(rc == 0, CAMG_ERR_NATIVE, "gmres: caller-supplied apply callback failed (status " + std::to_string(rc) + ")");
}

// the operator of a solve: a device matrix or a caller callback y = A x
struct Operator {
  const Csr* A = nullptr;
  camg_apply_fn fn = nullptr;
  void* user = nullptr;
  // y = A x
  void apply(const double* x, double* y, cudaStream_t s) const {
    if (A) spmv(A, 1.0, x, 0.0, y, s);
    else call_back(fn, user, x, y, s);
  }
};

// the preconditioner of a solve: a V-cycle (on a workspace), one block
// smoother sweep from zero (nested preconditioner), a caller callback, or none
struct Precond {
  Hierarchy* H = nullptr;
  VcycleWs* ws = nullptr;
  Level* L = nullptr;
  camg_apply_fn fn = nullptr;
  void* user = nullptr;
  bool any() const { return H || L || fn; }
  void apply(const double* v, double* out, int64_t n, cudaStream_t s) const {
    if (H) hierarchy_apply_ws(H, ws, v, out, s);
    else if (L) level_precond(L, v, out, s);
    else if (fn) call_back(fn, user, v, out, s);
    else CAMG_CUDA(cudaMemcpyAsync(out, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
};

struct Gmres {
  int64_t n;
  int m;
  int store_z;  // 1 keep Z, 0 never, -1 when 4 GB remain free (checked per solve)
  DBuf<double> V, Z, w, z, r, u, part, hdev;
  double* hhost = nullptr;
  int chunk = kMaxOrthoK;  // basis vectors per k_ortho launch (CAMG_ORTHO_CHUNK lowers it: tests)
  Gmres(int64_t n_, int m_, int store_z_) : n(n_), m(m_), store_z(store_z_) {
    if (const char* e = getenv("CAMG_ORTHO_CHUNK")) chunk = std::max(1, std::min(kMaxOrthoK, atoi(e)));
    V = DBuf<double>((size_t)n * (m + 1));
    w = DBuf<double>(n);
    z = DBuf<double>(n);
    r = DBuf<double>(n);
    u = DBuf<double>(n);
    part = DBuf<double>((size_t)kGrid * (std::min(m, kMaxOrthoK) + 2));
    hdev = DBuf<double>(3 * (m + 2) + 8);
    CAMG_CUDA(cudaMallocHost(&hhost, sizeof(double) * (3 * (m + 2) + 8)));
    if (store_z == 1) Z = DBuf<double>((size_t)n * m);
  }
  ~Gmres() { if (hhost) cudaFreeHost(hhost); }

  // Z (n x m, the preconditioned basis) when policy and free memory allow;
  // CAMG_GMRES_STORE_Z=0 disables it for the per-thread cache
  void ensure_z() {
    if (store_z != -1 || Z.p) return;
    const char* e = getenv("CAMG_GMRES_STORE_Z");
    if (e && e[0] == '0') return;
    size_t fr = 0, tot = 0;
    CAMG_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t need = sizeof(double) * (size_t)n * m;
    if (fr > need + (size_t(4) << 30)) Z = DBuf<double>((size_t)n * m);
  }

  double norm(const double* v, cudaStream_t s) {
    dot_device(n, v, v, hdev.p, part.p, s);
    CAMG_CUDA(cudaMemcpyAsync(hhost, hdev.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    return std::sqrt(hhost[0]);
  }

  void residual(const Operator& A, const double* b, const double* x, double* r_, cudaStream_t s) {
    if (A.A) {
      CAMG_CUDA(cudaMemcpyAsync(r_, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      spmv(A.A, -1.0, x, 1.0, r_, s);
      return;
    }
    A.apply(x, u.p, s);  // r = b - A x
    note_launch();
    k_sub<<<grid_for(n, 256), 256, 0, s>>>(n, b, u.p, r_);
  }

  // one k_ortho pass over basis vectors [i0, i0 + k) (k <= kMaxOrthoK)
  template <int MODE>
  void ortho_part(int i0, int k, const double* h, double* out, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
      CAMG_CUDA(cudaFuncSetAttribute(k_ortho<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * (kWarps + 1) * kMaxOrthoK)));
      attr = true;
    }
    const int nacc = MODE == 2 ? 1 : k;
    const size_t sh = sizeof(double) * (kWarps * nacc + k);
    note_launch(2);
    k_ortho<MODE><<<kGrid, kBlk, sh, s>>>(V.p + (int64_t)i0 * n, n, k, n, h ? h + i0 : nullptr, w.p, part.p);
    CAMG_LAUNCH_CHECK();
    k_reduce_cols<<<std::min(nacc, 1024), 256, 0, s>>>(part.p, kGrid, nacc, out + (MODE == 2 ? 0 : i0));
    CAMG_LAUNCH_CHECK();
  }

  // MODE 0: out = V^T w; 1: w -= V h, out = V^T w; 2: w -= V h, out[0] = w.w
  // over the first k basis vectors.  Bases longer than kMaxOrthoK vectors
  // (restart > 2048) go in chunks: all subtractions first, then the dots.
  template <int MODE>
  void ortho(int k, const double* h, double* out, cudaStream_t s) {
    const int ck = chunk;
    if (k <= ck) return ortho_part<MODE>(0, k, h, out, s);
    if (MODE != 0)
      for (int i0 = 0; i0 < k; i0 += ck) ortho_part<2>(i0, std::min(ck, k - i0), h, out, s);
    if (MODE != 2)
      for (int i0 = 0; i0 < k; i0 += ck) ortho_part<0>(i0, std::min(ck, k - i0), nullptr, out, s);
  }
};

static thread_local std::unique_ptr<Gmres> g_gmres_cache;

void gmres_run(int64_t n, const Operator& A, const Precond& M, Gmres* ws, const double* b, double* x, double rtol,
               int max_iters, int restart, int* iterations, double* hist, int* converged, cudaStream_t s) {
  if (A.A) {
    CAMG_CHECK(A.A->n_rows == A.A->n_cols, CAMG_ERR_DIMENSION, "gmres: operator must be square");
    CAMG_CHECK(A.A->n_rows == n, CAMG_ERR_DIMENSION, "gmres: operator size does not match");
  }
  CAMG_CHECK(A.A || A.fn, CAMG_ERR_ARG, "gmres: no operator");
  CAMG_CHECK(n >= 1, CAMG_ERR_DIMENSION, "gmres: empty system");
  CAMG_CHECK(rtol > 0.0 && rtol < 1.0, CAMG_ERR_CONFIG, "rel_tol must lie in (0, 1)");
  CAMG_CHECK(restart >= 1 && max_iters >= 1, CAMG_ERR_CONFIG, "restart and max_iters must be >= 1");
  if (M.H) CAMG_CHECK(hierarchy_rows(M.H) == n, CAMG_ERR_DIMENSION, "gmres: preconditioner size does not match");
  if (M.L) CAMG_CHECK(level_rows(M.L) == n, CAMG_ERR_DIMENSION, "gmres: preconditioner size does not match");
  const int mmax = std::min(restart, max_iters);
  if (!ws) {
    // the Krylov basis (n x (m+1), 19 GB at C5) is allocated once and reused
    // by later solves of the same size on this thread (camg_gmres_release frees it)
    if (!g_gmres_cache || g_gmres_cache->n != n || g_gmres_cache->m != mmax) {
      g_gmres_cache.reset();
      g_gmres_cache.reset(new Gmres(n, mmax, -1));
    }
    ws = g_gmres_cache.get();
  }
  CAMG_CHECK(ws->n == n && ws->m >= mmax, CAMG_ERR_DIMENSION, "gmres: workspace is smaller than the solve");
  if (M.any() && !M.fn) ws->ensure_z();
  Gmres& G = *ws;
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
    // x0 = 0: the first residual is b and its norm is known (a caller
    // callback operator is still applied to x0, the reference's call
    // sequence, krylov.py:69)
    double beta = norm_b;
    if (first && A.A) {
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
    // stored Z replaces the restart-cycle M^-1 (V y) of a native
    // preconditioner; caller callbacks see the reference's calls (krylov.py:122)
    const bool keep_z = M.any() && !M.fn && G.Z.p;
    for (int j = 0; j < m; ++j) {
      const double* vj = G.V.p + (int64_t)j * n;
      double* zj = keep_z ? G.Z.p + (int64_t)j * n : G.z.p;
      M.apply(vj, zj, n, s);
      A.apply(zj, G.w.p, s);
      const int k = j + 1;
      double* h1 = G.hdev.p;
      double* h2 = G.hdev.p + (G.m + 2);
      double* nr = G.hdev.p + 2 * (G.m + 2);
      G.ortho<0>(k, nullptr, h1, s);
      G.ortho<1>(k, h1, h2, s);
      G.ortho<2>(k, h2, nr, s);
      CAMG_CUDA(cudaMemcpyAsync(G.hhost, G.hdev.p, sizeof(double) * (2 * (G.m + 2) + 1), cudaMemcpyDeviceToHost, s));
      CAMG_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i <= j; ++i) Hij(i, j) = G.hhost[i] + G.hhost[(G.m + 2) + i];
      Hij(j + 1, j) = std::sqrt(G.hhost[2 * (G.m + 2)]);
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
      M.apply(G.u.p, G.z.p, n, s);
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
    Operator op;
    op.A = A->m;
    Precond M;
    M.H = H ? H->H : nullptr;
    gmres_run(A->m->n_rows, op, M, nullptr, b, x, rel_tol, max_iters, restart, iterations, history, converged,
              (cudaStream_t)stream);
  });
}

extern "C" int camg_gmres_ex(int64_t n, const camg_csr* A, camg_apply_fn apply_A, void* user_A, camg_hierarchy* H,
                             camg_vcycle_workspace* vws, camg_level* L, camg_apply_fn apply_M, void* user_M,
                             camg_gmres_workspace* gws, const double* b, double* x, double rel_tol, int max_iters,
                             int restart, int* iterations, double* history, int* converged, void* stream) {
  return guarded([&] {
    CAMG_CHECK((A != nullptr) != (apply_A != nullptr), CAMG_ERR_ARG, "gmres: give exactly one of A and apply_A");
    CAMG_CHECK((H != nullptr) + (L != nullptr) + (apply_M != nullptr) <= 1, CAMG_ERR_ARG,
               "gmres: give at most one preconditioner (hierarchy, level or callback)");
    CAMG_CHECK(!vws || (H && vws->H == H->H), CAMG_ERR_ARG, "gmres: V-cycle workspace of another hierarchy");
    Operator op;
    op.A = A ? A->m : nullptr;
    op.fn = apply_A;
    op.user = user_A;
    Precond M;
    M.H = H ? H->H : nullptr;
    M.ws = vws ? vws->W : nullptr;
    M.L = L ? L->L : nullptr;
    M.fn = apply_M;
    M.user = user_M;
    gmres_run(n, op, M, gws ? gws->G : nullptr, b, x, rel_tol, max_iters, restart, iterations, history, converged,
              (cudaStream_t)stream);
  });
}

extern "C" int camg_gmres_release(void) {
  return guarded([&] { g_gmres_cache.reset(); });
}

extern "C" int camg_gmres_workspace_create(int64_t n, int restart, int store_z, camg_gmres_workspace** out) {
  return guarded([&] {
    CAMG_CHECK(n >= 1 && restart >= 1, CAMG_ERR_CONFIG, "gmres workspace: n and restart must be >= 1");
    CAMG_CHECK(store_z >= -1 && store_z <= 1, CAMG_ERR_ARG, "gmres workspace: store_z must be -1, 0 or 1");
    *out = new camg_gmres_workspace{new Gmres(n, restart, store_z)};
  });
}

extern "C" int camg_gmres_workspace_destroy(camg_gmres_workspace* ws) {
  return guarded([&] {
    if (ws) { delete ws->G; delete ws; }
  });
}

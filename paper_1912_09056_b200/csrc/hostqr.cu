// Host batched pivoted QR of the tentative prolongator's aggregate blocks
// (transfer.py:86-145: scipy.linalg.qr(B, mode="economic", pivoting=True) per
// aggregate, i.e. LAPACK dgeqp3 + dorgqr).  The LAPACK routines are the very
// ones scipy calls -- scipy's bundled OpenBLAS, opened with dlopen -- so every
// block's Q, R and pivots are bit-identical to the reference's; the blocks
// are factored concurrently by a pool of host threads (one LAPACK call per
// block, OpenBLAS pinned to one thread per caller), which replaces the
// earlier fork()-based process pool (no fork of a process holding a CUDA
// context).  Host code: no device work.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace camg {

using geqp3_t = void (*)(const int*, const int*, double*, const int*, int*, double*, double*, const int*, int*);
using orgqr_t = void (*)(const int*, const int*, const int*, double*, const int*, const double*, double*, const int*,
                         int*);
using setthr_t = int (*)(int);

struct Lapack {
  geqp3_t geqp3 = nullptr;
  orgqr_t orgqr = nullptr;
  setthr_t set_threads_local = nullptr;
};

static std::mutex g_lapack_mu;
static std::string g_lapack_path;
static Lapack g_lapack;

static const Lapack& lapack(const char* path) {
  std::lock_guard<std::mutex> lk(g_lapack_mu);
  if (g_lapack.geqp3 && g_lapack_path == path) return g_lapack;
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  CAMG_CHECK(h != nullptr, CAMG_ERR_NATIVE, std::string("cannot open LAPACK library ") + path);
  Lapack L;
  // scipy-openblas exports the Fortran symbols with a scipy_ prefix
  L.geqp3 = reinterpret_cast<geqp3_t>(dlsym(h, "scipy_dgeqp3_"));
  L.orgqr = reinterpret_cast<orgqr_t>(dlsym(h, "scipy_dorgqr_"));
  if (!L.geqp3) L.geqp3 = reinterpret_cast<geqp3_t>(dlsym(h, "dgeqp3_"));
  if (!L.orgqr) L.orgqr = reinterpret_cast<orgqr_t>(dlsym(h, "dorgqr_"));
  L.set_threads_local = reinterpret_cast<setthr_t>(dlsym(h, "openblas_set_num_threads_local"));
  CAMG_CHECK(L.geqp3 && L.orgqr, CAMG_ERR_NATIVE, std::string("dgeqp3 / dorgqr not found in ") + path);
  g_lapack = L;
  g_lapack_path = path;
  return g_lapack;
}

}  // namespace camg

using namespace camg;

// G blocks of M rows and k columns: block g = vecs[dofs[g*M + i], :] (vecs
// row-major n_dofs x k).  Outputs (C order): Q (G, M, kk), R (G, kk, k),
// piv (G, k) 0-based, kk = min(M, k).  info_out: first failing block or -1.
extern "C" int camg_qr_batch(const char* lapack_path, int64_t G, int M, int k, const double* vecs, int64_t n_dofs,
                             const int64_t* dofs, double* q_out, double* r_out, int64_t* piv_out, int nthreads,
                             int64_t* info_out) {
  return guarded([&] {
    CAMG_CHECK(G >= 0 && M >= 1 && k >= 1 && vecs && dofs && q_out && r_out && piv_out, CAMG_ERR_ARG,
               "qr_batch: bad arguments");
    const Lapack& L = lapack(lapack_path);
    const int kk = std::min(M, k);
    std::atomic<int64_t> next(0), failed(-1);
    std::atomic<bool> bad_dof(false);
    auto work = [&]() {
      int prev = L.set_threads_local ? L.set_threads_local(1) : 0;
      std::vector<double> A((size_t)M * k), tau(kk);
      std::vector<int> jpvt(k);
      int info = 0, lwork = -1, m = M, n = k, lda = M, kq = kk;
      double q1 = 0.0, q2 = 0.0;
      // workspace queries (as scipy does); the unblocked kernels run for k <= NB
      std::fill(jpvt.begin(), jpvt.end(), 0);
      L.geqp3(&m, &n, A.data(), &lda, jpvt.data(), tau.data(), &q1, &lwork, &info);
      L.orgqr(&m, &kq, &kq, A.data(), &lda, tau.data(), &q2, &lwork, &info);
      int lw = std::max(std::max((int)q1, (int)q2), 3 * n + 1);
      std::vector<double> wk((size_t)lw);
      const int64_t chunk = 256;
      for (;;) {
        const int64_t g0 = next.fetch_add(chunk);
        if (g0 >= G) break;
        for (int64_t g = g0; g < std::min(G, g0 + chunk); ++g) {
          const int64_t* d = dofs + g * M;
          for (int i = 0; i < M; ++i) {
            if (d[i] < 0 || d[i] >= n_dofs) { bad_dof = true; continue; }
            for (int j = 0; j < k; ++j) A[(size_t)i + (size_t)j * M] = vecs[d[i] * k + j];
          }
          std::fill(jpvt.begin(), jpvt.end(), 0);
          L.geqp3(&m, &n, A.data(), &lda, jpvt.data(), tau.data(), wk.data(), &lw, &info);
          if (info != 0) { int64_t e = -1; failed.compare_exchange_strong(e, g); continue; }
          double* R = r_out + g * (int64_t)kk * k;
          for (int i = 0; i < kk; ++i)
            for (int j = 0; j < k; ++j) R[(size_t)i * k + j] = (j >= i) ? A[(size_t)i + (size_t)j * M] : 0.0;
          for (int j = 0; j < k; ++j) piv_out[g * k + j] = jpvt[j] - 1;
          L.orgqr(&m, &kq, &kq, A.data(), &lda, tau.data(), wk.data(), &lw, &info);
          if (info != 0) { int64_t e = -1; failed.compare_exchange_strong(e, g); continue; }
          double* Q = q_out + g * (int64_t)M * kk;
          for (int i = 0; i < M; ++i)
            for (int j = 0; j < kk; ++j) Q[(size_t)i * kk + j] = A[(size_t)i + (size_t)j * M];
        }
      }
      if (L.set_threads_local) L.set_threads_local(prev);
    };
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads, (G + 255) / 256));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    CAMG_CHECK(!bad_dof, CAMG_ERR_ARG, "qr_batch: DOF index out of range");
    if (info_out) *info_out = failed.load();
  });
}

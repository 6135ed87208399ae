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

#include <cmath>

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

// QR of G blocks of M x k (block g = rows dofs[g*M ..) of vecs) on nthreads
// host threads; returns the first block LAPACK rejected, or -1
static int64_t qr_blocks(const Lapack& L, int64_t G, int M, int k, const double* vecs, int64_t n_dofs,
                         const int64_t* dofs, double* q_out, double* r_out, int64_t* piv_out, int nthreads) {
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
  return failed.load();
}

Csr* tentative_assemble(int64_t n_dofs, int64_t ncoarse, int64_t ngroups, const int64_t* meta, const int64_t* dofs,
                        int64_t ndofs_total, const double* Q, int64_t nq, const int64_t* rank, const int64_t* col0,
                        int64_t naggs);

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
    const int64_t f = qr_blocks(L, G, M, k, vecs, n_dofs, dofs, q_out, r_out, piv_out, nthreads);
    if (info_out) *info_out = f;
  });
}

// The whole tentative prolongator (transfer.py:86-145) natively: DOFs grouped
// by aggregate (ascending within, as a stable sort), aggregates grouped by
// size (ascending, ids ascending within), one LAPACK pivoted QR per aggregate
// on host threads, rank by |r_ii| > tol |r_00|, the coarse null space rows
// R P^T of the kept columns, and the CSR of P on the device.  Outputs:
// rank_out (na), coarse_ns (rows in aggregate order, <= na*k rows x k),
// *ncoarse.  Errors name the aggregate (empty; identically zero block).
extern "C" int camg_tentative(const char* lapack_path, int64_t n_dofs, int k, const double* vecs,
                              const int64_t* dof_node, const int64_t* node_to_agg, int64_t num_nodes, int64_t na,
                              double rank_tol, int nthreads, camg_csr** P_out, int64_t* rank_out, double* coarse_ns,
                              int64_t* ncoarse) {
  return guarded([&] {
    CAMG_CHECK(n_dofs >= 1 && k >= 1 && na >= 1, CAMG_ERR_ARG, "tentative: bad sizes");
    const Lapack& L = lapack(lapack_path);
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
    for (int64_t i = 0; i < n_dofs; ++i) order[at[agg_of[i]]++] = i;  // stable by aggregate
    // size groups (ascending size; aggregate ids ascending within)
    std::vector<std::pair<int64_t, int64_t>> bysize(na);
    for (int64_t a = 0; a < na; ++a) bysize[a] = {cnt[a + 1], a};
    std::sort(bysize.begin(), bysize.end());
    std::vector<int64_t> meta, dofs_f(n_dofs), rank_f(na), col0_f(na), agg_f(na);
    // Q of every group in one uninitialised buffer (about 1 GB at C5 level 0)
    int64_t q_total = 0;
    for (int64_t a = 0; a < na; ++a) q_total += bysize[a].first * std::min<int64_t>(bysize[a].first, k);
    std::unique_ptr<double[]> q_f(new double[(size_t)std::max<int64_t>(q_total, 1)]);
    int64_t dof_off = 0, q_off = 0, agg_off = 0;
    std::vector<int64_t> r_all(na);
    std::vector<double> Rf_all((size_t)na * k * k);  // R P^T rows of every aggregate (kk <= k rows)
    std::vector<int> kk_of(na);
    for (int64_t g0 = 0; g0 < na;) {
      const int64_t M = bysize[g0].first;
      int64_t g1 = g0;
      while (g1 < na && bysize[g1].first == M) ++g1;
      const int64_t G = g1 - g0;
      const int kk = (int)std::min<int64_t>(M, k);
      std::vector<int64_t> dofs((size_t)G * M);
      for (int64_t g = 0; g < G; ++g) {
        const int64_t a = bysize[g0 + g].second;
        agg_f[agg_off + g] = a;
        for (int64_t i = 0; i < M; ++i) dofs[g * M + i] = order[start[a] + i];
      }
      std::copy(dofs.begin(), dofs.end(), dofs_f.begin() + dof_off);
      std::vector<double> R((size_t)G * kk * k);
      std::vector<int64_t> piv((size_t)G * k);
      const int64_t f = qr_blocks(L, G, (int)M, k, vecs, n_dofs, dofs.data(), q_f.get() + q_off, R.data(), piv.data(),
                                  nthreads);
      if (f >= 0) throw Error(CAMG_ERR_SETUP, "pivoted QR failed on aggregate " + std::to_string(bysize[g0 + f].second));
      for (int64_t g = 0; g < G; ++g) {
        const int64_t a = bysize[g0 + g].second;
        const double* Rg = R.data() + g * (int64_t)kk * k;
        const double d0 = std::fabs(Rg[0]);
        if (!(d0 > 0.0))
          throw Error(CAMG_ERR_SETUP, "aggregate " + std::to_string(a) + ": near-kernel block is identically zero");
        int64_t r = 0;
        for (int i = 0; i < kk; ++i) r += std::fabs(Rg[(size_t)i * k + i]) > rank_tol * d0;
        r_all[a] = r;
        rank_f[agg_off + g] = r;
        kk_of[a] = kk;
        double* Rf = Rf_all.data() + (size_t)a * k * k;
        for (int i = 0; i < kk; ++i)
          for (int j = 0; j < k; ++j) Rf[(size_t)i * k + piv[g * k + j]] = Rg[(size_t)i * k + j];
      }
      meta.insert(meta.end(), {G, M, (int64_t)kk, dof_off, q_off, agg_off});
      dof_off += G * M;
      q_off += G * M * kk;
      agg_off += G;
      g0 = g1;
    }
    std::vector<int64_t> col0(na + 1, 0);
    for (int64_t a = 0; a < na; ++a) col0[a + 1] = col0[a] + r_all[a];
    for (int64_t a = 0; a < na; ++a) {
      rank_out[a] = r_all[a];
      for (int64_t i = 0; i < r_all[a]; ++i)
        for (int j = 0; j < k; ++j) coarse_ns[(size_t)(col0[a] + i) * k + j] = Rf_all[(size_t)a * k * k + i * k + j];
    }
    for (int64_t g = 0; g < na; ++g) col0_f[g] = col0[agg_f[g]];
    *ncoarse = col0[na];
    *P_out = new camg_csr{tentative_assemble(n_dofs, col0[na], (int64_t)meta.size() / 6, meta.data(), dofs_f.data(),
                                             n_dofs, q_f.get(), q_total, rank_f.data(), col0_f.data(),
                                             na)};
  });
}

// Reference-semantics point smoothers on the device (smoothers.py:141-199).
//
// sgs:   x += (tril(A,-1) + D/w)^-1 (b - A x);  x += (triu(A,1) + D/w)^-1 (b - A x)
//        per sweep (smoothers.py:155-164, 189-191: SuperLU solves of the two
//        triangles with natural ordering);
// ilu0:  x += U^-1 L^-1 (b - A x) with the reference IKJ factor values on A's
//        pattern, L unit lower, U upper with its diagonal (smoothers.py:80-138,
//        193-196);
// jacobi x += (w/d) (b - A x) (smoothers.py:185-187);
// direct x = LU^-1 b (smoothers.py:182-183; LAPACK factors from the host).
//
// Triangular solves are sync-free (the order of the lexicographic sweep is
// kept exactly; only the summation order inside a row differs from SuperLU's
// column sweep, a last-bit effect): every warp takes the next row from a
// global ticket (increasing for lower, decreasing for upper solves), so a row
// is only ever waited on by rows handed out after it -- the warps holding the
// rows it depends on are already running, which makes the scheme
// deadlock-free for any grid size.  A lane waits (ld.acquire.gpu) for the
// completion flag of each column it reads, then reads that entry coherently
// (ld.relaxed.gpu); the row's lane 0 publishes y_i and its flag with
// st.release.gpu.  A watchdog bounds every wait (err flag, no hang).

#include "pointsolve.cuh"

namespace camg {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kTrsvSpinLimit = 1 << 22;

template <bool LOWER>
__global__ void __launch_bounds__(256) k_sptrsv(int64_t n, CsrView T, const double* __restrict__ diag,
                                                const double* __restrict__ r, double* y, unsigned* flags,
                                                unsigned long long* ticket, int* err) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= (unsigned long long)n) return;
    const int64_t i = LOWER ? (int64_t)t : n - 1 - (int64_t)t;
    const int64_t s0 = T.rowptr[i], e0 = T.rowptr[i + 1];
    double acc = 0.0;
    for (int64_t q = s0 + lane; q < e0; q += 32) {
      const int32_t j = T.col[q];
      CAMG_DCHECK(j >= 0 && j < n && (LOWER ? j < i : j > i), "triangular solve column out of range / wrong side");
      const double a = T.val[q];
      unsigned f = ld_acquire_u32(flags + j);
      int spins = 0;
      while (!f) {
        if (++spins > kTrsvSpinLimit) {
          atomicExch(err, 1);
          break;
        }
        __nanosleep(64);
        f = ld_acquire_u32(flags + j);
      }
      acc = fma(a, ld_relaxed_f64(y + j), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const double v = r[i] - acc;
      y[i] = diag ? v / diag[i] : v;
      st_release_u32(flags + i, 1u);
    }
    __syncwarp();
  }
}

size_t sptrsv_sync_bytes(int64_t n) { return 8 + 4 * (size_t)n; }

void sptrsv(const Csr* Toff, const double* diag, bool lower, const double* r, double* y, void* sync, int* err,
            cudaStream_t s) {
  const int64_t n = Toff->n_rows;
  if (n == 0) return;
  CAMG_CUDA(cudaMemsetAsync(sync, 0, sptrsv_sync_bytes(n), s));
  auto* ticket = static_cast<unsigned long long*>(sync);
  auto* flags = reinterpret_cast<unsigned*>(static_cast<char*>(sync) + 8);
  const unsigned grid = grid_for(n * 32, 256, 148LL * 8);
  note_launch();
  if (lower)
    k_sptrsv<true><<<grid, 256, 0, s>>>(n, view(Toff), diag, r, y, flags, ticket, err);
  else
    k_sptrsv<false><<<grid, 256, 0, s>>>(n, view(Toff), diag, r, y, flags, ticket, err);
  CAMG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------

__global__ void k_tri_count(CsrView A, bool lower, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n_rows; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int64_t q = A.rowptr[i]; q < A.rowptr[i + 1]; ++q) c += lower ? (A.col[q] < i) : (A.col[q] > i);
    cnt[i] = c;
  }
}

__global__ void k_tri_fill(CsrView A, bool lower, const int64_t* __restrict__ rp, int32_t* __restrict__ col,
                          double* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n_rows; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = rp[i];
    for (int64_t q = A.rowptr[i]; q < A.rowptr[i + 1]; ++q) {
      const int32_t c = A.col[q];
      if (lower ? (c < i) : (c > i)) {
        col[o] = c;
        val[o] = A.val[q];
        ++o;
      }
    }
  }
}

// strict lower / upper triangle of A (pattern order kept)
static Csr* strict_triangle(const Csr* A, bool lower, cudaStream_t s) {
  const int64_t n = A->n_rows;
  DBuf<int64_t> cnt(n + 1);
  note_launch();
  k_tri_count<<<grid_for(n, 256), 256, 0, s>>>(view(A), lower, cnt.p);
  DBuf<int64_t> rp(n + 1);
  exclusive_scan_i64(cnt.p, rp.p, n, s);
  const int64_t nnz = read_i64(rp.p + n);
  Csr* T = csr_alloc(n, A->n_cols, nnz);
  CAMG_CUDA(cudaMemcpyAsync(T->rowptr, rp.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  note_launch();
  k_tri_fill<<<grid_for(n, 256), 256, 0, s>>>(view(A), lower, T->rowptr, T->col, T->val);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  T->avg_row = n ? double(nnz) / n : 0.0;
  return T;
}

static Csr* upload_csr(int64_t n, const std::vector<int64_t>& rp, const std::vector<int32_t>& ci,
                       const std::vector<double>& va) {
  Csr* T = csr_alloc(n, n, rp[n]);
  CAMG_CUDA(cudaMemcpy(T->rowptr, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  if (rp[n]) {
    CAMG_CUDA(cudaMemcpy(T->col, ci.data(), sizeof(int32_t) * rp[n], cudaMemcpyHostToDevice));
    CAMG_CUDA(cudaMemcpy(T->val, va.data(), sizeof(double) * rp[n], cudaMemcpyHostToDevice));
  }
  T->avg_row = n ? double(rp[n]) / n : 0.0;
  return T;
}

__global__ void k_first_zero_i(int64_t n, const double* __restrict__ d, unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (d[i] == 0.0) atomicMin(out, (unsigned long long)i);
}

__global__ void k_scale_div(int64_t n, const double* __restrict__ d, double num, double den, double* __restrict__ o,
                            bool recip) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = recip ? num / d[i] : d[i] / den;
}

// out = (zero ? 0 : out) + (d ? d .* v : v)
__global__ void k_ps_update(int64_t n, bool zero, const double* __restrict__ d, const double* __restrict__ v,
                            double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double add = d ? d[i] * v[i] : v[i];
    out[i] = zero ? add : out[i] + add;
  }
}

void PointSolver::setup(const Csr* A_, int kind_, int sweeps_, double damping_) {
  CAMG_CHECK(A_->n_rows == A_->n_cols, CAMG_ERR_DIMENSION, "point smoother needs a square matrix");
  CAMG_CHECK(kind_ == CAMG_PT_JACOBI || kind_ == CAMG_PT_SGS || kind_ == CAMG_PT_ILU0 || kind_ == CAMG_PT_DIRECT,
             CAMG_ERR_CONFIG, "point smoother kind must be jacobi, sgs, ilu0 or direct");
  CAMG_CHECK(sweeps_ >= 1, CAMG_ERR_CONFIG, "point smoother sweeps must be >= 1");
  A = A_;
  n = A->n_rows;
  kind = kind_;
  sweeps = sweeps_;
  damping = damping_;
  cudaStream_t s = 0;
  err = DBuf<int>(1);
  CAMG_CUDA(cudaMemset(err.p, 0, sizeof(int)));
  w_r = DBuf<double>(n + 1);
  w_d = DBuf<double>(n + 1);
  w_sync = DBuf<double>(sptrsv_sync_bytes(n) / 8 + 1);
  if (kind == CAMG_PT_DIRECT || n == 0) return;  // factors come from set_lu
  if (kind == CAMG_PT_JACOBI || kind == CAMG_PT_SGS) {
    DBuf<double> d(n + 1);
    csr_diagonal(A, 0, d.p, s);
    DBuf<unsigned long long> first(1);
    unsigned long long init = ~0ull;
    CAMG_CUDA(cudaMemcpy(first.p, &init, sizeof(init), cudaMemcpyHostToDevice));
    note_launch();
    k_first_zero_i<<<grid_for(n, 256), 256>>>(n, d.p, first.p);
    unsigned long long h = 0;
    CAMG_CUDA(cudaMemcpy(&h, first.p, sizeof(h), cudaMemcpyDeviceToHost));
    if (h != ~0ull)
      throw Error(CAMG_ERR_SINGULAR, std::string(kind == CAMG_PT_JACOBI ? "jacobi" : "sgs") +
                                         ": zero diagonal in row " + std::to_string(h));
    if (kind == CAMG_PT_JACOBI) {
      dinv = DBuf<double>(n + 1);
      note_launch();
      k_scale_div<<<grid_for(n, 256), 256>>>(n, d.p, damping, 1.0, dinv.p, true);  // smoothers.py:152
    } else {
      dsgs = DBuf<double>(n + 1);
      note_launch();
      k_scale_div<<<grid_for(n, 256), 256>>>(n, d.p, 0.0, damping, dsgs.p, false);  // smoothers.py:160
      Lo.reset(strict_triangle(A, true, s));
      Uo.reset(strict_triangle(A, false, s));
    }
    CAMG_LAUNCH_CHECK();
    CAMG_CUDA(cudaDeviceSynchronize());
    return;
  }
  // ilu0: the reference factorization on the host (smoothers.py:80-123), split
  // into the strict lower part (unit L) and the strict upper part + diagonal
  std::vector<int64_t> rp(n + 1);
  std::vector<int32_t> ci(A->nnz);
  std::vector<double> va(A->nnz);
  CAMG_CUDA(cudaMemcpy(rp.data(), A->rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
  if (A->nnz) {
    CAMG_CUDA(cudaMemcpy(ci.data(), A->col, sizeof(int32_t) * A->nnz, cudaMemcpyDeviceToHost));
    CAMG_CUDA(cudaMemcpy(va.data(), A->val, sizeof(double) * A->nnz, cudaMemcpyDeviceToHost));
  }
  std::vector<int64_t> dpos = ilu0_ikj(n, rp.data(), ci.data(), va.data(), nullptr);
  std::vector<int64_t> lrp(n + 1, 0), urp(n + 1, 0);
  std::vector<int32_t> lci, uci;
  std::vector<double> lva, uva, ud(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      if (ci[q] < i) { lci.push_back(ci[q]); lva.push_back(va[q]); }
      else if (ci[q] > i) { uci.push_back(ci[q]); uva.push_back(va[q]); }
    }
    ud[i] = va[dpos[i]];
    lrp[i + 1] = (int64_t)lci.size();
    urp[i + 1] = (int64_t)uci.size();
  }
  Lo.reset(upload_csr(n, lrp, lci, lva));
  Uo.reset(upload_csr(n, urp, uci, uva));
  udiag = DBuf<double>(n + 1);
  CAMG_CUDA(cudaMemcpy(udiag.p, ud.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
}

void PointSolver::set_lu(int64_t n_, const double* lu_h, const int32_t* piv_h) {
  CAMG_CHECK(n_ == n, CAMG_ERR_DIMENSION, "LU factors do not match the matrix");
  lu = DBuf<double>(n * n + 1);
  piv = DBuf<int32_t>(n + 1);
  CAMG_CUDA(cudaMemcpy(lu.p, lu_h, sizeof(double) * n * n, cudaMemcpyHostToDevice));
  CAMG_CUDA(cudaMemcpy(piv.p, piv_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
}

void PointSolver::smooth(const double* x, const double* b, double* out, cudaStream_t s) {
  if (n == 0) return;
  if (kind == CAMG_PT_DIRECT) {  // smoothers.py:182-183: the solve ignores x and sweeps
    CAMG_CHECK(lu.p != nullptr, CAMG_ERR_SETUP, "direct smoother factors were not set");
    lu_solve((int)n, lu.p, piv.p, b, out, s);
    return;
  }
  bool zero = (x == nullptr);
  if (!zero && x != out) CAMG_CUDA(cudaMemcpyAsync(out, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  void* sync = w_sync.p;
  // r = b - A out (zero: r = b)
  auto resid = [&]() -> const double* {
    if (zero) return b;
    CAMG_CUDA(cudaMemcpyAsync(w_r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    spmv(A, -1.0, out, 1.0, w_r.p, s);
    return w_r.p;
  };
  auto add = [&](const double* d, const double* v) {
    note_launch();
    k_ps_update<<<grid_for(n, 256), 256, 0, s>>>(n, zero, d, v, out);
    zero = false;
  };
  for (int k = 0; k < sweeps; ++k) {
    if (kind == CAMG_PT_JACOBI) {
      const double* r = resid();
      add(dinv.p, r);
    } else if (kind == CAMG_PT_SGS) {
      const double* r = resid();
      sptrsv(Lo.get(), dsgs.p, true, r, w_d.p, sync, err.p, s);
      add(nullptr, w_d.p);
      r = resid();
      sptrsv(Uo.get(), dsgs.p, false, r, w_d.p, sync, err.p, s);
      add(nullptr, w_d.p);
    } else {  // ilu0
      const double* r = resid();
      sptrsv(Lo.get(), nullptr, true, r, w_d.p, sync, err.p, s);
      sptrsv(Uo.get(), udiag.p, false, w_d.p, w_r.p, sync, err.p, s);
      add(nullptr, w_r.p);
    }
  }
  CAMG_LAUNCH_CHECK();
}

void PointSolver::check_watchdog() {
  if (!err.p) return;
  int h = 0;
  CAMG_CUDA(cudaMemcpy(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost));
  CAMG_CHECK(h == 0, CAMG_ERR_NATIVE, "triangular solve watchdog tripped (dependency never completed)");
}

}  // namespace camg

using namespace camg;

struct camg_point { camg::PointSolver P; };

extern "C" {

int camg_point_create(const camg_csr* A, int kind, int sweeps, double damping, camg_point** out) {
  return guarded([&] {
    std::unique_ptr<camg_point> p(new camg_point());
    p->P.setup(A->m, kind, sweeps, damping);
    *out = p.release();
  });
}

int camg_point_set_lu(camg_point* P, int64_t n, const double* lu, const int32_t* piv) {
  return guarded([&] {
    CAMG_CHECK(P->P.kind == CAMG_PT_DIRECT, CAMG_ERR_CONFIG, "LU factors belong to a direct smoother");
    P->P.set_lu(n, lu, piv);
  });
}

int camg_point_smooth(camg_point* P, const double* x, const double* b, double* out, void* stream) {
  return guarded([&] {
    P->P.smooth(x, b, out, (cudaStream_t)stream);
    CAMG_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    P->P.check_watchdog();
  });
}

int camg_point_destroy(camg_point* P) {
  return guarded([&] { delete P; });
}

}  // extern "C"

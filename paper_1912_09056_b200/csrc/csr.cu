// Device CSR matrices, SpMV, transpose, diagonals, sparse add, saddle merge,
// deterministic dot products.  Replaces the scipy kernels behind
// pkg/src/contactamg/sparse.py (spmv :149, sp_transpose :157,
// extract_diagonal :176) and saddle.py:58-67 (merged operator).
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"
#include "sell.cuh"

namespace camg {

static thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
thread_local int64_t g_thread_launches = 0;

void set_last_error(const std::string& msg) { g_last_error = msg; }

Csr::~Csr() {
  dfree(rowptr);
  dfree(col);
  dfree(val);
  delete sell;
}

Csr* csr_alloc(int64_t n_rows, int64_t n_cols, int64_t nnz) {
  Csr* A = new Csr();
  A->n_rows = n_rows;
  A->n_cols = n_cols;
  A->nnz = nnz;
  A->rowptr = dalloc<int64_t>(n_rows + 1);
  A->col = dalloc<int32_t>(nnz);
  A->val = dalloc<double>(nnz);
  A->avg_row = n_rows ? double(nnz) / double(n_rows) : 0.0;
  return A;
}

int64_t read_i64(const int64_t* dptr) {
  int64_t v = 0;
  CAMG_CUDA(cudaMemcpy(&v, dptr, sizeof(v), cudaMemcpyDeviceToHost));
  return v;
}

// ---------------------------------------------------------------------------
// scans

__global__ void k_set_zero_i64(int64_t* p) { *p = 0; }

void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  // out[0] = 0, out[i+1] = sum(in[0..i])
  note_launch();
  k_set_zero_i64<<<1, 1, 0, s>>>(out);
  if (n == 0) return;
  size_t tmp = 0;
  CAMG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, n, s));
  DBuf<char> t(tmp);
  note_launch();
  CAMG_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, in, out + 1, n, s));
}

// ---------------------------------------------------------------------------
// SpMV: y = alpha*A*x + beta*y over rows [row0, row0+nrows); x optionally
// split in a u part (columns < split) and a lambda part.

template <int G, bool BETA, bool SPLIT>
__global__ void __launch_bounds__(256) k_spmv(CsrView A, int64_t row0, int64_t nrows, double alpha,
                                              const double* __restrict__ xu,
                                              const double* __restrict__ xl, int64_t split,
                                              double beta, double* __restrict__ y) {
  CAMG_PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & (G - 1);
  const unsigned mask = group_mask<G>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  for (int64_t r = tid / G; r < nrows; r += stride) {
    const int64_t row = row0 + r;
    double acc = row_dot<G, SPLIT>(A, row, xu, xl, split, lane);
    acc = group_sum<G>(acc, mask);
    if (lane == 0) y[row] = BETA ? alpha * acc + beta * y[row] : alpha * acc;
  }
}

template <int G>
static void spmv_launch(const Csr* A, int64_t row0, int64_t nrows, double alpha, const double* xu,
                        const double* xl, int64_t split, double beta, double* y, cudaStream_t s) {
  const int block = 256;
  unsigned grid = grid_for(nrows * G, block, int64_t(kNumSMs) * 16);
  note_launch();
  bool sp = split < A->n_cols;
  if (beta != 0.0) {
    if (sp) launch_k(k_spmv<G, true, true>, grid, block, 0, s, view(A), row0, nrows, alpha, xu, xl, split, beta, y);
    else launch_k(k_spmv<G, true, false>, grid, block, 0, s, view(A), row0, nrows, alpha, xu, xl, split, beta, y);
  } else {
    if (sp) launch_k(k_spmv<G, false, true>, grid, block, 0, s, view(A), row0, nrows, alpha, xu, xl, split, beta, y);
    else launch_k(k_spmv<G, false, false>, grid, block, 0, s, view(A), row0, nrows, alpha, xu, xl, split, beta, y);
  }
  CAMG_LAUNCH_CHECK();
}

void spmv_rows(const Csr* A, int64_t row0, int64_t nrows, double alpha, const double* xu,
               const double* xl, int64_t split, double beta, double* y, cudaStream_t s) {
  if (nrows <= 0) return;
  switch (group_for(A->avg_row)) {
    case 1: spmv_launch<1>(A, row0, nrows, alpha, xu, xl, split, beta, y, s); break;
    case 2: spmv_launch<2>(A, row0, nrows, alpha, xu, xl, split, beta, y, s); break;
    case 4: spmv_launch<4>(A, row0, nrows, alpha, xu, xl, split, beta, y, s); break;
    case 8: spmv_launch<8>(A, row0, nrows, alpha, xu, xl, split, beta, y, s); break;
    case 16: spmv_launch<16>(A, row0, nrows, alpha, xu, xl, split, beta, y, s); break;
    default: spmv_launch<32>(A, row0, nrows, alpha, xu, xl, split, beta, y, s); break;
  }
}

void spmv(const Csr* A, double alpha, const double* x, double beta, double* y, cudaStream_t s) {
  if (A->nnz == 0) {  // y = beta*y
    vec_scale(A->n_rows, beta, y, s);
    return;
  }
  int64_t row0 = 0;
  if (A->sell) {
    SellEpi e;
    e.y = y;
    e.alpha = alpha;
    e.beta = beta;
    sell_launch(A->sell, 0, false, x, nullptr, -1, e, s);
    row0 = A->sell->rows();
  }
  spmv_rows(A, row0, A->n_rows - row0, alpha, x, nullptr, A->n_cols, beta, y, s);
}

// ---------------------------------------------------------------------------
// transpose: stable radix sort of entries by column keeps rows ascending

__global__ void k_iota_i64(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}

__global__ void k_row_of_entry(const int64_t* __restrict__ rowptr, int64_t n_rows, int32_t* __restrict__ row_of) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) row_of[p] = (int32_t)r;
}

__global__ void k_gather_transpose(const int64_t* __restrict__ perm, const int32_t* __restrict__ row_of,
                                   const double* __restrict__ val, int64_t nnz, int32_t* __restrict__ out_col,
                                   double* __restrict__ out_val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = perm[i];
    out_col[i] = row_of[e];
    out_val[i] = val[e];
  }
}

__global__ void k_count_cols(const int32_t* __restrict__ sorted_cols, int64_t nnz, int64_t n_out_rows,
                             int64_t* __restrict__ rowptr) {
  // rowptr[c] = first index i with sorted_cols[i] >= c  (lower bound), c in [0, n_out_rows]
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= n_out_rows; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sorted_cols[mid] < c) lo = mid + 1; else hi = mid;
    }
    rowptr[c] = lo;
  }
}

Csr* csr_transpose(const Csr* A, cudaStream_t s) {
  Csr* T = csr_alloc(A->n_cols, A->n_rows, A->nnz);
  const int64_t nnz = A->nnz;
  if (nnz == 0) {
    CAMG_CUDA(cudaMemsetAsync(T->rowptr, 0, sizeof(int64_t) * (T->n_rows + 1), s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    return T;
  }
  DBuf<int32_t> keys_out(nnz), row_of(nnz);
  DBuf<int64_t> idx_in(nnz), idx_out(nnz);
  note_launch(3);
  k_iota_i64<<<grid_for(nnz, 256), 256, 0, s>>>(idx_in.p, nnz);
  k_row_of_entry<<<grid_for(A->n_rows, 256), 256, 0, s>>>(A->rowptr, A->n_rows, row_of.p);
  size_t tmp = 0;
  int end_bit = 1;
  while (end_bit < 31 && (int64_t(1) << end_bit) < A->n_cols) ++end_bit;
  CAMG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, A->col, keys_out.p, idx_in.p, idx_out.p, nnz, 0, end_bit, s));
  DBuf<char> t(tmp);
  CAMG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, A->col, keys_out.p, idx_in.p, idx_out.p, nnz, 0, end_bit, s));
  note_launch(2);
  k_gather_transpose<<<grid_for(nnz, 256), 256, 0, s>>>(idx_out.p, row_of.p, A->val, nnz, T->col, T->val);
  k_count_cols<<<grid_for(T->n_rows + 1, 256), 256, 0, s>>>(keys_out.p, nnz, T->n_rows, T->rowptr);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  return T;
}

// ---------------------------------------------------------------------------
// diagonals

__global__ void k_diag(CsrView A, int mode, double* __restrict__ d) {
  const int64_t n = A.n_rows;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = A.rowptr[r], e = A.rowptr[r + 1];
    double v = 0.0;
    if (mode == 0) {
      int64_t lo = s, hi = e;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (A.col[mid] < r) lo = mid + 1; else hi = mid;
      }
      if (lo < e && A.col[lo] == r) v = A.val[lo];
    } else {
      // sequential row order, matching scipy's abs(A).sum(axis=1) closely
      for (int64_t p = s; p < e; ++p) v += fabs(A.val[p]);
    }
    d[r] = v;
  }
}

void csr_diagonal(const Csr* A, int mode, double* d, cudaStream_t s) {
  note_launch();
  k_diag<<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), mode, d);
  CAMG_LAUNCH_CHECK();
}

Csr* csr_copy(const Csr* A, cudaStream_t s) {
  Csr* C = csr_alloc(A->n_rows, A->n_cols, A->nnz);
  CAMG_CUDA(cudaMemcpyAsync(C->rowptr, A->rowptr, sizeof(int64_t) * (A->n_rows + 1), cudaMemcpyDeviceToDevice, s));
  CAMG_CUDA(cudaMemcpyAsync(C->col, A->col, sizeof(int32_t) * A->nnz, cudaMemcpyDeviceToDevice, s));
  CAMG_CUDA(cudaMemcpyAsync(C->val, A->val, sizeof(double) * A->nnz, cudaMemcpyDeviceToDevice, s));
  CAMG_CUDA(cudaStreamSynchronize(s));
  return C;
}

// ---------------------------------------------------------------------------
// C = alpha*A + beta*B (canonical inputs, scipy csr_binop_csr_canonical order)

template <bool FILL>
__global__ void k_axpby(CsrView A, CsrView B, double alpha, double beta, int64_t* __restrict__ cnt,
                        const int64_t* __restrict__ crow, int32_t* __restrict__ ccol, double* __restrict__ cval) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t pa = A.rowptr[r], ea = A.rowptr[r + 1], pb = B.rowptr[r], eb = B.rowptr[r + 1];
    int64_t out = FILL ? crow[r] : 0;
    int64_t n = 0;
    while (pa < ea || pb < eb) {
      int32_t ca = pa < ea ? A.col[pa] : INT32_MAX;
      int32_t cb = pb < eb ? B.col[pb] : INT32_MAX;
      double v;
      int32_t c;
      if (ca == cb) { v = __dadd_rn(__dmul_rn(alpha, A.val[pa]), __dmul_rn(beta, B.val[pb])); c = ca; ++pa; ++pb; }
      else if (ca < cb) { v = __dadd_rn(__dmul_rn(alpha, A.val[pa]), 0.0); c = ca; ++pa; }
      else { v = __dadd_rn(0.0, __dmul_rn(beta, B.val[pb])); c = cb; ++pb; }
      if (fabs(v) >= kDropTol) {
        if (FILL) { ccol[out + n] = c; cval[out + n] = v; }
        ++n;
      }
    }
    if (!FILL) cnt[r] = n;
  }
}

Csr* csr_axpby(double alpha, const Csr* A, double beta, const Csr* B, cudaStream_t s) {
  CAMG_CHECK(A->n_rows == B->n_rows && A->n_cols == B->n_cols, CAMG_ERR_DIMENSION, "axpby: shape mismatch");
  DBuf<int64_t> cnt(A->n_rows + 1);
  note_launch();
  k_axpby<false><<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), view(B), alpha, beta, cnt.p, nullptr, nullptr, nullptr);
  CAMG_LAUNCH_CHECK();
  DBuf<int64_t> rp(A->n_rows + 1);
  exclusive_scan_i64(cnt.p, rp.p, A->n_rows, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  int64_t nnz = read_i64(rp.p + A->n_rows);
  Csr* C = new Csr();
  C->n_rows = A->n_rows; C->n_cols = A->n_cols; C->nnz = nnz;
  C->rowptr = rp.release();
  C->col = dalloc<int32_t>(nnz);
  C->val = dalloc<double>(nnz);
  C->avg_row = C->n_rows ? double(nnz) / C->n_rows : 0.0;
  note_launch();
  k_axpby<true><<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), view(B), alpha, beta, nullptr, C->rowptr, C->col, C->val);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  return C;
}

// ---------------------------------------------------------------------------
// C = diag(s) A, exact zeros / denormals dropped (scipy multiply + canon)

template <bool FILL>
__global__ void k_scale_rows(CsrView A, const double* __restrict__ sc, int64_t* __restrict__ cnt,
                             const int64_t* __restrict__ crow, int32_t* __restrict__ ccol, double* __restrict__ cval) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = 0, out = FILL ? crow[r] : 0;
    const double f = sc[r];
    for (int64_t p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) {
      double v = __dmul_rn(A.val[p], f);
      if (fabs(v) >= kDropTol) {
        if (FILL) { ccol[out + n] = A.col[p]; cval[out + n] = v; }
        ++n;
      }
    }
    if (!FILL) cnt[r] = n;
  }
}

Csr* csr_scale_rows(const Csr* A, const double* sc, cudaStream_t s) {
  DBuf<int64_t> cnt(A->n_rows + 1);
  note_launch();
  k_scale_rows<false><<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), sc, cnt.p, nullptr, nullptr, nullptr);
  DBuf<int64_t> rp(A->n_rows + 1);
  exclusive_scan_i64(cnt.p, rp.p, A->n_rows, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  int64_t nnz = read_i64(rp.p + A->n_rows);
  Csr* C = new Csr();
  C->n_rows = A->n_rows; C->n_cols = A->n_cols; C->nnz = nnz;
  C->rowptr = rp.release();
  C->col = dalloc<int32_t>(nnz);
  C->val = dalloc<double>(nnz);
  C->avg_row = C->n_rows ? double(nnz) / C->n_rows : 0.0;
  note_launch();
  k_scale_rows<true><<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), sc, nullptr, C->rowptr, C->col, C->val);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  return C;
}

// ---------------------------------------------------------------------------
// merged saddle operator [[K, B1], [B2, -Cz]]

__global__ void k_merge_counts(CsrView K, CsrView B1, CsrView B2, CsrView Cz, int64_t* __restrict__ cnt) {
  const int64_t nu = K.n_rows, n = K.n_rows + Cz.n_rows;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (r < nu) cnt[r] = (K.rowptr[r + 1] - K.rowptr[r]) + (B1.rowptr[r + 1] - B1.rowptr[r]);
    else {
      int64_t q = r - nu;
      cnt[r] = (B2.rowptr[q + 1] - B2.rowptr[q]) + (Cz.rowptr[q + 1] - Cz.rowptr[q]);
    }
  }
}

__global__ void k_merge_fill(CsrView K, CsrView B1, CsrView B2, CsrView Cz, const int64_t* __restrict__ rp,
                             int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t nu = K.n_rows, n = K.n_rows + Cz.n_rows;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    const CsrView& L = r < nu ? K : B2;
    const CsrView& Rm = r < nu ? B1 : Cz;
    const int64_t q = r < nu ? r : r - nu;
    const double sgn = r < nu ? 1.0 : -1.0;
    int64_t o = rp[r];
    int64_t ls = L.rowptr[q], le = L.rowptr[q + 1];
    for (int64_t p = ls + lane; p < le; p += 32) { col[o + p - ls] = L.col[p]; val[o + p - ls] = L.val[p]; }
    o += le - ls;
    int64_t rs = Rm.rowptr[q], re = Rm.rowptr[q + 1];
    for (int64_t p = rs + lane; p < re; p += 32) {
      col[o + p - rs] = (int32_t)(Rm.col[p] + nu);
      val[o + p - rs] = sgn * Rm.val[p];
    }
  }
}

Csr* csr_saddle_merge(const Csr* K, const Csr* B1, const Csr* B2, const Csr* Cz, cudaStream_t s) {
  const int64_t nu = K->n_rows, nl = Cz->n_rows;
  CAMG_CHECK(K->n_cols == nu && Cz->n_cols == nl, CAMG_ERR_DIMENSION, "K and Cz must be square");
  CAMG_CHECK(B1->n_rows == nu && B1->n_cols == nl && B2->n_rows == nl && B2->n_cols == nu,
             CAMG_ERR_DIMENSION, "saddle block dimensions are inconsistent");
  const int64_t n = nu + nl;
  DBuf<int64_t> cnt(n + 1);
  note_launch();
  k_merge_counts<<<grid_for(n, 256), 256, 0, s>>>(view(K), view(B1), view(B2), view(Cz), cnt.p);
  DBuf<int64_t> rp(n + 1);
  exclusive_scan_i64(cnt.p, rp.p, n, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  int64_t nnz = read_i64(rp.p + n);
  Csr* C = new Csr();
  C->n_rows = n; C->n_cols = n; C->nnz = nnz;
  C->rowptr = rp.release();
  C->col = dalloc<int32_t>(nnz);
  C->val = dalloc<double>(nnz);
  C->avg_row = n ? double(nnz) / n : 0.0;
  note_launch();
  k_merge_fill<<<grid_for(n * 32, 256), 256, 0, s>>>(view(K), view(B1), view(B2), view(Cz), C->rowptr, C->col, C->val);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  return C;
}

// ---------------------------------------------------------------------------
// vector helpers (deterministic reductions)

__global__ void k_dot_partial(int64_t n, const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(x[i], y[i], acc);
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_sum_partials(const double* __restrict__ part, int n, double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) *out = acc;
}

void dot_device(int64_t n, const double* x, const double* y, double* out_dev, double* part, cudaStream_t s) {
  note_launch(2);
  k_dot_partial<<<kDotBlocks, 256, 0, s>>>(n, x, y, part);
  k_sum_partials<<<1, 256, 0, s>>>(part, kDotBlocks, out_dev);
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

void vec_axpy(int64_t n, double a, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  note_launch();
  k_axpy<<<grid_for(n, 256), 256, 0, s>>>(n, a, x, y);
}

__global__ void k_scale(int64_t n, double a, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a == 0.0 ? 0.0 : a * y[i];
}

void vec_scale(int64_t n, double a, double* y, cudaStream_t s) {
  if (n <= 0) return;
  note_launch();
  k_scale<<<grid_for(n, 256), 256, 0, s>>>(n, a, y);
}

// w = (A v) / d in scipy csr_matvec order (sequential over the row, no FMA
// contraction): one warp per row loads 32 entries at a time coalesced, forms
// the products in parallel and lane 0 adds them in row order.
__global__ void k_power_step(CsrView A, const double* __restrict__ d, const double* __restrict__ v, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < A.n_rows; r += nwarps) {
    const int64_t s = A.rowptr[r], e = A.rowptr[r + 1];
    double acc = 0.0;
    for (int64_t c0 = s; c0 < e; c0 += 32) {
      const int64_t p = c0 + lane;
      const double prod = p < e ? __dmul_rn(A.val[p], v[A.col[p]]) : 0.0;
      const int n = (int)((e - c0) < 32 ? (e - c0) : 32);
      for (int j = 0; j < n; ++j) {
        const double t = __shfl_sync(0xffffffffu, prod, j);
        acc = __dadd_rn(acc, t);
      }
    }
    if (lane == 0) w[r] = __ddiv_rn(acc, d[r]);
  }
}

__global__ void k_div(int64_t n, const double* __restrict__ w, double s, double* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __ddiv_rn(w[i], s);
}

bool use_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CAMG_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// lambda_max(D^-1 A) by power iteration from ones/sqrt(n) (the algorithm of
// transfer.py:148-161, device norms): bounds of the Chebyshev predictor
double lambda_max_dinv(const Csr* A, const double* d, int iters, cudaStream_t s) {
  const int64_t n = A->n_rows;
  if (n == 0) return 1.0;
  DBuf<double> v(n + 1), w(n + 1), part(kDotBlocks + 1);
  std::vector<double> ones(n, 1.0 / std::sqrt((double)n));
  CAMG_CUDA(cudaMemcpy(v.p, ones.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  double lam = 1.0;
  for (int k = 0; k < iters; ++k) {
    note_launch();
    k_power_step<<<grid_for(n * 32, 256), 256, 0, s>>>(view(A), d, v.p, w.p);
    dot_device(n, w.p, w.p, part.p + kDotBlocks, part.p, s);
    double nn = 0.0;
    CAMG_CUDA(cudaMemcpyAsync(&nn, part.p + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    const double nrm = std::sqrt(nn);
    if (nrm == 0.0) return 1.0;
    lam = nrm;
    note_launch();
    k_div<<<grid_for(n, 256), 256, 0, s>>>(n, w.p, nrm, v.p);
  }
  CAMG_LAUNCH_CHECK();
  return lam;
}

}  // namespace camg

// lambda_max(D^-1 A) by `iters` power steps from ones/sqrt(n) with device
// norms (transfer.py:148-161) for hosts that do not reproduce numpy's norm;
// d = diag(A) on the device (null: extracted here)
extern "C" int camg_lambda_max(const camg_csr* A, const double* d, int iters, double* out) {
  return camg::guarded([&] {
    const camg::Csr* M = A->m;
    CAMG_CHECK(M->n_rows == M->n_cols, CAMG_ERR_DIMENSION, "lambda_max: square matrix required");
    camg::DBuf<double> dd;
    if (!d) {
      dd = camg::DBuf<double>(M->n_rows + 1);
      camg::csr_diagonal(M, 0, dd.p, 0);
      d = dd.p;
    }
    *out = camg::lambda_max_dinv(M, d, iters, 0);
  });
}

using namespace camg;

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char* camg_last_error(void) { return g_last_error.c_str(); }
int camg_version(void) { return 100; }
int64_t camg_launch_count(void) { return g_launches.load(); }

int camg_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) { cudaGetLastError(); n = 0; }
    *count = n;
  });
}

int camg_csr_from_host(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rowptr,
                       const int64_t* col, const double* val, camg_csr** out) {
  return guarded([&] {
    CAMG_CHECK(n_rows >= 0 && n_cols >= 0 && nnz >= 0, CAMG_ERR_DIMENSION, "negative size");
    CAMG_CHECK(n_cols < INT32_MAX, CAMG_ERR_DIMENSION, "n_cols exceeds int32 column range");
    CAMG_CHECK(rowptr[0] == 0 && rowptr[n_rows] == nnz, CAMG_ERR_DIMENSION,
               "row_offsets must start at 0 and end at nnz");
    std::vector<int32_t> c32(nnz);
    for (int64_t i = 0; i < nnz; ++i) {
      CAMG_CHECK(col[i] >= 0 && col[i] < n_cols, CAMG_ERR_DIMENSION, "column index out of range");
      c32[i] = (int32_t)col[i];
    }
    Csr* A = csr_alloc(n_rows, n_cols, nnz);
    CAMG_CUDA(cudaMemcpy(A->rowptr, rowptr, sizeof(int64_t) * (n_rows + 1), cudaMemcpyHostToDevice));
    if (nnz) {
      CAMG_CUDA(cudaMemcpy(A->col, c32.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
      CAMG_CUDA(cudaMemcpy(A->val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
    *out = new camg_csr{A};
  });
}

int camg_csr_from_device(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rowptr,
                         const int32_t* col, const double* val, camg_csr** out) {
  return guarded([&] {
    Csr* A = csr_alloc(n_rows, n_cols, nnz);
    CAMG_CUDA(cudaMemcpy(A->rowptr, rowptr, sizeof(int64_t) * (n_rows + 1), cudaMemcpyDeviceToDevice));
    if (nnz) {
      CAMG_CUDA(cudaMemcpy(A->col, col, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice));
      CAMG_CUDA(cudaMemcpy(A->val, val, sizeof(double) * nnz, cudaMemcpyDeviceToDevice));
    }
    *out = new camg_csr{A};
  });
}

int camg_csr_alloc(int64_t n_rows, int64_t n_cols, int64_t nnz, camg_csr** out) {
  return guarded([&] { *out = new camg_csr{csr_alloc(n_rows, n_cols, nnz)}; });
}

int camg_csr_destroy(camg_csr* A) {
  return guarded([&] {
    if (A) { delete A->m; delete A; }
  });
}

int camg_csr_shape(const camg_csr* A, int64_t* n_rows, int64_t* n_cols, int64_t* nnz) {
  return guarded([&] {
    *n_rows = A->m->n_rows;
    *n_cols = A->m->n_cols;
    *nnz = A->m->nnz;
  });
}

int camg_csr_to_host(const camg_csr* A, int64_t* rowptr, int64_t* col, double* val) {
  return guarded([&] {
    const Csr* M = A->m;
    CAMG_CUDA(cudaDeviceSynchronize());
    CAMG_CUDA(cudaMemcpy(rowptr, M->rowptr, sizeof(int64_t) * (M->n_rows + 1), cudaMemcpyDeviceToHost));
    if (M->nnz) {
      std::vector<int32_t> c32(M->nnz);
      CAMG_CUDA(cudaMemcpy(c32.data(), M->col, sizeof(int32_t) * M->nnz, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < M->nnz; ++i) col[i] = c32[i];
      CAMG_CUDA(cudaMemcpy(val, M->val, sizeof(double) * M->nnz, cudaMemcpyDeviceToHost));
    }
  });
}

int camg_csr_saddle_merge(const camg_csr* K, const camg_csr* B1, const camg_csr* B2, const camg_csr* Cz,
                          camg_csr** out) {
  return guarded([&] { *out = new camg_csr{csr_saddle_merge(K->m, B1->m, B2->m, Cz->m, 0)}; });
}

int camg_spmv(const camg_csr* A, double alpha, const double* x, double beta, double* y, void* stream) {
  return guarded([&] {
    spmv(A->m, alpha, x, beta, y, (cudaStream_t)stream);
    CAMG_LAUNCH_CHECK();
  });
}

int camg_transpose(const camg_csr* A, camg_csr** out) {
  return guarded([&] { *out = new camg_csr{csr_transpose(A->m, 0)}; });
}

int camg_diagonal(const camg_csr* A, int mode, double* d) {
  return guarded([&] {
    CAMG_CHECK(A->m->n_rows == A->m->n_cols, CAMG_ERR_DIMENSION, "extract_diagonal: matrix must be square");
    CAMG_CHECK(mode == 0 || mode == 1, CAMG_ERR_ARG, "unknown diagonal mode");
    csr_diagonal(A->m, mode, d, 0);
    CAMG_CUDA(cudaDeviceSynchronize());
  });
}

int camg_csr_axpby(double alpha, const camg_csr* A, double beta, const camg_csr* B, camg_csr** out) {
  return guarded([&] { *out = new camg_csr{csr_axpby(alpha, A->m, beta, B->m, 0)}; });
}

int camg_csr_scale_rows(const camg_csr* A, const double* s, camg_csr** out) {
  return guarded([&] { *out = new camg_csr{csr_scale_rows(A->m, s, 0)}; });
}

int camg_power_step(const camg_csr* A, const double* d, const double* v, double* w, void* stream) {
  return guarded([&] {
    note_launch();
    k_power_step<<<grid_for(A->m->n_rows * 32, 256), 256, 0, (cudaStream_t)stream>>>(view(A->m), d, v, w);
    CAMG_LAUNCH_CHECK();
  });
}

int camg_vec_scale_div(int64_t n, const double* w, double s, double* v, void* stream) {
  return guarded([&] {
    note_launch();
    k_div<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, w, s, v);
    CAMG_LAUNCH_CHECK();
  });
}

int camg_dot(int64_t n, const double* x, const double* y, double* result, void* stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    DBuf<double> part(kDotBlocks + 1);
    dot_device(n, x, y, part.p + kDotBlocks, part.p, s);
    CAMG_CUDA(cudaMemcpyAsync(result, part.p + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
  });
}

int camg_axpy(int64_t n, double alpha, const double* x, double* y, void* stream) {
  return guarded([&] {
    vec_axpy(n, alpha, x, y, (cudaStream_t)stream);
    CAMG_LAUNCH_CHECK();
  });
}

void camg_free_host(void* p) { free(p); }

}  // extern "C"

// Device assembly of the structured two-block stiffness matrix from the
// per-(boundary type, neighbour offset) stencil table built on the host by
// paper_1912_09056_b200/problem.py (stencil_table).  Problem generation is
// not part of the reference hot path (problem.py is a host
// prerequisite); the large configs (C4/C5: up to 1.5e9 non-zeros) are
// assembled here because the host cannot hold their COO form.  The table
// values are looked up, not summed, so device K == host K bit for bit.
#include "common.cuh"
#include "kernels.cuh"

namespace camg {

struct Grid {
  int dim;
  int64_t N[3];
  int clamp_lo, clamp_hi;
  int64_t node_offset;
  int64_t layer;       // nodes per horizontal layer
  int64_t n_kept;
};

__device__ __forceinline__ bool kept_node(const Grid& g, int64_t iz) {
  if (g.clamp_lo && iz == 0) return false;
  if (g.clamp_hi && iz == g.N[g.dim - 1] - 1) return false;
  return true;
}

// kept-node index k (0-based within the block) -> lexicographic index
__device__ __forceinline__ int64_t lex_of_kept(const Grid& g, int64_t k) { return g.clamp_lo ? k + g.layer : k; }

template <bool FILL>
__global__ void k_stencil(Grid g, const double* __restrict__ table, int64_t row_offset, int64_t* __restrict__ cnt,
                          const int64_t* __restrict__ rp, int32_t* __restrict__ col, double* __restrict__ val) {
  const int dim = g.dim;
  const int noff = dim == 3 ? 27 : 9;
  const int64_t nrows = g.n_kept * dim;
  for (int64_t rr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; rr < nrows; rr += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = rr / dim;
    const int r = (int)(rr % dim);
    const int64_t lex = lex_of_kept(g, k);
    int64_t idx[3] = {0, 0, 0};
    int64_t rem = lex;
    int type = 0, p3 = 1;
    for (int a = 0; a < dim; ++a) {
      idx[a] = rem % g.N[a];
      rem /= g.N[a];
      const int t = idx[a] == 0 ? 0 : (idx[a] == g.N[a] - 1 ? 2 : 1);
      type += t * p3;
      p3 *= 3;
    }
    int64_t n = 0;
    int64_t out = FILL ? rp[row_offset + rr] : 0;
    for (int oi = 0; oi < noff; ++oi) {
      int off[3] = {oi % 3 - 1, (oi / 3) % 3 - 1, (oi / 9) % 3 - 1};
      bool ok = true;
      int64_t q = 0, stride = 1;
      for (int a = 0; a < dim; ++a) {
        const int64_t c = idx[a] + off[a];
        if (c < 0 || c >= g.N[a]) ok = false;
        q += c * stride;
        stride *= g.N[a];
      }
      if (!ok) continue;
      const int64_t qz = q / g.layer;
      if (!kept_node(g, qz)) continue;
      const int64_t qnew = g.node_offset + (g.clamp_lo ? q - g.layer : q);
      const double* blk = table + (((int64_t)type * noff + oi) * dim + r) * dim;
      for (int c = 0; c < dim; ++c) {
        const double v = blk[c];
        if (v == 0.0) continue;
        if (FILL) {
          col[out + n] = (int32_t)(dim * qnew + c);
          val[out + n] = v;
        }
        ++n;
      }
    }
    if (!FILL) cnt[rr] = n;
  }
}

__global__ void k_add_base(int64_t* __restrict__ rp, int64_t n, const int64_t* __restrict__ scan) {
  // rp[1..n] = rp[0] + scan[1..n]
  const int64_t base = rp[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rp[i + 1] = base + scan[i + 1];
}

static Grid make_grid(int dim, const int64_t* grid, int clamp_lo, int clamp_hi, int64_t node_offset) {
  Grid g{};
  g.dim = dim;
  for (int a = 0; a < 3; ++a) g.N[a] = a < dim ? grid[a] : 1;
  g.clamp_lo = clamp_lo;
  g.clamp_hi = clamp_hi;
  g.node_offset = node_offset;
  g.layer = 1;
  for (int a = 0; a < dim - 1; ++a) g.layer *= g.N[a];
  int64_t total = g.layer * g.N[dim - 1];
  g.n_kept = total - (clamp_lo ? g.layer : 0) - (clamp_hi ? g.layer : 0);
  return g;
}

}  // namespace camg

using namespace camg;

extern "C" {

int camg_stencil_block_counts(int dim, const int64_t* grid, int clamp_lo, int clamp_hi, const double* table,
                              int64_t* nnz_out) {
  return guarded([&] {
    CAMG_CHECK(dim == 2 || dim == 3, CAMG_ERR_ARG, "dim must be 2 or 3");
    Grid g = make_grid(dim, grid, clamp_lo, clamp_hi, 0);
    const int noff = dim == 3 ? 27 : 9;
    const int ntype = dim == 3 ? 27 : 9;
    const size_t tsz = (size_t)ntype * noff * dim * dim;
    DBuf<double> t(tsz);
    CAMG_CUDA(cudaMemcpy(t.p, table, sizeof(double) * tsz, cudaMemcpyHostToDevice));
    const int64_t nrows = g.n_kept * dim;
    DBuf<int64_t> cnt(nrows + 1), sc(nrows + 1);
    note_launch();
    k_stencil<false><<<grid_for(nrows, 256), 256>>>(g, t.p, 0, cnt.p, nullptr, nullptr, nullptr);
    exclusive_scan_i64(cnt.p, sc.p, nrows, 0);
    CAMG_CUDA(cudaDeviceSynchronize());
    *nnz_out = read_i64(sc.p + nrows);
  });
}

int camg_assemble_stencil(int dim, const int64_t* grid, int clamp_lo, int clamp_hi, int64_t node_offset,
                          int64_t n_rows_total, const double* table, camg_csr* K, int64_t row_offset) {
  return guarded([&] {
    Csr* M = K->m;
    CAMG_CHECK(M->n_rows == n_rows_total, CAMG_ERR_DIMENSION, "row count mismatch");
    Grid g = make_grid(dim, grid, clamp_lo, clamp_hi, node_offset);
    const int noff = dim == 3 ? 27 : 9;
    const int ntype = dim == 3 ? 27 : 9;
    const size_t tsz = (size_t)ntype * noff * dim * dim;
    DBuf<double> t(tsz);
    CAMG_CUDA(cudaMemcpy(t.p, table, sizeof(double) * tsz, cudaMemcpyHostToDevice));
    const int64_t nrows = g.n_kept * dim;
    CAMG_CHECK(row_offset + nrows <= M->n_rows, CAMG_ERR_DIMENSION, "block rows exceed the matrix");
    if (row_offset == 0) CAMG_CUDA(cudaMemset(M->rowptr, 0, sizeof(int64_t)));
    DBuf<int64_t> cnt(nrows + 1), sc(nrows + 1);
    note_launch();
    k_stencil<false><<<grid_for(nrows, 256), 256>>>(g, t.p, 0, cnt.p, nullptr, nullptr, nullptr);
    exclusive_scan_i64(cnt.p, sc.p, nrows, 0);
    note_launch();
    k_add_base<<<grid_for(nrows, 256), 256>>>(M->rowptr + row_offset, nrows, sc.p);
    note_launch();
    k_stencil<true><<<grid_for(nrows, 256), 256>>>(g, t.p, row_offset, nullptr, M->rowptr, M->col, M->val);
    CAMG_LAUNCH_CHECK();
    CAMG_CUDA(cudaDeviceSynchronize());
    const int64_t end = read_i64(M->rowptr + row_offset + nrows);
    CAMG_CHECK(end <= M->nnz, CAMG_ERR_DIMENSION, "assembled more entries than allocated");
    if (row_offset + nrows == M->n_rows) {
      M->nnz = end;
      M->avg_row = M->n_rows ? double(end) / M->n_rows : 0.0;
    }
  });
}

}  // extern "C"

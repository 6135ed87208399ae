// Node graph (device) and the integer aggregation (host).
//
// filtered_node_graph (aggregation.py:127-145 with NodeGraph.from_edges
// :47-63): an edge p-q exists iff some DOF pair (i in p, j in q) has a kept
// entry (|K_ij| > 0, or > eps*sqrt|K_ii K_jj|), p != q and both nodes are in
// the same body; the graph is symmetrised and sorted.  On the device this is
// the pattern of N^T F N + (N^T F N)^T with F the filtered 0/1 matrix and N
// the DOF->node incidence (all values positive, so no cancellation).
//
// aggregate_greedy (aggregation.py:186-258) and aggregate_lagrange
// (aggregation.py:261-303) are sequential integer sweeps; they run on the
// host in C++ (aggregation stays host-side in v1) and are
// bit-exact to the reference.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <unordered_map>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace camg {

Csr* galerkin(const Csr* R, const Csr* A, const Csr* P, cudaStream_t s);

template <bool FILL>
__global__ void k_filter(CsrView K, const int64_t* __restrict__ dof_node, const int8_t* __restrict__ body,
                         const double* __restrict__ diag, double eps, int64_t* __restrict__ cnt,
                         const int64_t* __restrict__ rp, int32_t* __restrict__ col, double* __restrict__ val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < K.n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ni = dof_node[r];
    int64_t n = 0, o = FILL ? rp[r] : 0;
    for (int64_t p = K.rowptr[r]; p < K.rowptr[r + 1]; ++p) {
      const int32_t c = K.col[p];
      const int64_t nj = dof_node[c];
      if (ni == nj || body[ni] != body[nj]) continue;
      const double v = fabs(K.val[p]);
      const bool keep = eps > 0.0 ? v > eps * sqrt(diag[r] * diag[c]) : v > 0.0;
      if (!keep) continue;
      if (FILL) { col[o + n] = c; val[o + n] = 1.0; }
      ++n;
    }
    if (!FILL) cnt[r] = n;
  }
}

__global__ void k_incidence(const int64_t* __restrict__ dof_node, int64_t n, int64_t* __restrict__ rp,
                            int32_t* __restrict__ col, double* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    rp[i] = i;
    if (i < n) { col[i] = (int32_t)dof_node[i]; val[i] = 1.0; }
  }
}

__global__ void k_absdiag(double* d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = fabs(d[i]);
}

// Uniform node blocks (dof_node = i / bs): node p's neighbours are the
// distinct col/bs of its bs DOF rows, filtered -- one merge per node, no
// filtered copy of K and no Galerkin product.
template <bool FILL>
__global__ void k_block_graph(CsrView K, int bs, int64_t nn, const int8_t* __restrict__ body,
                              const double* __restrict__ diag, double eps, int64_t* __restrict__ cnt,
                              const int64_t* __restrict__ rp, int32_t* __restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nn; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t pos[6], end[6];
    for (int r = 0; r < bs; ++r) {
      pos[r] = K.rowptr[p * bs + r];
      end[r] = K.rowptr[p * bs + r + 1];
    }
    int64_t n = 0, o = FILL ? rp[p] : 0;
    while (true) {
      int32_t best = INT32_MAX;
      for (int r = 0; r < bs; ++r)
        if (pos[r] < end[r]) best = min(best, K.col[pos[r]] / bs);
      if (best == INT32_MAX) break;
      bool keep = false;
      for (int r = 0; r < bs; ++r)
        while (pos[r] < end[r] && K.col[pos[r]] / bs == best) {
          const double v = fabs(K.val[pos[r]]);
          const int64_t i = p * bs + r, j = K.col[pos[r]];
          keep |= eps > 0.0 ? v > eps * sqrt(diag[i] * diag[j]) : v > 0.0;
          ++pos[r];
        }
      // columns past the node range (e.g. B1 in a merged operator) are not nodes
      if (keep && best != p && best < nn && (!body || body[best] == body[p])) {
        if (FILL) out[o + n] = best;
        ++n;
      }
    }
    if (!FILL) cnt[p] = n;
  }
}

Csr* block_graph(const Csr* K, int bs, int64_t nn, const int8_t* body, const double* diag, double eps) {
  cudaStream_t s = 0;
  DBuf<int64_t> cnt(nn + 1);
  note_launch();
  k_block_graph<false><<<grid_for(nn, 256), 256>>>(view(K), bs, nn, body, diag, eps, cnt.p, nullptr, nullptr);
  DBuf<int64_t> rp(nn + 1);
  exclusive_scan_i64(cnt.p, rp.p, nn, s);
  CAMG_CUDA(cudaDeviceSynchronize());
  const int64_t nnz = read_i64(rp.p + nn);
  Csr* G = new Csr();
  G->n_rows = nn; G->n_cols = nn; G->nnz = nnz;
  G->rowptr = rp.release();
  G->col = dalloc<int32_t>(nnz);
  G->val = dalloc<double>(nnz);
  G->avg_row = nn ? double(nnz) / nn : 0.0;
  CAMG_CUDA(cudaMemset(G->val, 0, sizeof(double) * nnz));
  note_launch();
  k_block_graph<true><<<grid_for(nn, 256), 256>>>(view(K), bs, nn, body, diag, eps, nullptr, G->rowptr, G->col);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaDeviceSynchronize());
  return G;
}

__global__ void k_fill_ones(double* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v[i] = 1.0;
}

// symmetrised node graph of uniform node blocks: no filter, no bodies, columns
// past the node range ignored (the multicolour predictor's colouring graph)
Csr* block_graph_sym(const Csr* K, int bs, int64_t nn) {
  cudaStream_t s = 0;
  std::unique_ptr<Csr> G(block_graph(K, bs, nn, nullptr, nullptr, 0.0));
  note_launch();
  k_fill_ones<<<grid_for(G->nnz, 256), 256>>>(G->val, G->nnz);
  std::unique_ptr<Csr> GT(csr_transpose(G.get(), s));
  return csr_axpby(1.0, G.get(), 1.0, GT.get(), s);
}

// symmetrised node graph on the device (caller owns the result)
Csr* node_graph_dev(const Csr* K, const int64_t* dof_node_h, int64_t num_nodes, const int8_t* body_h, double eps) {
  cudaStream_t s = 0;
  const int64_t n = K->n_rows;
  int bs = (num_nodes > 0 && n % num_nodes == 0) ? (int)(n / num_nodes) : 0;
  if (bs < 1 || bs > 6) bs = 0;
  for (int64_t i = 0; bs && i < n; ++i)
    if (dof_node_h[i] != i / bs) bs = 0;
  if (bs) {
    DBuf<int8_t> bd(num_nodes + 1);
    CAMG_CUDA(cudaMemcpy(bd.p, body_h, num_nodes, cudaMemcpyHostToDevice));
    DBuf<double> diag(n + 1);
    if (eps > 0.0) {
      csr_diagonal(K, 0, diag.p, s);
      note_launch();
      k_absdiag<<<grid_for(n, 256), 256>>>(diag.p, n);
    }
    std::unique_ptr<Csr> G(block_graph(K, bs, num_nodes, bd.p, diag.p, eps));
    note_launch();
    k_fill_ones<<<grid_for(G->nnz, 256), 256>>>(G->val, G->nnz);
    std::unique_ptr<Csr> GT(csr_transpose(G.get(), s));
    return csr_axpby(1.0, G.get(), 1.0, GT.get(), s);
  }
  DBuf<int64_t> dn(n + 1);
  DBuf<int8_t> bd(num_nodes + 1);
  CAMG_CUDA(cudaMemcpy(dn.p, dof_node_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  CAMG_CUDA(cudaMemcpy(bd.p, body_h, num_nodes, cudaMemcpyHostToDevice));
  DBuf<double> diag(n + 1);
  if (eps > 0.0) {
    csr_diagonal(K, 0, diag.p, s);
    note_launch();
    k_absdiag<<<grid_for(n, 256), 256>>>(diag.p, n);
  }
  // F
  DBuf<int64_t> cnt(n + 1);
  note_launch();
  k_filter<false><<<grid_for(n, 256), 256>>>(view(K), dn.p, bd.p, diag.p, eps, cnt.p, nullptr, nullptr, nullptr);
  DBuf<int64_t> rp(n + 1);
  exclusive_scan_i64(cnt.p, rp.p, n, s);
  CAMG_CUDA(cudaDeviceSynchronize());
  const int64_t nnz = read_i64(rp.p + n);
  Csr F;
  F.n_rows = n; F.n_cols = n; F.nnz = nnz;
  F.rowptr = rp.release();
  F.col = dalloc<int32_t>(nnz);
  F.val = dalloc<double>(nnz);
  F.avg_row = n ? double(nnz) / n : 0.0;
  note_launch();
  k_filter<true><<<grid_for(n, 256), 256>>>(view(K), dn.p, bd.p, diag.p, eps, nullptr, F.rowptr, F.col, F.val);
  CAMG_LAUNCH_CHECK();
  // N (n x num_nodes) and N^T
  Csr N;
  N.n_rows = n; N.n_cols = num_nodes; N.nnz = n;
  N.rowptr = dalloc<int64_t>(n + 1);
  N.col = dalloc<int32_t>(n);
  N.val = dalloc<double>(n);
  N.avg_row = 1.0;
  note_launch();
  k_incidence<<<grid_for(n + 1, 256), 256>>>(dn.p, n, N.rowptr, N.col, N.val);
  CAMG_CUDA(cudaDeviceSynchronize());
  std::unique_ptr<Csr> NT(csr_transpose(&N, s));
  std::unique_ptr<Csr> G(galerkin(NT.get(), &F, &N, s));
  std::unique_ptr<Csr> GT(csr_transpose(G.get(), s));
  return csr_axpby(1.0, G.get(), 1.0, GT.get(), s);
}

// ---------------------------------------------------------------------------
// host aggregation

void greedy(int64_t n, const int64_t* ip, const int64_t* ix, int64_t min_size, int64_t* agg_out, int64_t* num_out,
            int64_t* roots_out, int64_t* singles_out) {
  const int64_t U = -1;
  std::vector<int64_t> agg(n, U), roots;
  // phase 1: root nodes whose neighbourhood is untouched
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] != U) continue;
    bool free_nb = true;
    for (int64_t p = ip[i]; p < ip[i + 1] && free_nb; ++p) free_nb = agg[ix[p]] == U;
    if (!free_nb) continue;
    const int64_t a = (int64_t)roots.size();
    agg[i] = a;
    for (int64_t p = ip[i]; p < ip[i + 1]; ++p) agg[ix[p]] = a;
    roots.push_back(i);
  }
  // phase 2: leftovers join the most-connected neighbouring aggregate (lowest id on ties)
  std::vector<int64_t> tally;
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] != U) continue;
    int64_t best = U, best_cnt = 0;
    tally.clear();
    for (int64_t p = ip[i]; p < ip[i + 1]; ++p)
      if (agg[ix[p]] != U) tally.push_back(agg[ix[p]]);
    if (tally.empty()) {
      agg[i] = (int64_t)roots.size();
      roots.push_back(i);
      continue;
    }
    std::sort(tally.begin(), tally.end());
    for (size_t a = 0; a < tally.size();) {
      size_t b = a;
      while (b < tally.size() && tally[b] == tally[a]) ++b;
      if ((int64_t)(b - a) > best_cnt) { best_cnt = (int64_t)(b - a); best = tally[a]; }
      a = b;
    }
    agg[i] = best;
  }
  const int64_t na = (int64_t)roots.size();
  std::vector<int64_t> size(na, 0);
  for (int64_t i = 0; i < n; ++i) size[agg[i]]++;
  // phase 3: merge undersized aggregates into their best-connected neighbour
  if (min_size > 1) {
    std::vector<std::vector<int64_t>> members(na);
    for (int64_t i = 0; i < n; ++i) members[agg[i]].push_back(i);
    std::map<int64_t, int64_t> conn;
    for (int64_t a = 0; a < na; ++a) {
      if (size[a] == 0 || size[a] >= min_size) continue;
      conn.clear();
      for (int64_t v : members[a])
        for (int64_t p = ip[v]; p < ip[v + 1]; ++p) {
          const int64_t t = agg[ix[p]];
          if (t != a) conn[t]++;
        }
      if (conn.empty()) continue;
      int64_t best = -1, bc = -1;
      for (auto& kv : conn)
        if (kv.second > bc) { bc = kv.second; best = kv.first; }  // ascending keys: first max = lowest id
      for (int64_t v : members[a]) agg[v] = best;
      members[best].insert(members[best].end(), members[a].begin(), members[a].end());
      size[best] += size[a];
      size[a] = 0;
      members[a].clear();
      members[a].shrink_to_fit();
    }
  }
  std::vector<int64_t> remap(na, U);
  int64_t m = 0;
  for (int64_t a = 0; a < na; ++a)
    if (size[a] > 0) { remap[a] = m; roots_out[m] = roots[a]; ++m; }
  std::vector<int64_t> sz(m, 0);
  for (int64_t i = 0; i < n; ++i) { agg_out[i] = remap[agg[i]]; sz[agg_out[i]]++; }
  int64_t singles = 0;
  for (int64_t a = 0; a < m; ++a) singles += sz[a] == 1;
  *num_out = m;
  *singles_out = singles;
}

}  // namespace camg

using namespace camg;

extern "C" {

int camg_node_graph(const camg_csr* K, const int64_t* dof_node, int64_t num_nodes, const int8_t* node_body,
                    double eps_drop, camg_csr** graph, int64_t* nnz) {
  return guarded([&] {
    CAMG_CHECK(K->m->n_rows == K->m->n_cols, CAMG_ERR_DIMENSION, "K must be square");
    for (int64_t i = 0; i < K->m->n_rows; ++i)
      CAMG_CHECK(dof_node[i] >= 0 && dof_node[i] < num_nodes, CAMG_ERR_DIMENSION, "dof->node map out of range");
    Csr* G = node_graph_dev(K->m, dof_node, num_nodes, node_body, eps_drop);
    *nnz = G->nnz;
    *graph = new camg_csr{G};
  });
}

int camg_pattern_to_host(const camg_csr* A, int64_t* indptr, int64_t* indices) {
  return guarded([&] {
    const Csr* M = A->m;
    CAMG_CUDA(cudaMemcpy(indptr, M->rowptr, sizeof(int64_t) * (M->n_rows + 1), cudaMemcpyDeviceToHost));
    if (!M->nnz) return;
    // int32 columns widened in chunks straight into the caller's buffer: two pinned staging buffers, the
    // copy of the next chunk in flight while host threads widen the current one (the C5 node graph has
    // 2e8 entries: 0.8 GB across PCIe, 1.6 GB of first-touched destination)
    const int64_t chunk = int64_t(1) << 24;
    const int64_t cap = std::min(M->nnz, chunk);
    int32_t* stage[2] = {nullptr, nullptr};
    cudaStream_t cs = nullptr;
    CAMG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CAMG_CUDA(cudaMallocHost(&stage[0], sizeof(int32_t) * cap));
    CAMG_CUDA(cudaMallocHost(&stage[1], sizeof(int32_t) * cap));
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = (int)std::max(1u, std::min(hw ? hw : 1u, 8u));
    auto widen = [&](const int32_t* src, int64_t o, int64_t m) {
      std::vector<std::thread> th;
      const int64_t per = (m + nt - 1) / nt;
      for (int t = 0; t < nt; ++t) {
        const int64_t a = t * per, b = std::min(m, a + per);
        if (a >= b) break;
        th.emplace_back([=] { for (int64_t i = a; i < b; ++i) indices[o + i] = src[i]; });
      }
      for (auto& x : th) x.join();
    };
    int cur = 0;
    CAMG_CUDA(cudaMemcpyAsync(stage[0], M->col, sizeof(int32_t) * std::min(chunk, M->nnz), cudaMemcpyDeviceToHost, cs));
    for (int64_t o = 0; o < M->nnz; o += chunk) {
      const int64_t m = std::min(chunk, M->nnz - o);
      CAMG_CUDA(cudaStreamSynchronize(cs));
      const int64_t o2 = o + chunk;
      if (o2 < M->nnz)
        CAMG_CUDA(cudaMemcpyAsync(stage[cur ^ 1], M->col + o2, sizeof(int32_t) * std::min(chunk, M->nnz - o2),
                                  cudaMemcpyDeviceToHost, cs));
      widen(stage[cur], o, m);
      cur ^= 1;
    }
    cudaStreamSynchronize(cs);
    cudaFreeHost(stage[0]);
    cudaFreeHost(stage[1]);
    cudaStreamDestroy(cs);
  });
}

int camg_aggregate_greedy(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t min_size,
                          int64_t* node_to_agg, int64_t* num_aggs, int64_t* roots, int64_t* singletons) {
  return guarded([&] {
    CAMG_CHECK(min_size >= 1, CAMG_ERR_ARG, "min_agg_size must be >= 1");
    greedy(n, indptr, indices, min_size, node_to_agg, num_aggs, roots, singletons);
  });
}

int camg_aggregate_lagrange(const int64_t* disp, int64_t n_rows, const int64_t* drp, const int64_t* dcol,
                            const double* dval, const int64_t* slave_dofs, const int64_t* row_node,
                            const int64_t* lm_node_of_lm_dof, int64_t n_lm_dofs, int64_t* lam, int64_t* num_aggs,
                            int64_t* roots, int64_t* overlaps) {
  return guarded([&] {
    int64_t n_lm = 0;
    for (int64_t i = 0; i < n_lm_dofs; ++i) n_lm = std::max(n_lm, lm_node_of_lm_dof[i] + 1);
    for (int64_t i = 0; i < n_lm; ++i) lam[i] = -1;
    std::vector<int64_t> order(n_rows);
    for (int64_t r = 0; r < n_rows; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return slave_dofs[a] < slave_dofs[b]; });
    std::unordered_map<int64_t, int64_t> owner;
    int64_t nroots = 0, ov = 0;
    for (int64_t r : order) {
      const int64_t k = disp[row_node[r]];
      CAMG_CHECK(k >= 0, CAMG_ERR_SETUP, "slave DOF " + std::to_string(slave_dofs[r]) + ": node is unaggregated");
      for (int64_t p = drp[r]; p < drp[r + 1]; ++p) {
        if (dval[p] == 0.0) continue;
        const int64_t pn = lm_node_of_lm_dof[dcol[p]];
        auto it = owner.find(k);
        if (lam[pn] == -1) {
          int64_t tgt;
          if (it == owner.end()) {
            tgt = nroots;
            owner[k] = tgt;
            roots[nroots++] = pn;
          } else {
            tgt = it->second;
          }
          lam[pn] = tgt;
        } else if (it == owner.end() || lam[pn] != it->second) {
          ++ov;
        }
      }
    }
    *num_aggs = nroots;
    *overlaps = ov;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// tentative prolongator assembly (transfer.py:86-145): the per-aggregate Q
// factors come from host LAPACK (batched, grouped by aggregate size); the
// device scatters them into canonical CSR (row = DOF, columns col0(agg)+c,
// c < rank, |q| >= 1e-300 kept as from_scipy does).

namespace camg {

struct PtGroup {
  int64_t G, M, kk, dof_off, q_off, agg_off;
};

template <bool FILL>
__global__ void k_ptent(PtGroup gp, const int64_t* __restrict__ dofs, const double* __restrict__ Q,
                        const int64_t* __restrict__ rank, const int64_t* __restrict__ col0, int64_t* __restrict__ cnt,
                        const int64_t* __restrict__ rp, int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t rows = gp.G * gp.M;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / gp.M;
    const int64_t dof = dofs[gp.dof_off + t];
    const int64_t r = rank[gp.agg_off + g];
    const double* q = Q + gp.q_off + t * gp.kk;
    int64_t n = 0, o = FILL ? rp[dof] : 0;
    for (int64_t c = 0; c < r; ++c) {
      const double v = q[c];
      if (fabs(v) >= kDropTol) {
        if (FILL) { col[o + n] = (int32_t)(col0[gp.agg_off + g] + c); val[o + n] = v; }
        ++n;
      }
    }
    if (!FILL) cnt[dof] = n;
  }
}

// device CSR of P_tent from the per-group QR factors already on the device
// (d_rank, d_col0 in group order)
Csr* tentative_assemble_dev(int64_t n_dofs, int64_t ncoarse, int64_t ngroups, const int64_t* meta,
                            const int64_t* d_dofs, const double* d_q, const int64_t* d_rank, const int64_t* d_col0) {
  cudaStream_t s = 0;
  DBuf<int64_t> cnt(n_dofs + 1);
  CAMG_CUDA(cudaMemset(cnt.p, 0, sizeof(int64_t) * (n_dofs + 1)));
  for (int64_t gi = 0; gi < ngroups; ++gi) {
    const int64_t* m = meta + 6 * gi;
    PtGroup gp{m[0], m[1], m[2], m[3], m[4], m[5]};
    note_launch();
    k_ptent<false><<<grid_for(gp.G * gp.M, 256), 256, 0, s>>>(gp, d_dofs, d_q, d_rank, d_col0, cnt.p, nullptr, nullptr,
                                                               nullptr);
  }
  DBuf<int64_t> rp(n_dofs + 1);
  exclusive_scan_i64(cnt.p, rp.p, n_dofs, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  const int64_t nnz = read_i64(rp.p + n_dofs);
  Csr* P = new Csr();
  P->n_rows = n_dofs; P->n_cols = ncoarse; P->nnz = nnz;
  P->rowptr = rp.release();
  P->col = dalloc<int32_t>(nnz);
  P->val = dalloc<double>(nnz);
  P->avg_row = n_dofs ? double(nnz) / n_dofs : 0.0;
  for (int64_t gi = 0; gi < ngroups; ++gi) {
    const int64_t* m = meta + 6 * gi;
    PtGroup gp{m[0], m[1], m[2], m[3], m[4], m[5]};
    note_launch();
    k_ptent<true><<<grid_for(gp.G * gp.M, 256), 256, 0, s>>>(gp, d_dofs, d_q, d_rank, d_col0, nullptr, P->rowptr, P->col,
                                                              P->val);
  }
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  return P;
}

// device CSR of P_tent from host QR factors (see camg_tentative_csr)
Csr* tentative_assemble(int64_t n_dofs, int64_t ncoarse, int64_t ngroups, const int64_t* meta, const int64_t* dofs,
                        int64_t ndofs_total, const double* Q, int64_t nq, const int64_t* rank, const int64_t* col0,
                        int64_t naggs) {
  CAMG_CHECK(ndofs_total == n_dofs, CAMG_ERR_DIMENSION, "every DOF must belong to one aggregate");
  DBuf<int64_t> d_dofs(ndofs_total + 1), d_rank(naggs + 1), d_col0(naggs + 1);
  DBuf<double> d_q(nq + 1);
  CAMG_CUDA(cudaMemcpy(d_dofs.p, dofs, sizeof(int64_t) * ndofs_total, cudaMemcpyHostToDevice));
  CAMG_CUDA(cudaMemcpy(d_q.p, Q, sizeof(double) * nq, cudaMemcpyHostToDevice));
  CAMG_CUDA(cudaMemcpy(d_rank.p, rank, sizeof(int64_t) * naggs, cudaMemcpyHostToDevice));
  CAMG_CUDA(cudaMemcpy(d_col0.p, col0, sizeof(int64_t) * naggs, cudaMemcpyHostToDevice));
  return tentative_assemble_dev(n_dofs, ncoarse, ngroups, meta, d_dofs.p, d_q.p, d_rank.p, d_col0.p);
}

}  // namespace camg

extern "C" int camg_tentative_csr(int64_t n_dofs, int64_t ncoarse, int64_t ngroups, const int64_t* meta,
                                  const int64_t* dofs, int64_t ndofs_total, const double* Q, int64_t nq,
                                  const int64_t* rank, const int64_t* col0, int64_t naggs, camg_csr** out) {
  return guarded([&] {
    *out = new camg_csr{tentative_assemble(n_dofs, ncoarse, ngroups, meta, dofs, ndofs_total, Q, nq, rank, col0,
                                           naggs)};
  });
}

// Two-pass (count, then fill) row-wise SpGEMM and the fused Galerkin triple
// product, reproducing scipy's csr_matmat accumulation order so that the
// exact-zero cancellations -- and therefore the coarse sparsity patterns the
// host aggregation reads -- are bit-identical to the reference
// (sparse.py:161-173, transfer.py:164-199, smoothers.py:220-239).
//
// scipy csr_matmat, row i:  sums[k] = 0 + v_1*b_1k + v_2*b_2k + ...  in the
// order of A's stored row; output order = reverse first touch; exact zeros
// dropped.  `(R@A)@P` therefore accumulates each coarse entry over the RA row
// in reverse-first-touch order.  The fused kernel recovers that order without
// materialising or sorting RA: RA column t belongs to "touch group" q (the
// position in R's row of the first A row containing t); walking q downwards
// and each A row backwards, and keeping only t whose group is q, enumerates
// exactly scipy's RA row order.
//
// One warp per output row; per-warp hash tables live in shared memory, rows
// that overflow them are recomputed with hash tables in global scratch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace camg {

namespace {

constexpr int32_t kEmpty = -1;
constexpr int kWarpsPerBlock = 2;
#ifndef CAMG_TRIPLE_MINB
#define CAMG_TRIPLE_MINB 12  // resident 64-thread CTAs per SM the Galerkin kernel is compiled for
#endif  // smem hash per warp: 2-warp blocks pack 3+ blocks per SM

__device__ __forceinline__ uint32_t hslot(int32_t k, uint32_t mask) {
  return ((uint32_t)k * 2654435761u) & mask;
}

// Hash table view (shared or global memory).
struct Hash {
  int32_t* keys;
  int16_t* ft;  // first-touch group (may be null); R rows are < 32768 long (checked)
  double* vals;
  uint32_t cap;  // power of two
};

// Accumulate (k, prod) for one lane; returns 1 if a new key was inserted.
__device__ __forceinline__ int hash_add(Hash h, int32_t k, double prod, int32_t group) {
  const uint32_t mask = h.cap - 1;
  uint32_t s = hslot(k, mask);
  while (true) {
    int32_t cur = atomicCAS(&h.keys[s], kEmpty, k);
    if (cur == kEmpty) {
      h.vals[s] = __dadd_rn(0.0, prod);
      if (h.ft) h.ft[s] = (int16_t)group;
      return 1;
    }
    if (cur == k) {
      h.vals[s] = __dadd_rn(h.vals[s], prod);
      return 0;
    }
    s = (s + 1) & mask;
  }
}

__device__ __forceinline__ int hash_find(const Hash& h, int32_t k) {
  const uint32_t mask = h.cap - 1;
  uint32_t s = hslot(k, mask);
  while (true) {
    int32_t cur = h.keys[s];
    if (cur == k) return (int)s;
    if (cur == kEmpty) return -1;
    s = (s + 1) & mask;
  }
}

__device__ __forceinline__ void hash_clear(Hash h, int lane) {
  for (uint32_t s = lane; s < h.cap; s += 32) h.keys[s] = kEmpty;
  __syncwarp();
}

// Compact entries with |v| >= tol (tol = 0 -> v != 0) to the front of the
// table arrays, bitonic-sort them by key, return the count.
__device__ int compact_sort(Hash h, int lane, double tol) {
  int n = 0;
  for (uint32_t base = 0; base < h.cap; base += 32) {
    const uint32_t s = base + lane;
    int32_t k = h.keys[s];
    double v = h.vals[s];
    bool keep = (k != kEmpty) && (tol > 0.0 ? fabs(v) >= tol : v != 0.0);
    unsigned b = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      int pos = n + __popc(b & ((1u << lane) - 1u));
      h.keys[pos] = k;
      h.vals[pos] = v;
    }
    n += __popc(b);
    __syncwarp();
  }
  int N = 1;
  while (N < n) N <<= 1;
  for (int s = n + lane; s < N; s += 32) h.keys[s] = INT32_MAX;
  __syncwarp();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < N; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          int32_t a = h.keys[i], b = h.keys[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            h.keys[i] = b;
            h.keys[ixj] = a;
            double t = h.vals[i];
            h.vals[i] = h.vals[ixj];
            h.vals[ixj] = t;
          }
        }
      }
      __syncwarp();
    }
  }
  return n;
}

__device__ int count_kept(const Hash& h, int lane, double tol) {
  int n = 0;
  for (uint32_t s = lane; s < h.cap; s += 32) {
    int32_t k = h.keys[s];
    if (k != kEmpty && (tol > 0.0 ? fabs(h.vals[s]) >= tol : h.vals[s] != 0.0)) ++n;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  return n;
}

// ---------------------------------------------------------------------------
// C = A*B for one row: returns false on overflow

__device__ bool row_product(const CsrView& A, const CsrView& B, int64_t row, bool reverse_a,
                            const double* __restrict__ scale_a, Hash h,
                            int lane, uint32_t limit) {
  hash_clear(h, lane);
  const int64_t s = A.rowptr[row], e = A.rowptr[row + 1];
  uint32_t count = 0;
  for (int64_t q = 0; q < e - s; ++q) {
    const int64_t jj = reverse_a ? (e - 1 - q) : (s + q);
    const int32_t j = A.col[jj];
    double v = A.val[jj];
    if (scale_a) {  // (diag(s) A)_ij exactly as scipy's A.multiply(s[:,None]); canon drops |v| < 1e-300
      v = __dmul_rn(v, scale_a[row]);
      if (fabs(v) < kDropTol) continue;
    }
    const int64_t bs = B.rowptr[j], be = B.rowptr[j + 1];
    for (int64_t base = bs; base < be; base += 32) {
      if (count + 32 > limit) return false;
      int ins = 0;
      const int64_t kk = base + lane;
      if (kk < be) ins = hash_add(h, B.col[kk], __dmul_rn(v, B.val[kk]), 0);
      count += __popc(__ballot_sync(0xffffffffu, ins));
      __syncwarp();
    }
  }
  return true;
}

// Same product with the row's products flattened into 32-wide chunks (for
// short B rows, where one A entry per warp step would idle most lanes).
// Order is kept exactly: lanes holding the same key in a chunk form a
// __match_any group whose lowest lane adds the members' products in lane
// order (= A-row order), i.e. sums[k] = ((sums[k] + p1) + p2) + ... as in
// csr_matmat.  `sp` is 32 doubles of per-warp scratch.
__device__ bool row_product_flat(const CsrView& A, const CsrView& B, int64_t row, bool reverse_a,
                                 const double* __restrict__ scale_a, Hash h, int lane, uint32_t limit,
                                 double* sp) {
  hash_clear(h, lane);
  const int64_t s = A.rowptr[row], e = A.rowptr[row + 1];
  const int64_t L = e - s;
  uint32_t count = 0;
  for (int64_t w0 = 0; w0 < L; w0 += 32) {
    // window of up to 32 A entries: lane t owns A entry w0 + t
    const int64_t q = w0 + lane;
    int32_t j = 0;
    double v = 0.0;
    int64_t blen = 0, bstart = 0;
    if (q < L) {
      const int64_t jj = reverse_a ? (e - 1 - q) : (s + q);
      j = A.col[jj];
      v = A.val[jj];
      if (scale_a) {
        v = __dmul_rn(v, scale_a[row]);
        if (fabs(v) < kDropTol) v = 0.0, j = -1;  // dropped entry of diag(s)A
      }
      if (j >= 0) {
        bstart = B.rowptr[j];
        blen = B.rowptr[j + 1] - bstart;
      }
    }
    // inclusive scan of the window's product counts
    int64_t incl = blen;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (int64_t f0 = 0; f0 < total; f0 += 32) {
      if (count + 32 > limit) return false;
      const int64_t f = f0 + lane;
      const bool act = f < total;
      // owner lane of product f: first t with incl[t] > f (binary search over shuffles)
      int lo = 0;
#pragma unroll
      for (int stepw = 16; stepw > 0; stepw >>= 1) {
        const int64_t c = __shfl_sync(0xffffffffu, incl, lo + stepw - 1);
        if (act && c <= f) lo += stepw;
      }
      const int owner = act ? lo : 0;
      const int64_t before = __shfl_sync(0xffffffffu, incl - blen, owner);
      const int64_t ob = __shfl_sync(0xffffffffu, bstart, owner);
      const double ov = __shfl_sync(0xffffffffu, v, owner);
      int32_t key = -1;
      double prod = 0.0;
      if (act) {
        const int64_t kk = ob + (f - before);
        key = B.col[kk];
        prod = __dmul_rn(ov, B.val[kk]);
      }
      sp[lane] = prod;
      const unsigned am = __ballot_sync(0xffffffffu, act);
      const unsigned grp = __match_any_sync(0xffffffffu, act ? key : -1 - lane);
      __syncwarp();
      int ins = 0;
      if (act && (__ffs(grp) - 1) == lane) {  // group leader
        const uint32_t mask = h.cap - 1;
        uint32_t slot = hslot(key, mask);
        double acc;
        while (true) {
          const int32_t cur = atomicCAS(&h.keys[slot], kEmpty, key);
          if (cur == kEmpty) { acc = 0.0; ins = 1; break; }
          if (cur == key) { acc = h.vals[slot]; break; }
          slot = (slot + 1) & mask;
        }
        unsigned m = grp & am;
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          acc = __dadd_rn(acc, sp[src]);
        }
        h.vals[slot] = acc;
      }
      count += __popc(__ballot_sync(0xffffffffu, ins));
      __syncwarp();
    }
  }
  return true;
}

// (R*A)*P for one row: hash1 holds RA with first-touch groups, hash2 the result
// ordered accumulation of one 32-wide chunk of (key, product) pairs into h:
// lanes with equal keys form a __match_any group, the lowest lane adds the
// members' products in lane order.  `ft` is recorded for new keys.
__device__ __forceinline__ int chunk_accumulate(Hash h, bool act, int32_t key, double prod, int32_t ft, int lane,
                                                double* sp) {
  sp[lane] = prod;
  const unsigned am = __ballot_sync(0xffffffffu, act);
  const unsigned grp = __match_any_sync(0xffffffffu, act ? key : -1 - lane);
  __syncwarp();
  int ins = 0;
  if (act && (__ffs(grp) - 1) == lane) {
    const uint32_t mask = h.cap - 1;
    uint32_t slot = hslot(key, mask);
    double acc;
    while (true) {
      const int32_t cur = atomicCAS(&h.keys[slot], kEmpty, key);
      if (cur == kEmpty) {
        acc = 0.0;
        ins = 1;
        if (h.ft) h.ft[slot] = (int16_t)ft;
        break;
      }
      if (cur == key) { acc = h.vals[slot]; break; }
      slot = (slot + 1) & mask;
    }
    unsigned m = grp & am;
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      acc = __dadd_rn(acc, sp[src]);
    }
    h.vals[slot] = acc;
  }
  const int n = __popc(__ballot_sync(0xffffffffu, ins));
  __syncwarp();
  return n;
}

// lane index owning flattened position f (first t with incl[t] > f)
__device__ __forceinline__ int owner_of(int64_t incl, int64_t f, bool act) {
  int lo = 0;
#pragma unroll
  for (int w = 16; w > 0; w >>= 1) {
    const int64_t c = __shfl_sync(0xffffffffu, incl, lo + w - 1);
    if (act && c <= f) lo += w;
  }
  return act ? lo : 0;
}

// (R*A)*P for one row: hash1 holds RA with first-touch groups, hash2 the result
__device__ bool row_triple(const CsrView& R, const CsrView& A, const CsrView& P, int64_t row, Hash h1,
                           Hash h2, int lane, uint32_t limit1, uint32_t limit2, double* sp, int32_t* bk,
                           double* bv, bool sorted_ra) {
  hash_clear(h1, lane);
  hash_clear(h2, lane);
  const int64_t rs = R.rowptr[row], re = R.rowptr[row + 1];
  const int64_t nR = re - rs;
  if (nR > 32767) return false;  // first-touch groups are 16-bit (never retried to success)
  uint32_t c1 = 0, c2 = 0;
  // ---- stage 1: RA row in R's order, one A-row chunk per step, next chunk prefetched
  for (int64_t w0 = 0; w0 < nR; w0 += 32) {
    const int64_t qq = w0 + lane;
    double vq = 0.0;
    int64_t aq = 0, lq = 0;
    if (qq < nR) {
      const int32_t j = R.col[rs + qq];
      vq = R.val[rs + qq];
      aq = A.rowptr[j];
      lq = A.rowptr[j + 1] - aq;
    }
    const int64_t nch = (lq + 31) >> 5;
    int64_t incl = nch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t T = __shfl_sync(0xffffffffu, incl, 31);
    auto fetch = [&](int64_t st, int32_t& col, double& val, double& vv, int& ql, bool& ok) {
      const bool act = st < T;
      const int o = owner_of(incl, st, act);
      const int64_t c = st - (__shfl_sync(0xffffffffu, incl - nch, o));
      const int64_t a = __shfl_sync(0xffffffffu, aq, o);
      const int64_t l = __shfl_sync(0xffffffffu, lq, o);
      vv = __shfl_sync(0xffffffffu, vq, o);
      ql = o;
      const int64_t off = 32 * c + lane;
      ok = act && off < l;
      col = ok ? A.col[a + off] : -1;
      val = ok ? A.val[a + off] : 0.0;
    };
    int32_t col, ncol;
    double val, vv, nval, nvv;
    int ql, nql;
    bool ok, nok;
    if (T > 0) fetch(0, col, val, vv, ql, ok);
    for (int64_t st = 0; st < T; ++st) {
      if (st + 1 < T) fetch(st + 1, ncol, nval, nvv, nql, nok);
      if (c1 + 32 > limit1) return false;
      int ins = 0;
      if (ok) ins = hash_add(h1, col, __dmul_rn(vv, val), (int32_t)(w0 + ql));
      c1 += __popc(__ballot_sync(0xffffffffu, ins));
      __syncwarp();
      col = ncol; val = nval; vv = nvv; ql = nql; ok = nok;
    }
  }
  // ---- stage 2: RA in scipy's stored order = descending (first-touch group,
  // column) -- csr_matmat's reverse first-touch linked list, exact zeros
  // dropped -- times the P rows, as ordered 32-wide chunks into h2.
  // expand(cnt): the first cnt (<= 32) RA entries (bk, bv) in order
  auto expand = [&](int cnt) -> bool {
    const int e = lane;
    double rav = 0.0;
    int64_t pb = 0, pl = 0;
    if (e < cnt) {
      const int32_t t = bk[e];
      rav = bv[e];
      pb = P.rowptr[t];
      pl = P.rowptr[t + 1] - pb;
    }
    int64_t incl = pl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t T = __shfl_sync(0xffffffffu, incl, 31);
    for (int64_t f0 = 0; f0 < T; f0 += 32) {
      if (c2 + 32 > limit2) return false;
      const int64_t f = f0 + lane;
      const bool act = f < T;
      const int o = owner_of(incl, f, act);
      const int64_t before = __shfl_sync(0xffffffffu, incl - pl, o);
      const int64_t ob = __shfl_sync(0xffffffffu, pb, o);
      const double ov = __shfl_sync(0xffffffffu, rav, o);
      int32_t key = -1;
      double prod = 0.0;
      if (act) {
        const int64_t pp = ob + (f - before);
        key = P.col[pp];
        prod = __dmul_rn(ov, P.val[pp]);
      }
      c2 += chunk_accumulate(h2, act, key, prod, 0, lane, sp);
    }
    return true;
  };
  if (!sorted_ra) {
    // Sort-free enumeration of that order: walk R's row backwards (groups
    // of 32 entries, then A-row chunks from the last) and each 32-entry
    // chunk of an A row from its end, lane 0 on the highest column; a
    // column is emitted at the A row of its first touch (h1.ft == q), so
    // every RA entry appears once, in descending (group, column) order.
    // Emitted entries queue in (bk, bv) and expand 32 at a time.
    int nb = 0;
    const int64_t last0 = ((nR - 1) / 32) * 32;
    for (int64_t w0 = last0; w0 >= 0; w0 -= 32) {
      const int64_t qq = w0 + lane;
      int64_t aq = 0, lq = 0;
      if (qq < nR) {
        const int32_t j = R.col[rs + qq];
        aq = A.rowptr[j];
        lq = A.rowptr[j + 1] - aq;
      }
      const int64_t nch = (lq + 31) >> 5;
      int64_t incl = nch;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int64_t T = __shfl_sync(0xffffffffu, incl, 31);
      // column of this lane at step st (-1: none) and the step's A row q;
      // the next step's column load is issued before this step's lookups
      auto col_at = [&](int64_t st, int& q) -> int32_t {
        const int o = owner_of(incl, st, true);
        const int64_t c = st - (__shfl_sync(0xffffffffu, incl - nch, o));
        const int64_t a = __shfl_sync(0xffffffffu, aq, o);
        const int64_t l = __shfl_sync(0xffffffffu, lq, o);
        const int64_t off = 32 * c + 31 - lane;
        q = (int)(w0 + o);
        return (off >= 0 && off < l) ? A.col[a + off] : -1;
      };
      int qn = 0;
      int32_t tn = T > 0 ? col_at(T - 1, qn) : -1;
      for (int64_t st = T - 1; st >= 0; --st) {
        const int32_t t = tn;
        const int q = qn;
        if (st > 0) tn = col_at(st - 1, qn);
        bool emit = false;
        double v = 0.0;
        if (t >= 0) {
          const int sl = hash_find(h1, t);
          if (sl >= 0 && h1.ft[sl] == (int16_t)q) {
            v = h1.vals[sl];
            emit = v != 0.0;
          }
        }
        const unsigned em = __ballot_sync(0xffffffffu, emit);
        if (emit) {
          const int pos = nb + __popc(em & ((1u << lane) - 1u));
          bk[pos] = t;
          bv[pos] = v;
        }
        nb += __popc(em);
        __syncwarp();
        if (nb >= 32) {
          if (!expand(32)) return false;
          __syncwarp();
          if (lane < nb - 32) {
            bk[lane] = bk[32 + lane];
            bv[lane] = bv[32 + lane];
          }
          nb -= 32;
          __syncwarp();
        }
      }
    }
    if (nb > 0 && !expand(nb)) return false;
    return true;
  }
  // (CAMG_RAP_SORT=1) compact the table, bitonic-sort it by that key, then
  // expand it in chunks of 32
  int n1 = 0;
  for (uint32_t base = 0; base < h1.cap; base += 32) {
    const uint32_t sl = base + lane;
    const int32_t k = h1.keys[sl];
    const double v = h1.vals[sl];
    const int16_t g = h1.ft[sl];
    const bool keep = (k != kEmpty) && v != 0.0;
    const unsigned bb = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      const int pos = n1 + __popc(bb & ((1u << lane) - 1u));
      h1.keys[pos] = k;
      h1.vals[pos] = v;
      h1.ft[pos] = g;
    }
    n1 += __popc(bb);
    __syncwarp();
  }
  int N = 1;
  while (N < n1) N <<= 1;
  for (int i = n1 + lane; i < N; i += 32) { h1.keys[i] = INT32_MIN; h1.ft[i] = -1; }
  __syncwarp();
  for (int k = 2; k <= N; k <<= 1) {
    for (int jb = k >> 1; jb > 0; jb >>= 1) {
      for (int i = lane; i < N; i += 32) {
        const int ixj = i ^ jb;
        if (ixj > i) {
          const int64_t ka = ((int64_t)h1.ft[i] << 32) | (uint32_t)(h1.keys[i] - INT32_MIN);
          const int64_t kb = ((int64_t)h1.ft[ixj] << 32) | (uint32_t)(h1.keys[ixj] - INT32_MIN);
          const bool desc = (i & k) == 0;
          if ((ka < kb) == desc) {
            int32_t tk = h1.keys[i]; h1.keys[i] = h1.keys[ixj]; h1.keys[ixj] = tk;
            int16_t tg = h1.ft[i]; h1.ft[i] = h1.ft[ixj]; h1.ft[ixj] = tg;
            double tv = h1.vals[i]; h1.vals[i] = h1.vals[ixj]; h1.vals[ixj] = tv;
          }
        }
      }
      __syncwarp();
    }
  }
  for (int e0 = 0; e0 < n1; e0 += 32) {
    const int cnt = min(32, n1 - e0);
    __syncwarp();
    if (lane < cnt) {
      bk[lane] = h1.keys[e0 + lane];
      bv[lane] = h1.vals[e0 + lane];
    }
    __syncwarp();
    if (!expand(cnt)) return false;
  }
  return true;
}

// ---------------------------------------------------------------------------
// kernels

struct OutArgs {
  int64_t* cnt;           // count pass
  const int64_t* rowptr;  // fill pass
  int32_t* col;
  double* val;
  int32_t* overflow;      // per row flag (count pass)
  double tol;
  // staging (count pass): a counted row is also stored, final order, at
  // soff[row] in (scol, sval) while the buffer lasts, so the fill pass
  // copies it instead of recomputing it; soff[row] = -1: recompute
  int32_t* scol = nullptr;
  double* sval = nullptr;
  int64_t* soff = nullptr;
  unsigned long long* stop = nullptr;
  int64_t scap = 0;
  bool rap_sort = false;  // k_triple: RA order by compaction + bitonic sort (CAMG_RAP_SORT=1)
  bool h2_smem = false;   // k_triple global tables: h2 in dynamic shared memory
};

template <bool FILL>
__device__ void emit(Hash h, int64_t row, int lane, const OutArgs& o) {
  if (!FILL && o.scol) {
    const int n = compact_sort(h, lane, o.tol);
    long long off = -1;
    if (lane == 0) {
      const unsigned long long t = atomicAdd(o.stop, (unsigned long long)n);
      off = (t + (unsigned long long)n <= (unsigned long long)o.scap) ? (long long)t : -1;
      o.cnt[row] = n;
      o.soff[row] = off;
    }
    off = __shfl_sync(0xffffffffu, off, 0);
    if (off >= 0)
      for (int i = lane; i < n; i += 32) {
        o.scol[off + i] = h.keys[i];
        o.sval[off + i] = h.vals[i];
      }
  } else if (!FILL) {
    int n = count_kept(h, lane, o.tol);
    if (lane == 0) o.cnt[row] = n;
  } else {
    int n = compact_sort(h, lane, o.tol);
    const int64_t base = o.rowptr[row];
    for (int i = lane; i < n; i += 32) {
      o.col[base + i] = h.keys[i];
      o.val[base + i] = h.vals[i];
    }
  }
}

template <bool FILL, bool GLOBAL>
__global__ void k_product(CsrView A, CsrView B, bool reverse_a, const double* __restrict__ scale_a,
                          const int64_t* __restrict__ rows, int64_t nrows,
                          uint32_t cap, char* __restrict__ gscratch, OutArgs o) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double sp_all[kWarpsPerBlock][32];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + w;
  const int64_t nw = (int64_t)gridDim.x * kWarpsPerBlock;
  char* base = GLOBAL ? gscratch + gw * (size_t)cap * 12 : smem + (size_t)w * cap * 12;
  Hash h{reinterpret_cast<int32_t*>(base + (size_t)cap * 8), nullptr, reinterpret_cast<double*>(base), cap};
  for (int64_t r = gw; r < nrows; r += nw) {
    const int64_t row = rows ? rows[r] : r;
    if (FILL && o.soff && o.soff[row] >= 0) continue;  // copied from the staging buffer
    bool ok = row_product_flat(A, B, row, reverse_a, scale_a, h, lane, (cap * 3) / 4, sp_all[w]);
    if (!ok) {
      if (!FILL && lane == 0) { o.overflow[row] = 1; o.cnt[row] = 0; }
      continue;
    }
    emit<FILL>(h, row, lane, o);
  }
}

template <bool FILL, bool GLOBAL>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, CAMG_TRIPLE_MINB) k_triple(CsrView R, CsrView A, CsrView P,
                                                                           const int64_t* __restrict__ rows, int64_t nrows,
                         uint32_t cap1, uint32_t cap2, char* __restrict__ gscratch, OutArgs o) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double sp_all[kWarpsPerBlock][32];
  __shared__ int32_t bk_all[kWarpsPerBlock][64];
  __shared__ double bv_all[kWarpsPerBlock][64];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + w;
  const int64_t nw = (int64_t)gridDim.x * kWarpsPerBlock;
  // per warp: vals f64 | keys i32 | ft i16 (14 B/slot) then vals f64 | keys i32 (12 B/slot)
  const size_t per = (size_t)cap1 * 14 + (size_t)cap2 * 12;
  char* base = GLOBAL ? gscratch + gw * per : smem + (size_t)w * per;
  Hash h1{reinterpret_cast<int32_t*>(base + (size_t)cap1 * 8), reinterpret_cast<int16_t*>(base + (size_t)cap1 * 12),
          reinterpret_cast<double*>(base), cap1};
  // global tables: the output table h2 (hit by every product) in shared
  // memory when the launch provides it (dynamic shared memory > 0)
  char* b2 = (GLOBAL && o.h2_smem) ? smem + (size_t)w * cap2 * 12 : base + (size_t)cap1 * 14;
  Hash h2{reinterpret_cast<int32_t*>(b2 + (size_t)cap2 * 8), nullptr, reinterpret_cast<double*>(b2), cap2};
  for (int64_t r = gw; r < nrows; r += nw) {
    const int64_t row = rows ? rows[r] : r;
    if (FILL && o.soff && o.soff[row] >= 0) continue;  // copied from the staging buffer
    bool ok = row_triple(R, A, P, row, h1, h2, lane, (cap1 * 3) / 4, (cap2 * 3) / 4, sp_all[w], bk_all[w], bv_all[w],
                         o.rap_sort);
    if (!ok) {
      if (!FILL && lane == 0) { o.overflow[row] = 1; o.cnt[row] = 0; }
      continue;
    }
    emit<FILL>(h2, row, lane, o);
  }
}

// fill the staged rows: warp per row, copy from the staging buffer
__global__ void k_copy_staged(int64_t n_rows, const int64_t* __restrict__ soff, const int64_t* __restrict__ rowptr,
                              const int32_t* __restrict__ scol, const double* __restrict__ sval,
                              int32_t* __restrict__ col, double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n_rows; row += nw) {
    const int64_t off = soff[row];
    if (off < 0) continue;
    const int64_t b = rowptr[row], n = rowptr[row + 1] - b;
    for (int64_t i = lane; i < n; i += 32) {
      col[b + i] = scol[off + i];
      val[b + i] = sval[off + i];
    }
  }
}

// upper bounds of products per row (for sizing the global fallback)
__global__ void k_row_products(CsrView A, CsrView B, int64_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = 0;
    for (int64_t p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) {
      int32_t j = A.col[p];
      t += B.rowptr[j + 1] - B.rowptr[j];
    }
    out[r] = t;
  }
}

uint32_t pow2_at_least(int64_t n) {
  uint32_t c = 64;
  while ((int64_t)c < n && c < (1u << 30)) c <<= 1;
  return c;
}

std::vector<int64_t> overflow_rows(const int32_t* dflag, int64_t n) {
  std::vector<int32_t> f(n);
  if (n) CAMG_CUDA(cudaMemcpy(f.data(), dflag, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  std::vector<int64_t> rows;
  for (int64_t i = 0; i < n; ++i)
    if (f[i]) rows.push_back(i);
  return rows;
}

// Driver shared by the product and the triple:
// `launch(fill, global, rows, nrows, cap1, cap2, scratch, out)`.
// Rows whose hash tables overflow shared memory are retried from global
// scratch with doubling table sizes until every row fits; each row is
// filled with the table size its count pass succeeded with.
template <class Launch>
Csr* two_pass(int64_t n_rows, int64_t n_cols, Launch launch, uint32_t c1_0, uint32_t c2_0, double tol,
              cudaStream_t s, int64_t est_nnz, bool start_global = false) {
  DBuf<int64_t> cnt(n_rows + 1);
  DBuf<int32_t> ovf(n_rows + 1);
  CAMG_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int32_t) * (n_rows + 1), s));
  OutArgs o{cnt.p, nullptr, nullptr, nullptr, ovf.p, tol};
  static const bool rap_sort = getenv("CAMG_RAP_SORT") && getenv("CAMG_RAP_SORT")[0] == '1';
  o.rap_sort = rap_sort;
  // staging buffer: the caller's output estimate, at most 40% of the free
  // memory and 16 GB; rows past it are recomputed by the fill pass
  // (CAMG_SPGEMM_STAGE=0 disables)
  DBuf<int32_t> scol;
  DBuf<double> sval;
  DBuf<int64_t> soff;
  DBuf<unsigned long long> stop;
  {
    const char* e = getenv("CAMG_SPGEMM_STAGE");
    size_t fr = 0, tot = 0;
    CAMG_CUDA(cudaMemGetInfo(&fr, &tot));
    const int64_t cap = std::min<int64_t>(std::min<int64_t>((int64_t)(0.4 * (double)fr) / 12, (int64_t(16) << 30) / 12),
                                          std::max<int64_t>(est_nnz, int64_t(1) << 16));
    if (!(e && e[0] == '0') && n_rows > 0 && cap > 0) {
      scol = DBuf<int32_t>(cap);
      sval = DBuf<double>(cap);
      soff = DBuf<int64_t>(n_rows + 1);
      stop = DBuf<unsigned long long>(1);
      CAMG_CUDA(cudaMemsetAsync(soff.p, 0xFF, sizeof(int64_t) * (n_rows + 1), s));
      CAMG_CUDA(cudaMemsetAsync(stop.p, 0, sizeof(unsigned long long), s));
      o.scol = scol.p;
      o.sval = sval.p;
      o.soff = soff.p;
      o.stop = stop.p;
      o.scap = cap;
    }
  }
  std::vector<int64_t> big;
  if (start_global) {
    // every row starts in the global-memory hash tables (L2-resident, full
    // occupancy) instead of the shared-memory ones
    big.resize(n_rows);
    for (int64_t i = 0; i < n_rows; ++i) big[i] = i;
  } else {
    if (n_rows) launch(false, false, nullptr, n_rows, 0, 0, nullptr, o);
    CAMG_CUDA(cudaStreamSynchronize(s));
    CAMG_LAUNCH_CHECK();
    big = overflow_rows(ovf.p, n_rows);
  }
  if (getenv("CAMG_DEBUG"))
    fprintf(stderr, "[camg] spgemm rows=%lld smem-overflow rows=%zu\n", (long long)n_rows, big.size());
  struct Batch { DBuf<int64_t> rows; int64_t n; uint32_t c1, c2; };
  std::vector<Batch> batches;
  uint32_t c1 = c1_0, c2 = c2_0;
  const size_t budget = size_t(2) << 30;
  while (!big.empty()) {
    CAMG_CHECK(c1 <= (1u << 28) && c2 <= (1u << 28), CAMG_ERR_NATIVE, "spgemm: row too large for the hash tables");
    DBuf<int64_t> rows(big.size() + 1);
    CAMG_CUDA(cudaMemcpy(rows.p, big.data(), sizeof(int64_t) * big.size(), cudaMemcpyHostToDevice));
    const size_t per = (size_t)c1 * 14 + (size_t)c2 * 12;
    int64_t warps = std::max<int64_t>(kWarpsPerBlock, std::min<int64_t>((int64_t)big.size(), (int64_t)(budget / per)));
    warps = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock * kWarpsPerBlock;
    DBuf<char> scratch((size_t)warps * per);
    CAMG_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int32_t) * (n_rows + 1), s));
    launch(false, true, rows.p, (int64_t)big.size(), c1, c2, scratch.p, o);
    CAMG_CUDA(cudaStreamSynchronize(s));
    CAMG_LAUNCH_CHECK();
    std::vector<int64_t> still = overflow_rows(ovf.p, n_rows);
    if (getenv("CAMG_DEBUG"))
      fprintf(stderr, "[camg] spgemm global pass caps %u/%u: rows %zu, overflow %zu\n", c1, c2, big.size(),
              still.size());
    std::vector<int64_t> done;
    size_t k = 0;
    for (int64_t r : big) {
      while (k < still.size() && still[k] < r) ++k;
      if (k < still.size() && still[k] == r) continue;
      done.push_back(r);
    }
    if (!done.empty()) {
      Batch b{DBuf<int64_t>(done.size() + 1), (int64_t)done.size(), c1, c2};
      CAMG_CUDA(cudaMemcpy(b.rows.p, done.data(), sizeof(int64_t) * done.size(), cudaMemcpyHostToDevice));
      batches.push_back(std::move(b));
    }
    big.swap(still);
    c1 *= 2;
    if (c2) c2 *= 2;
  }
  DBuf<int64_t> rp(n_rows + 1);
  exclusive_scan_i64(cnt.p, rp.p, n_rows, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  const int64_t nnz = read_i64(rp.p + n_rows);
  Csr* C = new Csr();
  C->n_rows = n_rows;
  C->n_cols = n_cols;
  C->nnz = nnz;
  C->rowptr = rp.release();
  C->col = dalloc<int32_t>(nnz);
  C->val = dalloc<double>(nnz);
  C->avg_row = n_rows ? double(nnz) / n_rows : 0.0;
  OutArgs f{nullptr, C->rowptr, C->col, C->val, nullptr, tol};
  f.rap_sort = rap_sort;
  f.soff = o.soff;
  if (o.scol && n_rows) {
    note_launch();
    k_copy_staged<<<grid_for(n_rows * 32, 256, int64_t(kNumSMs) * 16), 256, 0, s>>>(n_rows, o.soff, C->rowptr, o.scol,
                                                                                   o.sval, C->col, C->val);
    CAMG_LAUNCH_CHECK();
    unsigned long long used = 0;
    CAMG_CUDA(cudaMemcpyAsync(&used, o.stop, sizeof(used), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    if (getenv("CAMG_DEBUG"))
      fprintf(stderr, "[camg] spgemm staged %llu of %lld entries (cap %lld)\n", used, (long long)nnz,
              (long long)o.scap);
    if (used <= (unsigned long long)o.scap) {  // every row staged: nothing to recompute
      CAMG_CUDA(cudaStreamSynchronize(s));
      return C;
    }
  }
  // fill: small rows from shared memory (overflow rows are skipped there)
  if (n_rows && !start_global) launch(true, false, nullptr, n_rows, 0, 0, nullptr, f);
  for (auto& b : batches) {
    const size_t per = (size_t)b.c1 * 14 + (size_t)b.c2 * 12;
    int64_t warps = std::max<int64_t>(kWarpsPerBlock, std::min<int64_t>(b.n, (int64_t)(budget / per)));
    warps = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock * kWarpsPerBlock;
    DBuf<char> scratch((size_t)warps * per);
    launch(true, true, b.rows.p, b.n, b.c1, b.c2, scratch.p, f);
    CAMG_CUDA(cudaStreamSynchronize(s));
  }
  CAMG_CUDA(cudaStreamSynchronize(s));
  CAMG_LAUNCH_CHECK();
  return C;
}

constexpr uint32_t kCapProduct = 256;  // 3 KB per warp: products rows are short (D^-1 K P_tent: ~50), overflow -> global tables
constexpr uint32_t kCap1 = 2048, kCap2 = 512;

}  // namespace

Csr* spgemm_ex(const Csr* A, const Csr* B, bool reverse_a, double tol, cudaStream_t s, const double* scale_a) {
  CAMG_CHECK(A->n_cols == B->n_rows, CAMG_ERR_DIMENSION, "sp_matmul: inner dimensions differ");
  CAMG_CHECK(B->n_cols < INT32_MAX, CAMG_ERR_DIMENSION, "too many columns");
  static uint32_t capp = 0;
  if (!capp) {
    const char* e = getenv("CAMG_SPGEMM_CAP");
    capp = e ? (uint32_t)atoi(e) : kCapProduct;
  }
  const size_t smem = (size_t)kWarpsPerBlock * capp * 12;
  static size_t attr = 0;
  if (attr != smem) {
    CAMG_CUDA(cudaFuncSetAttribute(k_product<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CAMG_CUDA(cudaFuncSetAttribute(k_product<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  auto launch = [&](bool fill, bool global, const int64_t* rows, int64_t nrows, uint32_t c1, uint32_t c2,
                    char* scratch, OutArgs o) {
    note_launch();
    if (!global) {
      unsigned grid = (unsigned)std::min<int64_t>((nrows + kWarpsPerBlock - 1) / kWarpsPerBlock, kNumSMs * 32);
      if (fill) k_product<true, false><<<grid, 32 * kWarpsPerBlock, smem, s>>>(view(A), view(B), reverse_a, scale_a, rows, nrows, capp, nullptr, o);
      else k_product<false, false><<<grid, 32 * kWarpsPerBlock, smem, s>>>(view(A), view(B), reverse_a, scale_a, rows, nrows, capp, nullptr, o);
    } else {
      const size_t per = (size_t)c1 * 14 + (size_t)c2 * 12;
      int64_t warps = std::max<int64_t>(kWarpsPerBlock, std::min<int64_t>(nrows, (int64_t)((size_t(2) << 30) / per)));
      unsigned grid = (unsigned)((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
      if (fill) k_product<true, true><<<grid, 32 * kWarpsPerBlock, 0, s>>>(view(A), view(B), reverse_a, scale_a, rows, nrows, c1, scratch, o);
      else k_product<false, true><<<grid, 32 * kWarpsPerBlock, 0, s>>>(view(A), view(B), reverse_a, scale_a, rows, nrows, c1, scratch, o);
    }
    CAMG_LAUNCH_CHECK();
  };
  // output estimate: 2 (nnz(A) + nnz(B)) (D^-1 K P_tent: 0.4x; S~ products: small)
  return two_pass(A->n_rows, B->n_cols, launch, 2 * capp, 0, tol, s, 2 * (A->nnz + B->nnz));
}

Csr* spgemm(const Csr* A, const Csr* B, cudaStream_t s) { return spgemm_ex(A, B, false, kDropTol, s, nullptr); }

Csr* galerkin(const Csr* R, const Csr* A, const Csr* P, cudaStream_t s) {
  CAMG_CHECK(R->n_cols == A->n_rows && A->n_cols == P->n_rows, CAMG_ERR_DIMENSION,
             "galerkin_triple: dimension mismatch");
  // hash capacities per warp (powers of two; CAMG_RAP_CAP1/2 override for tuning)
  static uint32_t cap1 = 0, cap2 = 0;
  if (!cap1) {
    const char* e1 = getenv("CAMG_RAP_CAP1");
    const char* e2 = getenv("CAMG_RAP_CAP2");
    cap1 = e1 ? (uint32_t)atoi(e1) : kCap1;
    cap2 = e2 ? (uint32_t)atoi(e2) : kCap2;
  }
  const size_t per = (size_t)cap1 * 14 + (size_t)cap2 * 12;
  const size_t smem = (size_t)kWarpsPerBlock * per;
  static size_t attr = 0;
  if (attr != smem) {
    CAMG_CUDA(cudaFuncSetAttribute(k_triple<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CAMG_CUDA(cudaFuncSetAttribute(k_triple<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  auto launch = [&](bool fill, bool global, const int64_t* rows, int64_t nrows, uint32_t c1, uint32_t c2,
                    char* scratch, OutArgs o) {
    note_launch();
    if (!global) {
      unsigned grid = (unsigned)std::min<int64_t>((nrows + kWarpsPerBlock - 1) / kWarpsPerBlock, kNumSMs * 32);
      if (fill) k_triple<true, false><<<grid, 32 * kWarpsPerBlock, smem, s>>>(view(R), view(A), view(P), rows, nrows, cap1, cap2, nullptr, o);
      else k_triple<false, false><<<grid, 32 * kWarpsPerBlock, smem, s>>>(view(R), view(A), view(P), rows, nrows, cap1, cap2, nullptr, o);
    } else {
      const size_t pw = (size_t)c1 * 14 + (size_t)c2 * 12;
      int64_t warps = std::min<int64_t>(nrows, std::max<int64_t>(kWarpsPerBlock, (int64_t)((size_t(2) << 30) / pw)));
      unsigned grid = (unsigned)((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
      // h2 in shared memory up to 48 KB per block (CAMG_RAP_H2_SMEM=0: global)
      static const bool h2_env = !(getenv("CAMG_RAP_H2_SMEM") && getenv("CAMG_RAP_H2_SMEM")[0] == '0');
      const size_t sm2 = (size_t)kWarpsPerBlock * c2 * 12;
      static bool gattr = false;
      if (!gattr) {
        CAMG_CUDA(cudaFuncSetAttribute(k_triple<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        CAMG_CUDA(cudaFuncSetAttribute(k_triple<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        gattr = true;
      }
      o.h2_smem = h2_env && sm2 <= size_t(96) * 1024;
      const size_t dyn = o.h2_smem ? sm2 : 0;
      if (fill) k_triple<true, true><<<grid, 32 * kWarpsPerBlock, dyn, s>>>(view(R), view(A), view(P), rows, nrows, c1, c2, scratch, o);
      else k_triple<false, true><<<grid, 32 * kWarpsPerBlock, dyn, s>>>(view(R), view(A), view(P), rows, nrows, c1, c2, scratch, o);
    }
    CAMG_LAUNCH_CHECK();
  };
  // output estimate for the staging buffer: nnz(R) + nnz(A) + nnz(P) (C5
  // level 0: 2.8e9 for a 0.28e9-entry coarse K)
  const int64_t est = R->nnz + A->nnz + P->nnz;
  static int rap_global = -1;
  if (rap_global < 0) {
    const char* e = getenv("CAMG_RAP_GLOBAL");
    rap_global = (e && e[0] == '0') ? 0 : 1;
  }
  // long RA rows (K-block RAP: ~350 R entries x ~80 K entries per coarse
  // row) start in the global-memory tables: L2-resident, ~28 warps per SM
  // against 6 with shared-memory tables (C5: 7.0 s -> 4.7 s)
  if (rap_global && R->avg_row * A->avg_row > 4096.0)
    return two_pass(R->n_rows, P->n_cols, launch, cap1, cap2, kDropTol, s, est, true);
  return two_pass(R->n_rows, P->n_cols, launch, 2 * cap1, 2 * cap2, kDropTol, s, est);
}

}  // namespace camg

using namespace camg;

namespace camg {
Csr* spgemm_ex(const Csr* A, const Csr* B, bool reverse_a, double tol, cudaStream_t s, const double* scale_a);
void recip(int64_t n, const double* d, double* out, cudaStream_t s);
Csr* scale_cols(const Csr* A, const double* c, cudaStream_t s);

// P = P_tent - omega_eff * ((diag(1/d) A) P_tent)  (transfer.py:164-183)
Csr* smooth_prolongator(const Csr* Pt, const Csr* A, const double* d, double omega_eff, cudaStream_t s) {
  CAMG_CHECK(A->n_rows == A->n_cols && A->n_rows == Pt->n_rows, CAMG_ERR_DIMENSION,
             "smooth_prolongator: A and P_tent dimensions mismatch");
  DBuf<double> dinv(A->n_rows + 1);
  recip(A->n_rows, d, dinv.p, s);
  // X = (D^-1 A) P_tent as raw csr_matmat (exact zeros dropped); the row
  // scaling happens on the fly, bit-identical to materialising D^-1 A
  Csr* X = spgemm_ex(A, Pt, false, 0.0, s, dinv.p);
  Csr* P = csr_axpby(1.0, Pt, -omega_eff, X, s);  // P_tent - omega*X, canonical
  delete X;
  return P;
}

// S~ = scale*Cz + scale*((B2 diag(ainv)) B1)   (smoothers.py:233-238)
Csr* schur(const Csr* B2, const Csr* Cz, const Csr* B1, const double* ainv, double scale, cudaStream_t s) {
  // B2 @ diags(ainv): every entry b*a (0 + product); scipy's output row is in
  // reverse first-touch order, i.e. B2's row reversed -> the next product
  // walks it backwards.
  Csr* T = scale_cols(B2, ainv, s);
  Csr* X = spgemm_ex(T, B1, true, 0.0, s, nullptr);
  delete T;
  Csr* S = csr_axpby(scale, Cz, scale, X, s);
  delete X;
  return S;
}

__global__ void k_recip(int64_t n, const double* __restrict__ d, double* __restrict__ o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __drcp_rn(d[i]);
}

void recip(int64_t n, const double* d, double* out, cudaStream_t s) {
  note_launch();
  k_recip<<<grid_for(n, 256), 256, 0, s>>>(n, d, out);
}

// column scaling keeping exact zeros of the product out (csr_matmat with a
// diagonal right factor)
template <bool FILL>
__global__ void k_scale_cols(CsrView A, const double* __restrict__ c, int64_t* __restrict__ cnt,
                             const int64_t* __restrict__ crow, int32_t* __restrict__ ccol, double* __restrict__ cval) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = 0, out = FILL ? crow[r] : 0;
    for (int64_t p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) {
      double v = __dadd_rn(0.0, __dmul_rn(A.val[p], c[A.col[p]]));
      if (v != 0.0) {
        if (FILL) { ccol[out + n] = A.col[p]; cval[out + n] = v; }
        ++n;
      }
    }
    if (!FILL) cnt[r] = n;
  }
}

Csr* scale_cols(const Csr* A, const double* c, cudaStream_t s) {
  DBuf<int64_t> cnt(A->n_rows + 1);
  note_launch();
  k_scale_cols<false><<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), c, cnt.p, nullptr, nullptr, nullptr);
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
  k_scale_cols<true><<<grid_for(A->n_rows, 256), 256, 0, s>>>(view(A), c, nullptr, C->rowptr, C->col, C->val);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  return C;
}

}  // namespace camg

extern "C" {

int camg_spgemm(const camg_csr* A, const camg_csr* B, camg_csr** out) {
  return guarded([&] { *out = new camg_csr{spgemm(A->m, B->m, 0)}; });
}

int camg_galerkin(const camg_csr* R, const camg_csr* A, const camg_csr* P, camg_csr** out) {
  return guarded([&] { *out = new camg_csr{galerkin(R->m, A->m, P->m, 0)}; });
}

int camg_smooth_prolongator(const camg_csr* P_tent, const camg_csr* A, const double* d, double omega_eff,
                            camg_csr** out) {
  return guarded([&] { *out = new camg_csr{smooth_prolongator(P_tent->m, A->m, d, omega_eff, 0)}; });
}

int camg_schur(const camg_csr* B2, const camg_csr* Cz, const camg_csr* B1, const double* ainv, double scale,
               camg_csr** out) {
  return guarded([&] {
    CAMG_CHECK(B2->m->n_cols == B1->m->n_rows && B2->m->n_rows == Cz->m->n_rows && B1->m->n_cols == Cz->m->n_cols,
               CAMG_ERR_DIMENSION, "schur: inconsistent block shapes");
    *out = new camg_csr{schur(B2->m, Cz->m, B1->m, ainv, scale, 0)};
  });
}

}  // extern "C"

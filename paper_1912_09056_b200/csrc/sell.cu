// Block SELL-32 mirror of the leading rows of a CSR matrix, with BR x BC
// node blocks (BR = DOFs per row node, BC = DOFs per column node), used for
// the fine-level [K | B1] stream (3x3 in 3-D) and the transfers (P: 3x6,
// R: 6x3 with rigid-body coarse spaces).
//
// Slice = 32 consecutive block rows, one lane per block row.  Slot k of a
// slice holds block k of each of its 32 rows: one int32 column per lane, and
// the block values interleaved as [value][lane] so every load of the warp is
// one contiguous 128 B (columns) / 256 B (values) transaction.  Each lane
// keeps BR independent FMA chains in registers; no shuffles.  Rows shorter
// than the slice width skip their padding (per-row length byte).
//
// Masked slots: a slot stores only the block positions that are non-zero in
// at least one lane of its slice (a per-slot bit mask, warp-uniform).
// Structured-mesh stencils repeat along a slice, so the union equals the
// exact pattern of interior nodes: a hex8 interior node row has 183 non-zeros
// in its 27 3x3 blocks, so the slice streams 183*8 + 27*4 = 1572 B per node
// row instead of 2052 B (full blocks) or 2316 B (int32 CSR of the same
// matrix).  Unstructured patterns fall back to the union (never worse than
// full blocks).
#include <algorithm>
#include <cstdlib>

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"
#include "sell.cuh"

// 4 CTAs of 256 threads per SM (64 registers): every slot's value loads go
// out in one batch (at 5-6 CTAs / 40-48 registers ptxas interleaves them with
// their FMAs: C5 V-cycle 20.0 ms vs 24.2 / 27.3 ms)
#ifndef CAMG_MASKED_MINB
#define CAMG_MASKED_MINB 4
#endif
// blocks of >= 18 entries (6x6 level-1 operators, 3x6 / 6x3 transfers): at
// the default 40 registers ptxas interleaves each load with its FMA (a few
// loads in flight per warp); 4 CTAs/SM (62 registers) batches them (C5
// V-cycle 21.72 -> 21.35 ms; 2 CTAs / 122 registers, all 36 loads of a 6x6
// slot in one batch, measured the same)
// 64-thread CTAs for the one-lane-per-row kernels: finer CTA granularity
// rebalances the per-SM load (C5 fine predictor pass 2.113 -> 2.067 ms,
// V-cycle 19.8 -> 19.5 ms; 128: 2.083 ms, 512: 2.140 ms, 32: 2.34 ms -- the
// 32-CTA/SM limit caps 1-warp CTAs at 32 warps)
#ifndef CAMG_SELL_THREADS
#define CAMG_SELL_THREADS 64
#endif
#ifndef CAMG_BIG_MINB
#define CAMG_BIG_MINB 4
#endif
// shared-value-group passes are bound by L1 / issue, not by loads in flight
#ifndef CAMG_DEDUP_MINB
#define CAMG_DEDUP_MINB 4
#endif
// non-uniform shared slots stored dense (a group per block position) instead of their union pattern:
// same pass time, twice the dictionary (92 vs 44 MB on C5), merged SpMV 0.905 -> 0.957 ms
#ifndef CAMG_DEDUP_NUDENSE
#define CAMG_DEDUP_NUDENSE 0
#endif



namespace camg {

constexpr int kSellThreads = CAMG_SELL_THREADS;  // threads per CTA of the one-lane-per-row kernels

Sell::~Sell() {
  dfree(slice_ptr);
  dfree(len);
  dfree(bcol);
  dfree(bval);
  dfree(mask);
  dfree(voff);
  dfree(desc);
  dfree(zero);
  dfree(vo);
  dfree(uslice);
  dfree(witems);
  dfree(wmode);
  dfree(wdist);
  dfree(xpart);
  dfree(perm);
  dfree(dblk);
}

namespace {

// Walk the distinct block columns of block row p (union over its BR rows);
// f(k, block_col, pos[]) is called per block with the row cursors positioned
// at that block's entries.
template <int BR, int BC, class F>
__device__ int for_blocks(const CsrView& A, int64_t p, F f) {
  int64_t pos[BR], end[BR];
#pragma unroll
  for (int r = 0; r < BR; ++r) {
    pos[r] = A.rowptr[p * BR + r];
    end[r] = A.rowptr[p * BR + r + 1];
  }
  int k = 0;
  while (true) {
    int32_t best = INT32_MAX;
#pragma unroll
    for (int r = 0; r < BR; ++r)
      if (pos[r] < end[r]) best = min(best, A.col[pos[r]] / BC);
    if (best == INT32_MAX) break;
    uint64_t m = 0;
#pragma unroll
    for (int r = 0; r < BR; ++r)
      while (pos[r] < end[r] && A.col[pos[r]] / BC == best) {
        const int c = A.col[pos[r]] - best * BC;
        f(k, best, r, c, A.val[pos[r]]);
        m |= 1ull << (r * BC + c);
        ++pos[r];
      }
    f(k, best, -1, -1, (double)m);  // end of block k: m = its entry mask
    ++k;
  }
  return k;
}

template <int BR, int BC>
__global__ void k_sell_count(CsrView A, int64_t nbr, int64_t ncols_blocked, const int32_t* __restrict__ perm,
                             uint8_t* __restrict__ len, int32_t* __restrict__ overflow) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nbr; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = perm ? perm[t] : t;  // position t holds block row p (-1: padding)
    if (p < 0) { len[t] = 0; continue; }
    for (int r = 0; r < BR; ++r) {
      const int64_t e = A.rowptr[p * BR + r + 1];
      if (e > A.rowptr[p * BR + r] && A.col[e - 1] >= ncols_blocked) atomicExch(overflow, 1);
    }
    int n = for_blocks<BR, BC>(A, p, [](int, int32_t, int, int, double) {});
    if (n > 255) { atomicExch(overflow, 2); n = 255; }
    len[t] = (uint8_t)n;
  }
}

__global__ void k_slice_width(const uint8_t* __restrict__ len, int64_t nbr, int64_t nslices, int64_t* __restrict__ w) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x) {
    int m = 0;
    for (int l = 0; l < 32; ++l) {
      int64_t p = s * 32 + l;
      if (p < nbr) m = max(m, (int)len[p]);
    }
    w[s] = m;
  }
}

// Offset-aligned slots (masked mirrors).  Slot k of a slice normally holds every lane's k-th block; where the
// block rows of a slice share one set of block-column offsets (column - row: the stencil of a structured
// mesh), slot j holds instead, in every lane, the block at the j-th offset of that set -- an explicit zero
// block (same fma(0, x, acc) as an absent position of a masked block) where a lane has none (a boundary
// node).  Slices that straddle a mesh row or touch a boundary then have the interior's linear, lane-uniform
// slots (kind 1 / 2) instead of per-lane columns and values.  A slice is aligned when the union of its
// lanes' offsets has at most kOffCap entries and pads its longest row by at most an eighth (an
// unstructured matrix never qualifies and keeps the rank order).  The order of a lane's own blocks is
// unchanged (ascending columns), so every result is.
constexpr int kOffCap = 32;

template <int BR, int BC>
__global__ void k_slice_offsets(CsrView A, int64_t nbr, int64_t nslices, const uint8_t* __restrict__ len,
                                int32_t* __restrict__ otab, uint8_t* __restrict__ wal) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = warp; sl < nslices; sl += nwarps) {
    const int64_t p = sl * 32 + lane;
    const bool active = p < nbr;
    int64_t pos[BR], end[BR];
#pragma unroll
    for (int r = 0; r < BR; ++r) {
      pos[r] = active ? A.rowptr[p * BR + r] : 0;
      end[r] = active ? A.rowptr[p * BR + r + 1] : 0;
    }
    int maxlen = active ? (int)len[p] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    int cnt = 0;
    bool ok = true;
    while (true) {
      int32_t head = INT32_MAX;
#pragma unroll
      for (int r = 0; r < BR; ++r)
        if (pos[r] < end[r]) head = min(head, A.col[pos[r]] / BC);
      const int32_t off = head == INT32_MAX ? INT32_MAX : (int32_t)((int64_t)head - p);
      int32_t m = off;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (m == INT32_MAX) break;
      if (cnt == kOffCap) { ok = false; break; }
      if (lane == 0) otab[sl * kOffCap + cnt] = m;
      ++cnt;
      if (off == m) {
#pragma unroll
        for (int r = 0; r < BR; ++r)
          while (pos[r] < end[r] && A.col[pos[r]] / BC == head) ++pos[r];
      }
    }
    if (lane == 0) wal[sl] = (ok && cnt > 0 && cnt <= maxlen + max(1, maxlen / 8)) ? (uint8_t)cnt : 0;
  }
}

// widths and row lengths of the aligned slices: every lane holds a block (possibly zero) in every slot
__global__ void k_apply_aligned(const uint8_t* __restrict__ wal, int64_t nbr, int64_t nslices, int64_t* __restrict__ w,
                                uint8_t* __restrict__ len) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nslices * 32;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int a = wal[p >> 5];
    if (!a) continue;
    if ((p & 31) == 0) w[p >> 5] = a;
    if (p < nbr) len[p] = (uint8_t)a;
  }
}

// slot of block column bc in block row p: its rank k, or the position of its offset in an aligned slice
__device__ __forceinline__ int slot_of(const int32_t* __restrict__ otab, const uint8_t* __restrict__ wal, int64_t p,
                                       int k, int32_t bc) {
  const int n = wal ? (int)wal[p >> 5] : 0;
  if (!n) return k;
  const int32_t* t = otab + (p >> 5) * kOffCap;
  const int32_t off = (int32_t)((int64_t)bc - p);
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (t[mid] < off) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// union mask of every slot (masked mode) or all-ones (full blocks)
template <int BR, int BC>
__global__ void k_sell_masks(CsrView A, int64_t nbr, const int64_t* __restrict__ slice_ptr,
                             const int32_t* __restrict__ otab, const uint8_t* __restrict__ wal,
                             unsigned long long* __restrict__ mask) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nbr; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = slice_ptr[p >> 5];
    for_blocks<BR, BC>(A, p, [&](int k, int32_t bc, int r, int, double m) {
      if (r < 0) atomicOr(mask + base + slot_of(otab, wal, p, k, bc), (unsigned long long)m);
    });
  }
}

__global__ void k_slot_popc(const unsigned long long* __restrict__ mask, int64_t slots, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < slots; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = __popcll(mask[i]);
}

// linear slots of masked SELL: every lane of a full slice has a block in the
// slot and lane l's block column is c0 + l (interior nodes of a structured
// mesh: one stencil offset per slot).  The descriptor then carries c0 + 1 in
// bits 36-59 and the kernel derives the columns instead of loading them.
__global__ void k_slot_linear(const int64_t* __restrict__ slice_ptr, const uint8_t* __restrict__ len,
                              const int32_t* __restrict__ bcol, int64_t nbr, int64_t nslices,
                              unsigned long long* __restrict__ desc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = warp; sl < nslices; sl += nwarps) {
    const int64_t base = slice_ptr[sl], width = slice_ptr[sl + 1] - base;
    const int64_t p = sl * 32 + lane;
    const int n = p < nbr ? len[p] : -1;
    for (int64_t k = 0; k < width; ++k) {
      const int32_t c = n > k ? bcol[(base + k) * 32 + lane] : -1;
      const int32_t c0 = __shfl_sync(0xffffffffu, c, 0);
      const bool lin = __all_sync(0xffffffffu, n > k && c == c0 + lane) && c0 >= 0 && c0 + 1 < (1 << 24);
      if (lin && lane == 0) desc[base + k] |= (unsigned long long)(c0 + 1) << 36;
    }
  }
}

// slot descriptors of masked SELL with at most 9 positions per block: the
// kernel reads position q's value from group (nibble q) - 1 of the slot, or
// uses 0 when the nibble is 0, so every load address is a shift-and-mask of
// one warp-uniform word (no per-position branches, all loads independent)
__global__ void k_slot_desc(const unsigned long long* __restrict__ mask, int64_t slots, int be,
                            unsigned long long* __restrict__ desc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < slots; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long m = mask[i];
    unsigned long long d = 0;
    int rank = 0;
    for (int q = 0; q < be; ++q)
      if (m & (1ull << q)) d |= (unsigned long long)(++rank) << (4 * q);
    desc[i] = d | ((unsigned long long)rank << 60);
  }
}

template <int BR, int BC>
__global__ void k_sell_fill(CsrView A, int64_t nbr, const int32_t* __restrict__ perm,
                            const int64_t* __restrict__ slice_ptr, const unsigned long long* __restrict__ mask,
                            const int64_t* __restrict__ voff, int32_t* __restrict__ bcol, double* __restrict__ bval,
                            double* __restrict__ dblk, const int32_t* __restrict__ otab,
                            const uint8_t* __restrict__ wal, int64_t ncb_sq) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nbr; t += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(t & 31);
    const int64_t base = slice_ptr[t >> 5];
    const int64_t width = slice_ptr[(t >> 5) + 1] - base;
    const int64_t p = perm ? perm[t] : t;
    const int al = (wal && !perm) ? (int)wal[t >> 5] : 0;
    // aligned slice: a slot this lane has no block in reads the column at its offset (its own where that
    // falls outside the square part) against a zero block
    for (int j = 0; j < al; ++j) {
      const int64_t c = p + otab[(t >> 5) * kOffCap + j];
      bcol[(base + j) * 32 + lane] = (int32_t)((c >= 0 && c < ncb_sq) ? c : (p < ncb_sq ? p : 0));
    }
    int n = 0;
    if (p >= 0) n = for_blocks<BR, BC>(A, p, [&](int k, int32_t bc, int r, int c, double v) {
      const int64_t slot = base + (al ? slot_of(otab, wal, p, k, bc) : k);
      if (r < 0) {
        bcol[slot * 32 + lane] = bc;
        return;
      }
      const int e = r * BC + c;
      // diagonal node block, [slice][entry][lane] (Gauss-Seidel within the node)
      if (dblk && bc == p) dblk[((t >> 5) * (BR * BC) + e) * 32 + lane] = v;
      const uint64_t m = mask[slot];
      const int64_t idx = voff[slot] + __popcll(m & ((1ull << e) - 1ull));
      bval[idx * 32 + lane] = v;
    });
    if (!al)
      for (int k = n; k < width; ++k) bcol[(base + k) * 32 + lane] = 0;  // padding (never read)
  }
}

// per block row: its stored value bytes + column bytes (acc[0]) and blocks (acc[1])
__global__ void k_sell_row_bytes(const int64_t* __restrict__ slice_ptr, const uint8_t* __restrict__ len,
                                 const unsigned long long* __restrict__ mask,
                                 const unsigned long long* __restrict__ desc, int64_t nbr,
                                 unsigned long long* __restrict__ acc) {
  unsigned long long b = 0, u = 0, cb = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nbr; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = slice_ptr[p >> 5];
    const int n = len[p];
    for (int k = 0; k < n; ++k) {
      const unsigned long long c = (desc && ((desc[base + k] >> 36) & 0xFFFFFFull)) ? 0ull : 4ull;
      b += 8ull * __popcll(mask[base + k]) + c;
      cb += c;
    }
    u += n;
  }
  for (int o = 16; o > 0; o >>= 1) {
    b += __shfl_xor_sync(0xffffffffu, b, o);
    u += __shfl_xor_sync(0xffffffffu, u, o);
    cb += __shfl_xor_sync(0xffffffffu, cb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, b);
    atomicAdd(acc + 1, u);
    atomicAdd(acc + 2, cb);
  }
}


// ---------------------------------------------------------------------------
// Shared value groups of a masked mirror.  Two slots with the same mask and
// bit-identical stored values (every lane, every position) need one copy:
// on a structured mesh the interior stencil repeats from slice to slice, so
// the value stream of the mirror collapses to a small dictionary that lives
// in L1/L2, and a pass streams only descriptors, columns and the vectors.
// The result of every product is unchanged (same values, same order).
// Slots are grouped by a 64-bit hash of their content, sorted (stable radix
// sort), and every slot is compared bit for bit with the first slot of its
// hash run before it shares that slot's copy (a hash collision keeps its own).

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_slot_hash(const unsigned long long* __restrict__ mask, const int64_t* __restrict__ voff,
                            const double* __restrict__ bval, int64_t slots, unsigned long long* __restrict__ key,
                            uint32_t* __restrict__ idx, uint8_t* __restrict__ uni, uint32_t* __restrict__ uinfo) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < slots; s += nwarps) {
    const unsigned long long m = mask[s];
    const int ng = __popcll(m);
    const double* v = bval + voff[s] * 32 + lane;
    unsigned long long h = 0;
    for (int g = 0; g < ng; ++g)
      h += mix64((unsigned long long)__double_as_longlong(v[g * 32]) ^ mix64((unsigned long long)(g * 32 + lane + 1)));
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0) {
      key[s] = mix64(h ^ mix64(m));
      idx[s] = (uint32_t)s;
    }
    if (uni) {
      // kind 1: every lane holds the same block.  kind 2: all but one or two
      // lanes do (a slice that straddles a mesh row: the two boundary nodes
      // differ) -- info = majority lane | exception lanes << 8, << 16 (0xFF: none)
      unsigned kind = 0, info = 0;
      unsigned tried = 0;
      for (int t = 0; t < 3 && !kind; ++t) {
        // candidate majority lane: the lowest lane not yet known to be an exception
        const int a = __ffs(~tried) - 1;
        bool eq = true;
        for (int g = 0; g < ng; ++g) {
          const long long b = __double_as_longlong(v[g * 32]);
          eq &= b == __shfl_sync(0xffffffffu, b, a);
        }
        const unsigned same = __ballot_sync(0xffffffffu, eq);
        const unsigned exc = ~same;
        if (exc == 0) kind = 1;
        else if (__popc(exc) <= 2) {
          kind = 2;
          const int e0 = __ffs(exc) - 1;
          const unsigned rest = exc & (exc - 1);
          const int e1 = rest ? __ffs(rest) - 1 : 0xFF;
          info = (unsigned)a | ((unsigned)e0 << 8) | ((unsigned)e1 << 16);
        } else tried |= same;  // lane a and its equals are the exceptions, if anything
      }
      if (lane == 0) { uni[s] = (uint8_t)kind; uinfo[s] = info; }
    }
  }
}

__global__ void k_run_heads(const unsigned long long* __restrict__ key, int64_t n, int64_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? i : 0;
}

// rep[s] = the slot whose copy s shares (itself: s keeps its own values)
__global__ void k_slot_verify(const unsigned long long* __restrict__ mask, const int64_t* __restrict__ voff,
                              const double* __restrict__ bval, const uint32_t* __restrict__ sidx,
                              const int64_t* __restrict__ head, int64_t slots, uint32_t* __restrict__ rep) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < slots; i += nwarps) {
    const uint32_t s = sidx[i], r = sidx[head[i]];
    bool eq = true;
    if (s != r) {
      const unsigned long long m = mask[s];
      eq = m == mask[r];
      if (eq) {
        const int ng = __popcll(m);
        const double* a = bval + voff[s] * 32 + lane;
        const double* b = bval + voff[r] * 32 + lane;
        for (int g = 0; g < ng; ++g) eq &= __double_as_longlong(a[g * 32]) == __double_as_longlong(b[g * 32]);
      }
      eq = __all_sync(0xffffffffu, eq);
    }
    if (lane == 0) rep[s] = eq ? r : s;
  }
}

__global__ void k_slot_own_groups(const unsigned long long* __restrict__ mask, const uint32_t* __restrict__ rep,
                                  const uint8_t* __restrict__ uni, int64_t slots, int be,
                                  int64_t* __restrict__ cnt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < slots; s += (int64_t)gridDim.x * blockDim.x)
    cnt[s] = rep[s] == (uint32_t)s ? (uni[s] ? 1 : (CAMG_DEDUP_NUDENSE ? be : __popcll(mask[s]))) : 0;
}

// copy the kept slots' groups to the compact array; a lane-uniform slot (uni)
// becomes one group holding its dense block: entry q = the value at position
// q, or 0 where the slot's mask has no entry
__global__ void k_slot_compact(const unsigned long long* __restrict__ mask, const int64_t* __restrict__ voff,
                               const double* __restrict__ bval, const uint32_t* __restrict__ rep,
                               const int64_t* __restrict__ noff, int64_t slots, int be, double* __restrict__ nval,
                               const uint8_t* __restrict__ uni, const uint32_t* __restrict__ uinfo) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < slots; s += nwarps) {
    if (rep[s] != (uint32_t)s) continue;
    const unsigned long long m = mask[s];
    const double* a = bval + voff[s] * 32;
    double* o = nval + noff[s] * 32 + lane;
    if (uni[s]) {
      // one group: entries 0..be-1 the majority lane's dense block (zeros where
      // the mask has no entry); kind 2 adds the dense blocks of its exception
      // lanes at entries 10.. and 20.. (the lanes are named in the descriptor)
      const unsigned info = uni[s] == 2 ? uinfo[s] : 0u;
      const int src = lane < 10 ? (int)(info & 0xFF) : lane < 20 ? (int)((info >> 8) & 0xFF) : (int)((info >> 16) & 0xFF);
      const int q = lane < 10 ? lane : lane < 20 ? lane - 10 : lane - 20;
      double x = 0.0;
      if (q < be && src != 0xFF && (uni[s] == 2 || lane < 10) && ((m >> q) & 1ull))
        x = a[__popcll(m & ((1ull << q) - 1ull)) * 32 + src];
      *o = x;
    } else {
#if CAMG_DEDUP_NUDENSE
      // every position of the block gets a group (zeros where the mask has
      // none): the pass reads position q at a fixed offset
      for (int q = 0; q < be; ++q)
        o[q * 32] = (m >> q) & 1ull ? a[__popcll(m & ((1ull << q) - 1ull)) * 32 + lane] : 0.0;
#else
      const int ng = __popcll(m);
      for (int g = 0; g < ng; ++g) o[g * 32] = a[g * 32 + lane];
#endif
    }
  }
}

__global__ void k_slot_share(const uint32_t* __restrict__ rep, const int64_t* __restrict__ noff,
                             const uint8_t* __restrict__ uni, const uint32_t* __restrict__ uinfo, int64_t slots,
                             uint32_t* __restrict__ vo, unsigned long long* __restrict__ desc) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < slots; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rep[s];
    vo[s] = (uint32_t)noff[r];
    unsigned long long d = (desc[s] & ~(0xFull << 60)) | ((unsigned long long)uni[r] << 60);  // bits 60-61: slot kind
    // dense slots need no pattern nibbles; kind 2 keeps its exception lanes there (bits 0-7, 8-15)
    if (uni[r] == 2) d = (d & ~0xFFFFFFFFFull) | (unsigned long long)(uinfo[r] >> 8);
    desc[s] = d;
  }
}

// uniform slices: a full slice (32 block rows, at most 32 slots) whose slots are all linear and
// lane-uniform (kind 1, or kind 2: but for one or two lanes) and read block columns below `sq` (the square
// part: never the split vector)
__global__ void k_uniform_slices(const int64_t* __restrict__ slice_ptr, const uint8_t* __restrict__ len,
                                 const unsigned long long* __restrict__ desc, int64_t nbr, int64_t nslices,
                                 int64_t sq, uint8_t* __restrict__ us, unsigned long long* __restrict__ count) {
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nslices;
       sl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = slice_ptr[sl], width = slice_ptr[sl + 1] - base;
    bool ok = width > 0 && width <= 32 && sl * 32 + 31 < nbr, exc = false;
    for (int l = 0; ok && l < 32; ++l) ok = len[sl * 32 + l] == width;
    for (int64_t k = 0; ok && k < width; ++k) {
      const unsigned long long d = desc[base + k];
      const int64_t lin = (int64_t)((d >> 36) & 0xFFFFFFull);
      const unsigned kind = (unsigned)(d >> 60) & 3u;
      ok = (kind == 1u || kind == 2u) && lin > 0 && lin - 1 + 31 < sq;
      exc |= kind == 2u;
    }
    us[sl] = ok ? (exc ? 2 : 1) : 0;  // 2: some slots have one or two exception lanes (kind 2)
    if (ok) atomicAdd(count, 1ull);
  }
}

// groups of uniform slices: neighbouring slices with the same shared value groups slot by slot and columns
// 32 apart (one mesh row) run as one work item, each lane carrying two or three block rows, so the
// lane-uniform values -- 72 of the 96 bytes a lane receives per slot, the L1 data pipe's load -- are loaded
// once for the group.  A run of compatible slices (broken every 60) is cut into threes and twos (a lone
// slice stays 1): us = 3 / 5 leader of two / three, 4 / 6 first / second follower
__device__ bool uslice_compat(const int64_t* __restrict__ slice_ptr, const unsigned long long* __restrict__ desc,
                              const uint32_t* __restrict__ vo, int64_t s) {  // slices s and s + 1
  const int64_t b0 = slice_ptr[s], b1 = slice_ptr[s + 1], width = b1 - b0;
  if (slice_ptr[s + 2] - b1 != width) return false;
  for (int64_t k = 0; k < width; ++k)
    if (vo[b0 + k] != vo[b1 + k] ||
        ((desc[b1 + k] >> 36) & 0xFFFFFFull) != ((desc[b0 + k] >> 36) & 0xFFFFFFull) + 32ull)
      return false;
  return true;
}

__global__ void k_uniform_groups(const int64_t* __restrict__ slice_ptr, const unsigned long long* __restrict__ desc,
                                 const uint32_t* __restrict__ vo, int64_t nslices, const uint8_t* __restrict__ us,
                                 uint8_t* __restrict__ out, unsigned long long* __restrict__ count) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (us[s] != 1) continue;
    // run start: the slice before is not a compatible uniform slice, or a forced break
    if (s % 60 != 0 && s > 0 && us[s - 1] == 1 && uslice_compat(slice_ptr, desc, vo, s - 1)) continue;
    int64_t L = 1;
    while (s + L < nslices && (s + L) % 60 != 0 && us[s + L] == 1 && uslice_compat(slice_ptr, desc, vo, s + L - 1)) ++L;
    int64_t t = s;
    while (L > 1) {
      const int g = (L == 2 || L == 4) ? 2 : 3;
      out[t] = g == 2 ? 3 : 5;
      out[t + 1] = 4;
      if (g == 3) out[t + 2] = 6;
      atomicAdd(count, 1ull);
      t += g;
      L -= g;
    }
  }
}

// period of a slice with exception lanes: the distance d (in slices) to a slice with the same width, value
// groups and exception lanes, slot by slot, and first columns 32 d further on.  Candidates are the
// differences of the slice's own slot columns (on a structured mesh the mesh-row length is one of them: 32
// mesh rows of nx nodes are nx slices); 0 = none
__global__ void k_exc_partner(const int64_t* __restrict__ slice_ptr, const unsigned long long* __restrict__ desc,
                              const uint32_t* __restrict__ vo, const uint8_t* __restrict__ us, int64_t nslices,
                              int32_t* __restrict__ xpart) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices;
       s += (int64_t)gridDim.x * blockDim.x) {
    int32_t found = 0;
    if (us[s] == 2) {
      const int64_t b0 = slice_ptr[s], width = slice_ptr[s + 1] - b0;
      const int64_t c0 = (int64_t)((desc[b0] >> 36) & 0xFFFFFFull);
      for (int64_t q = 1; q < width && !found; ++q) {
        const int64_t d = (int64_t)((desc[b0 + q] >> 36) & 0xFFFFFFull) - c0;
        if (d < 2 || s + d >= nslices || us[s + d] != 2) continue;
        const int64_t b1 = slice_ptr[s + d];
        bool ok = slice_ptr[s + d + 1] - b1 == width;
        for (int64_t k = 0; ok && k < width; ++k) {
          const unsigned long long da = desc[b0 + k], db = desc[b1 + k];
          ok = vo[b0 + k] == vo[b1 + k] && (da >> 60) == (db >> 60) &&
               ((db >> 36) & 0xFFFFFFull) == ((da >> 36) & 0xFFFFFFull) + 32ull * (unsigned long long)d &&
               (((da >> 60) & 3ull) != 2ull || (da & 0xFFFFull) == (db & 0xFFFFull));
        }
        if (ok) found = (int32_t)d;
      }
    }
    xpart[s] = found;
  }
}

// Replace S's value array by the shared one when that at least halves it;
// returns the value groups kept (S->ngroups) -- S->dedup says whether it applied.
static void share_value_groups(Sell* S, cudaStream_t s) {
  const int64_t slots = S->slots;
  S->ngroups_full = S->ngroups;
  if (slots < 2 || slots >= (int64_t)1 << 32) return;
  DBuf<unsigned long long> key(slots), key2(slots);
  DBuf<uint32_t> idx(slots), sidx(slots), rep(slots);
  DBuf<uint8_t> uni(slots);
  DBuf<uint32_t> uinfo(slots);
  CAMG_CUDA(cudaMemsetAsync(uni.p, 0, slots, s));
  note_launch();
  k_slot_hash<<<grid_for(slots * 32, 256), 256, 0, s>>>(S->mask, S->voff, S->bval, slots, key.p, idx.p,
                                                        S->br * S->bc <= 9 ? uni.p : nullptr, uinfo.p);
  size_t tmp = 0;
  CAMG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, sidx.p, slots, 0, 64, s));
  {
    DBuf<char> t(tmp);
    note_launch();
    CAMG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, key.p, key2.p, idx.p, sidx.p, slots, 0, 64, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
  }
  DBuf<int64_t> head(slots);
  note_launch();
  k_run_heads<<<grid_for(slots, 256), 256, 0, s>>>(key2.p, slots, head.p);
  tmp = 0;
  CAMG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tmp, head.p, head.p, cub::Max(), slots, s));
  {
    DBuf<char> t(tmp);
    note_launch();
    CAMG_CUDA(cub::DeviceScan::InclusiveScan(t.p, tmp, head.p, head.p, cub::Max(), slots, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
  }
  note_launch();
  k_slot_verify<<<grid_for(slots * 32, 256), 256, 0, s>>>(S->mask, S->voff, S->bval, sidx.p, head.p, slots, rep.p);
  DBuf<int64_t> cnt(slots + 1), noff(slots + 1);
  note_launch();
  k_slot_own_groups<<<grid_for(slots, 256), 256, 0, s>>>(S->mask, rep.p, uni.p, slots, S->br * S->bc, cnt.p);
  exclusive_scan_i64(cnt.p, noff.p, slots, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  const int64_t kept = read_i64(noff.p + slots);
  if (kept * 2 > S->ngroups || kept >= (int64_t)1 << 32) return;  // little to share: keep the streaming layout
  DBuf<double> nval((size_t)std::max<int64_t>(kept, 1) * 32);
  note_launch();
  k_slot_compact<<<grid_for(slots * 32, 256), 256, 0, s>>>(S->mask, S->voff, S->bval, rep.p, noff.p, slots,
                                                           S->br * S->bc, nval.p, uni.p, uinfo.p);
  S->vo = dalloc<uint32_t>(slots + 1);
  note_launch();
  k_slot_share<<<grid_for(slots, 256), 256, 0, s>>>(rep.p, noff.p, uni.p, uinfo.p, slots, S->vo, S->desc);
  CAMG_LAUNCH_CHECK();
  CAMG_CUDA(cudaStreamSynchronize(s));
  dfree(S->bval);
  S->bval = nval.release();
  S->ngroups = kept;
  S->dedup = true;
}

static int g_share_override = -1;  // sell_share_override: -1 = CAMG_SELL_DEDUP decides

static bool dedup_enabled() {
  if (g_share_override >= 0) return g_share_override != 0;
  const char* e = getenv("CAMG_SELL_DEDUP");
  return !(e && e[0] == '0');
}

// CAMG_SELL_ALIGN=0: slots in rank order everywhere (no offset-aligned slices)
static bool align_enabled() {
  const char* e = getenv("CAMG_SELL_ALIGN");
  return !(e && e[0] == '0');
}

// CAMG_SELL_USLICE=0: no uniform-slice loop (every slice decodes its slot descriptors)
// 1: uniform-slice loop, one block row per lane; 2 (default): neighbouring uniform slices in pairs, two
// block rows per lane
static int uslice_mode() {
  const char* e = getenv("CAMG_SELL_USLICE");
  return e ? atoi(e) : 2;
}
static bool uslices_enabled() { return uslice_mode() != 0; }
// CAMG_SELL_XGROUPS=0: slices with exception lanes always run by themselves
static bool xgroups_enabled() {
  const char* e = getenv("CAMG_SELL_XGROUPS");
  return !(e && e[0] == '0');
}
// CAMG_SELL_WITEMS=0: the passes walk every slice and the followers' warps skip (no host-made work items)
static bool witems_enabled() {
  const char* e = getenv("CAMG_SELL_WITEMS");
  return !(e && e[0] == '0');
}

template <int BR, int BC>
Sell* build(const Csr* A, int64_t nrows, int64_t ncols_blocked, bool masked, cudaStream_t s,
            const std::vector<int32_t>* order = nullptr) {
  constexpr int BE = BR * BC;
  // natural order: position = block row; with `order`: position t holds
  // block row order[t] (-1 = padding lane) and the diagonal blocks are kept
  const int64_t nbr = order ? (int64_t)order->size() : nrows / BR;
  const int64_t nslices = (nbr + 31) / 32;
  std::unique_ptr<Sell> S(new Sell());
  S->br = BR;
  S->bc = BC;
  S->nbr = nbr;
  S->nslices = nslices;
  S->len = dalloc<uint8_t>(nbr + 1);
  if (order) {
    S->perm = dalloc<int32_t>(nbr + 1);
    CAMG_CUDA(cudaMemcpy(S->perm, order->data(), sizeof(int32_t) * nbr, cudaMemcpyHostToDevice));
    S->dblk = dalloc<double>((size_t)nslices * BE * 32 + 1);
    CAMG_CUDA(cudaMemsetAsync(S->dblk, 0, sizeof(double) * ((size_t)nslices * BE * 32 + 1), s));
  }
  DBuf<int32_t> ovf(1);
  CAMG_CUDA(cudaMemset(ovf.p, 0, sizeof(int32_t)));
  note_launch();
  k_sell_count<BR, BC><<<grid_for(nbr, 256), 256, 0, s>>>(view(A), nbr, ncols_blocked, S->perm, S->len, ovf.p);
  int32_t h_ovf = 0;
  CAMG_CUDA(cudaMemcpy(&h_ovf, ovf.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
  CAMG_CHECK(h_ovf != 2, CAMG_ERR_ARG, "block row with more than 255 blocks");
  CAMG_CHECK(h_ovf != 1, CAMG_ERR_ARG, "entries outside the blocked column range");
  DBuf<int64_t> w(nslices + 1);
  note_launch();
  k_slice_width<<<grid_for(nslices, 256), 256, 0, s>>>(S->len, nbr, nslices, w.p);
  // offset-aligned slots where a slice's rows share their block-column offsets (masked 3x3 mirrors)
  DBuf<int32_t> otab;
  DBuf<uint8_t> wal;
  const bool align = masked && BR * BC <= 9 && BR == BC && !order && align_enabled();
  if (align) {
    otab = DBuf<int32_t>((size_t)nslices * kOffCap + 1);
    wal = DBuf<uint8_t>(nslices + 1);
    note_launch();
    k_slice_offsets<BR, BC><<<grid_for(nslices * 32, 256), 256, 0, s>>>(view(A), nbr, nslices, S->len, otab.p, wal.p);
    note_launch();
    k_apply_aligned<<<grid_for(nslices * 32, 256), 256, 0, s>>>(wal.p, nbr, nslices, w.p, S->len);
    CAMG_LAUNCH_CHECK();
    std::vector<uint8_t> h_wal(nslices);
    CAMG_CUDA(cudaMemcpyAsync(h_wal.data(), wal.p, nslices, cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    for (uint8_t a : h_wal) S->n_aligned += a != 0;
  }
  S->slice_ptr = dalloc<int64_t>(nslices + 1);
  exclusive_scan_i64(w.p, S->slice_ptr, nslices, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  const int64_t slots = read_i64(S->slice_ptr + nslices);
  S->slots = slots;
  masked = masked && BE <= 9;  // slot descriptors hold at most 9 positions (bits 0-35)
  S->masked = masked;
  // slot masks and value offsets
  S->mask = dalloc<unsigned long long>(slots + 1);
  if (masked) {
    CAMG_CUDA(cudaMemsetAsync(S->mask, 0, sizeof(unsigned long long) * (slots + 1), s));
    note_launch();
    k_sell_masks<BR, BC><<<grid_for(nbr, 256), 256, 0, s>>>(view(A), nbr, S->slice_ptr, align ? otab.p : nullptr,
                                                            align ? wal.p : nullptr, S->mask);
  } else {
    std::vector<unsigned long long> full(slots + 1, (BE == 64) ? ~0ull : ((1ull << BE) - 1ull));
    CAMG_CUDA(cudaMemcpy(S->mask, full.data(), sizeof(unsigned long long) * (slots + 1), cudaMemcpyHostToDevice));
  }
  DBuf<int64_t> cnt(slots + 1);
  note_launch();
  k_slot_popc<<<grid_for(slots, 256), 256, 0, s>>>(S->mask, slots, cnt.p);
  if (masked) {
    S->zero = dalloc<double>(32);
    CAMG_CUDA(cudaMemsetAsync(S->zero, 0, sizeof(double) * 32, s));
    S->desc = dalloc<unsigned long long>(slots + 1);
    note_launch();
    k_slot_desc<<<grid_for(slots, 256), 256, 0, s>>>(S->mask, slots, BE, S->desc);
  }
  S->voff = dalloc<int64_t>(slots + 1);
  exclusive_scan_i64(cnt.p, S->voff, slots, s);
  CAMG_CUDA(cudaStreamSynchronize(s));
  const int64_t groups = read_i64(S->voff + slots);
  S->ngroups = groups;
  S->ncb = (A->n_cols + BC - 1) / BC;
  S->bcol = dalloc<int32_t>((size_t)slots * 32);
  S->bval = dalloc<double>((size_t)groups * 32);
  CAMG_CUDA(cudaMemsetAsync(S->bval, 0, sizeof(double) * (size_t)groups * 32, s));
  note_launch();
  k_sell_fill<BR, BC><<<grid_for(nbr, 256), 256, 0, s>>>(view(A), nbr, S->perm, S->slice_ptr, S->mask, S->voff,
                                                         S->bcol, S->bval, S->dblk, align ? otab.p : nullptr,
                                                         align ? wal.p : nullptr,
                                                         std::min<int64_t>(nbr, ncols_blocked / BC));
  CAMG_LAUNCH_CHECK();
  if (masked) {
    note_launch();
    k_slot_linear<<<grid_for(nslices * 32, 256), 256, 0, s>>>(S->slice_ptr, S->len, S->bcol, nbr, nslices, S->desc);
    CAMG_LAUNCH_CHECK();
  }
  if (masked && dedup_enabled()) share_value_groups(S.get(), s);
  if (S->dedup && BR == 3 && BC == 3 && !order && uslices_enabled()) {
    S->uslice = dalloc<uint8_t>(nslices + 1);
    DBuf<unsigned long long> nu_(1);
    CAMG_CUDA(cudaMemsetAsync(nu_.p, 0, sizeof(unsigned long long), s));
    note_launch();
    k_uniform_slices<<<grid_for(nslices, 256), 256, 0, s>>>(S->slice_ptr, S->len, S->desc, nbr, nslices,
                                                            std::min<int64_t>(nbr, ncols_blocked / BC), S->uslice,
                                                            nu_.p);
    CAMG_LAUNCH_CHECK();
    unsigned long long h = 0;
    CAMG_CUDA(cudaMemcpyAsync(&h, nu_.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CAMG_CUDA(cudaStreamSynchronize(s));
    S->n_uslices = (int64_t)h;
    if (h == 0) { dfree(S->uslice); S->uslice = nullptr; }
    if (h > 0 && uslice_mode() >= 2) {
      CAMG_CUDA(cudaMemsetAsync(nu_.p, 0, sizeof(unsigned long long), s));
      note_launch();
      // groups are written to a copy: every thread reads the ungrouped flags
      uint8_t* grouped = dalloc<uint8_t>(nslices + 1);
      CAMG_CUDA(cudaMemcpyAsync(grouped, S->uslice, nslices, cudaMemcpyDeviceToDevice, s));
      k_uniform_groups<<<grid_for(nslices, 256), 256, 0, s>>>(S->slice_ptr, S->desc, S->vo, nslices, S->uslice, grouped,
                                                              nu_.p);
      CAMG_LAUNCH_CHECK();
      CAMG_CUDA(cudaStreamSynchronize(s));
      dfree(S->uslice);
      S->uslice = grouped;
      CAMG_CUDA(cudaMemcpyAsync(&h, nu_.p, sizeof(h), cudaMemcpyDeviceToHost, s));
      CAMG_CUDA(cudaStreamSynchronize(s));
      S->n_upairs = (int64_t)h;
      if (S->n_upairs > 0 && witems_enabled()) {
        if (xgroups_enabled()) {
          S->xpart = dalloc<int32_t>(nslices + 1);
          note_launch();
          k_exc_partner<<<grid_for(nslices, 256), 256, 0, s>>>(S->slice_ptr, S->desc, S->vo, S->uslice, nslices,
                                                               S->xpart);
          CAMG_LAUNCH_CHECK();
          S->h_xpart.resize(nslices);
          CAMG_CUDA(cudaMemcpyAsync(S->h_xpart.data(), S->xpart, sizeof(int32_t) * nslices, cudaMemcpyDeviceToHost, s));
          CAMG_CUDA(cudaStreamSynchronize(s));
        }
        std::vector<int32_t> all(nslices), wd;
        for (int64_t i = 0; i < nslices; ++i) all[i] = (int32_t)i;
        std::vector<uint8_t> wm;
        sell_compact_list(S.get(), all, wm, wd);
        for (uint8_t m : wm) S->n_xgroups += (m & 4) != 0;
        S->n_witems = (int64_t)all.size();
        S->witems = dalloc<int32_t>(all.size() + 1);
        S->wmode = dalloc<uint8_t>(all.size() + 1);
        S->wdist = dalloc<int32_t>(all.size() + 1);
        CAMG_CUDA(cudaMemcpy(S->witems, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice));
        CAMG_CUDA(cudaMemcpy(S->wmode, wm.data(), all.size(), cudaMemcpyHostToDevice));
        CAMG_CUDA(cudaMemcpy(S->wdist, wd.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice));
      }
    }
  }
  // compulsory bytes of one pass: for every row, its blocks' stored values and
  // column (the padding of shorter rows is skipped; linear slots load no
  // column), summed on the device
  DBuf<unsigned long long> acc(3);
  CAMG_CUDA(cudaMemsetAsync(acc.p, 0, 3 * sizeof(unsigned long long), s));
  note_launch();
  k_sell_row_bytes<<<grid_for(nbr, 256), 256, 0, s>>>(S->slice_ptr, S->len, S->mask, masked ? S->desc : nullptr, nbr,
                                                      acc.p);
  CAMG_LAUNCH_CHECK();
  unsigned long long h_acc[3] = {0, 0, 0};
  CAMG_CUDA(cudaMemcpyAsync(h_acc, acc.p, sizeof(h_acc), cudaMemcpyDeviceToHost, s));
  CAMG_CUDA(cudaStreamSynchronize(s));
  const double bytes = (double)h_acc[0];
  const int64_t used = (int64_t)h_acc[1];
  S->used_blocks = used;
  S->pass_bytes = bytes + (double)nbr + 16.0 * (double)(nslices + 1) + 16.0 * (double)slots / 32.0;
  // shared value groups: the rows' column bytes, every kept group once, a descriptor and a group offset per slot
  if (S->dedup)
    S->pass_bytes = (double)h_acc[2] + 256.0 * (double)S->ngroups + (double)nbr + 16.0 * (double)(nslices + 1) +
                    12.0 * (double)slots;
  return S.release();
}

}  // namespace

void sell_share_override(int v) { g_share_override = v; }

Sell* sell_build(const Csr* A, int br, int bc, int64_t nrows, int64_t ncols_blocked, cudaStream_t s, bool masked) {
  CAMG_CHECK(nrows % br == 0 && nrows <= A->n_rows, CAMG_ERR_DIMENSION, "block rows must divide the row range");
  CAMG_CHECK(ncols_blocked % bc == 0 && ncols_blocked <= A->n_cols, CAMG_ERR_DIMENSION,
             "block columns must divide the column range");
#define CAMG_SELL_CASE(R_, C_) \
  if (br == R_ && bc == C_) return build<R_, C_>(A, nrows, ncols_blocked, masked, s);
  CAMG_SELL_CASE(2, 2) CAMG_SELL_CASE(3, 3) CAMG_SELL_CASE(6, 6)
  CAMG_SELL_CASE(3, 6) CAMG_SELL_CASE(6, 3) CAMG_SELL_CASE(2, 3) CAMG_SELL_CASE(3, 2)
#undef CAMG_SELL_CASE
  throw Error(CAMG_ERR_ARG, "unsupported block shape");
}

Sell* sell_build_ordered(const Csr* A, int bs, int64_t nrows, int64_t ncols_blocked, const std::vector<int32_t>& order,
                         cudaStream_t s) {
  CAMG_CHECK(order.size() % 32 == 0, CAMG_ERR_ARG, "ordered SELL positions must fill whole slices");
  CAMG_CHECK(nrows % bs == 0 && nrows <= A->n_rows && ncols_blocked % bs == 0, CAMG_ERR_DIMENSION,
             "block rows must divide the row range");
  if (bs == 1) return build<1, 1>(A, nrows, ncols_blocked, false, s, &order);
  if (bs == 2) return build<2, 2>(A, nrows, ncols_blocked, false, s, &order);
  if (bs == 3) return build<3, 3>(A, nrows, ncols_blocked, false, s, &order);
  if (bs == 6) return build<6, 6>(A, nrows, ncols_blocked, false, s, &order);
  throw Error(CAMG_ERR_ARG, "unsupported node block size");
}

// ---------------------------------------------------------------------------
// SELL row kernels

// fused epilogue of one block row p (acc = its BR row products)
template <int BR, bool ZERO, int MODE>
__device__ __forceinline__ void sell_epilogue(const SellEpi& e, int64_t p, const double* acc) {
#pragma unroll
  for (int r = 0; r < BR; ++r) {
    const int64_t i = p * BR + r;
    if constexpr (MODE == 0) {
      e.y[i] = e.beta != 0.0 ? e.alpha * acc[r] + e.beta * e.y[i] : e.alpha * acc[r];
    } else if constexpr (MODE == 1) {
      const double res = e.b[i] - acc[r];
      if (e.out_r) e.out_r[i] = res;
      if (e.dscale) {
        double d = e.dscale[i] * res;
        if (e.dprev) d = e.c1 * e.dprev[i] + e.c2 * d;
        else if (e.c2 != 1.0) d = e.c2 * d;
        if (e.out_d) e.out_d[i] = d;
        const double xi = (ZERO || !e.x) ? 0.0 : e.x[i];
        const double y = xi + d;
        if (e.out_y) e.out_y[i] = y;
        if (e.out_x) {
          if (e.xmode) {
            const double o = e.x0 ? e.x0[i] : 0.0;
            e.out_x[i] = o + e.coef * (y - o);
          } else {
            e.out_x[i] = xi + e.coef * d;
          }
        }
      }
    } else {
      const double dn = e.d[i] + e.dscale[i] * (e.r[i] - acc[r]);
      e.out_d[i] = dn;
      if (e.out_x) e.out_x[i] = (e.x ? e.x[i] : 0.0) + e.coef * dn;
    }
  }
}

// uniform-slice loops: the epilogue's own-row vectors (b, D^-1, x: compulsory DRAM reads) are prefetched to
// L2 before the slot loop, so the slice does not end on a serial DRAM round trip
// (C5 K pass 0.836 -> 0.814 ms; with the column prefetch of the other slices 0.765 ms)
#ifndef CAMG_US_PREFETCH
#define CAMG_US_PREFETCH 1
#endif
// unroll of the one-row uniform loop: at 2 ptxas serialises the two slots under the 64-register cap
// (0.807 vs 0.814 ms), kept at 1
#ifndef CAMG_US_UNROLL
#define CAMG_US_UNROLL 1
#endif
constexpr int kUsUnroll = CAMG_US_UNROLL;
// column-index prefetch of the non-uniform slices to L1 instead of L2: measured the same
#if CAMG_PF_L1
#define CAMG_BCOL_PF "prefetch.global.L1"
#else
#define CAMG_BCOL_PF "prefetch.global.L2"
#endif
template <int BR, int MODE>
__device__ __forceinline__ void sell_epilogue_prefetch(const SellEpi& e, int64_t p) {
#if CAMG_US_PREFETCH
  const int64_t i = p * BR;
  auto pf = [&](const double* a) {
    if (a) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + i));
  };
  if constexpr (MODE == 0) {
    if (e.beta != 0.0) pf(e.y);
  } else if constexpr (MODE == 1) {
    pf(e.b); pf(e.dscale); pf(e.x); pf(e.dprev);
  } else {
    pf(e.d); pf(e.dscale); pf(e.r); pf(e.x);
  }
#endif
}

// NB neighbouring uniform 3x3 slices (same shared value groups, columns 32 apart) as one work item: each lane
// carries NB block rows (p, p + 32, ...), the slot's lane-uniform values are loaded once for all of them
template <int NB, bool EXC, bool ZERO, int MODE>
__device__ __forceinline__ void uniform_group(const SellView& S, const double* __restrict__ xu, const SellEpi& e,
                                              int64_t p, int32_t c0, uint32_t o0, uint32_t ex, int dn, int width,
                                              int lane) {
  // dn: block rows between the members (32 for neighbouring slices).  EXC: the members are slices with the
  // same exception lanes (a mesh-row period apart); such a lane reads its own dense block (entries 10.. /
  // 20.. of the group) for all its rows
  double acc[NB][3];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
    sell_epilogue_prefetch<3, MODE>(e, p + (int64_t)dn * j);
  }
#pragma unroll 1
  for (int k = 0; k < width; ++k) {
    const int32_t c = __shfl_sync(0xffffffffu, c0, k);
    const uint32_t o = __shfl_sync(0xffffffffu, o0, k);
    CAMG_DCHECK(c >= 0 && (S.ncb == 0 || (int64_t)c + lane + (int64_t)dn * (NB - 1) < S.ncb),
                "uniform group: block column out of range");
    CAMG_DCHECK(S.ngroups == 0 || (int64_t)o < S.ngroups, "uniform group: value group out of range");
    const double* xs = xu + (int64_t)(c + lane) * 3;
    const double* vu = S.bval + (int64_t)o * 32;
    if constexpr (EXC) {
      const uint32_t xk = __shfl_sync(0xffffffffu, ex, k);
      vu += lane == (int)(xk & 0xFFu) ? 10 : (lane == (int)(xk >> 8) ? 20 : 0);
    }
    const double2* v2 = reinterpret_cast<const double2*>(vu);
    double x[NB][3];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double* xj = xs + (int64_t)(3 * dn) * j;
      x[j][0] = __ldg(xj); x[j][1] = __ldg(xj + 1); x[j][2] = __ldg(xj + 2);
    }
    const double2 a = __ldg(v2), b = __ldg(v2 + 1), cc = __ldg(v2 + 2), d = __ldg(v2 + 3);
    const double v8 = __ldg(vu + 8);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      acc[j][0] = fma(a.x, x[j][0], acc[j][0]); acc[j][0] = fma(a.y, x[j][1], acc[j][0]);
      acc[j][0] = fma(b.x, x[j][2], acc[j][0]);
      acc[j][1] = fma(b.y, x[j][0], acc[j][1]); acc[j][1] = fma(cc.x, x[j][1], acc[j][1]);
      acc[j][1] = fma(cc.y, x[j][2], acc[j][1]);
      acc[j][2] = fma(d.x, x[j][0], acc[j][2]); acc[j][2] = fma(d.y, x[j][1], acc[j][2]);
      acc[j][2] = fma(v8, x[j][2], acc[j][2]);
    }
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) sell_epilogue<3, ZERO, MODE>(e, p + (int64_t)dn * j, acc[j]);
}

template <int BR, int BC, bool ZERO, bool SPLIT, int MODE, bool MASKED, bool DEDUP = false>
__global__ void __launch_bounds__(kSellThreads, (MASKED ? (DEDUP ? CAMG_DEDUP_MINB : CAMG_MASKED_MINB) : (BR * BC >= 18 ? CAMG_BIG_MINB : 6)) * 256 / kSellThreads) k_sell_row(SellView S, const double* __restrict__ xu,
                                                  const double* __restrict__ xl, int64_t split_blocks,
                                                  SellEpi e) {
  CAMG_PDL_ENTRY();
  // MODE 0: spmv y = alpha*acc + beta*y
  // MODE 1: residual / fused Jacobi epilogue (RowEpi semantics)
  // MODE 2: extra Jacobi sweep: d_new = d + dinv*(r - acc), optional x update
  constexpr int BE = BR * BC;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < S.nwork; w += nwarps) {
    const int64_t s = S.slist ? (int64_t)S.slist[w] : w;
    const int64_t p = s * 32 + lane;
    const bool active = p < S.nbr;
    double acc[BR];
#pragma unroll
    for (int r = 0; r < BR; ++r) acc[r] = 0.0;
    if (!ZERO) {
      const int n = active ? S.len[p] : 0;
      const int64_t base = S.slice_ptr[s];
      auto load_x = [&](int64_t slot, double* xv, uint32_t lin = 0) {
        const int32_t bc = lin ? (int32_t)(lin - 1) + lane : __ldcs(S.bcol + slot * 32 + lane);
        CAMG_DCHECK(bc >= 0 && (S.ncb == 0 || bc < S.ncb), "sell block column out of range");
        const double* xs;
        if (!SPLIT || bc < split_blocks) xs = xu + (int64_t)bc * BC;
        else xs = xl ? xl + ((int64_t)bc - split_blocks) * BC : nullptr;
#pragma unroll
        for (int c = 0; c < BC; ++c) xv[c] = xs ? __ldg(xs + c) : 0.0;
      };
      if constexpr (!MASKED) {
        // full blocks: addresses follow from the slot index alone
        for (int k = 0; k < n; ++k) {
          const int64_t slot = base + k;
          double xv[BC];
          load_x(slot, xv);
          const double* v = S.bval + slot * (BE * 32) + lane;
#pragma unroll
          for (int q = 0; q < BE; ++q) acc[q / BC] = fma(__ldcs(v + q * 32), xv[q % BC], acc[q / BC]);
        }
      } else if constexpr (BE <= 9) {
        // masked slots: the slice's slot descriptors arrive in one coalesced
        // load and are broadcast by shuffles; the value offset is a running sum
        const int width = (int)(S.slice_ptr[s + 1] - base);
        const uint64_t m0 = lane < width ? __ldg(S.desc + base + lane) : 0ull;
        const uint64_t m1 = lane + 32 < width ? __ldg(S.desc + base + 32 + lane) : 0ull;
        auto slot_desc = [&](int k) -> uint64_t {
          return k < 32 ? __shfl_sync(0xffffffffu, m0, k)
                        : (k < 64 ? __shfl_sync(0xffffffffu, m1, k - 32) : __ldg(S.desc + base + k));
        };
        if constexpr (DEDUP) {
          // shared value groups: every slot names the first group of its
          // copy: its union-pattern groups, or, for a slot whose lanes all hold
          // the same block (bits 60-61 = 1) or all but one or two of them
          // (= 2: slices that straddle a mesh row), ONE group with the dense
          // BR x BC block(s), loaded as broadcasts.  An absent position enters
          // as fma(0, x, acc), as in the other layouts.
          const uint32_t o0 = lane < width ? __ldg(S.vo + base + lane) : 0u;
          if constexpr (BE == 9) {
            // uniform slice: all slots linear and lane-uniform, columns in xu: no decoding, no branches
            const int us = S.uslice ? S.uslice[s] : 0;
            if (us >= 3) {
              // group of two or three uniform slices (leader us = 3 / 5; followers 4 / 6 at distance 1 / 2),
              // all in this launch's list: the leader's warp carries the group, NB block rows per lane
              int dist = us == 4 ? 1 : (us == 6 ? 2 : 0);
              int gsz;
              bool whole = true;
              if (S.wmode) {
                // work items: the host dropped the followers and decided which leaders run their group
                gsz = S.wmode[w];
                whole = gsz >= 2;
                dist = 0;
              } else {
                gsz = S.uslice[s - dist] == 5 ? 3 : 2;
                if (S.slist) {
                  whole = w - dist >= 0 && w - dist + gsz <= S.nwork;
                  for (int j = 0; whole && j < gsz; ++j) whole = S.slist[w - dist + j] == (int32_t)(s - dist + j);
                }
              }
              if (whole && dist) continue;
              if (whole) {
                const int32_t c0 = (int32_t)((uint32_t)(m0 >> 36) & 0xFFFFFFu) - 1;
                if (gsz == 2) uniform_group<2, false, ZERO, MODE>(S, xu, e, p, c0, o0, 0u, 32, width, lane);
                else uniform_group<3, false, ZERO, MODE>(S, xu, e, p, c0, o0, 0u, 32, width, lane);
                continue;
              }
            }
            if (us == 2) {
              // uniform but for one or two lanes in some slots (a slice across the end of a mesh row: its two
              // boundary nodes): those lanes read their own dense block at entries 10.. / 20.. of the group
              const int32_t c0 = (int32_t)((uint32_t)(m0 >> 36) & 0xFFFFFFu) - 1;
              const uint32_t ex = ((unsigned)(m0 >> 60) & 3u) == 2u ? (uint32_t)(m0 & 0xFFFFull) : 0xFFFFu;
              if (S.wmode && (S.wmode[w] & 3) >= 2) {
                // work item: a group of such slices a period apart (same lanes, same groups)
                const int dn = 32 * S.wdist[w];
                uniform_group<2, true, ZERO, MODE>(S, xu, e, p, c0, o0, ex, dn, width, lane);  // pairs only: registers
                continue;
              }
              sell_epilogue_prefetch<BR, MODE>(e, p);
#pragma unroll 1
              for (int k = 0; k < width; ++k) {
                const int32_t c = __shfl_sync(0xffffffffu, c0, k);
                const uint32_t o = __shfl_sync(0xffffffffu, o0, k);
                const uint32_t x = __shfl_sync(0xffffffffu, ex, k);
                CAMG_DCHECK(c >= 0 && (S.ncb == 0 || (int64_t)c + lane < S.ncb) &&
                                (S.ngroups == 0 || (int64_t)o < S.ngroups),
                            "uniform slice (exception lanes): column or value group out of range");
                const double* xs = xu + (int64_t)(c + lane) * 3;
                const int sh = lane == (int)(x & 0xFFu) ? 10 : (lane == (int)(x >> 8) ? 20 : 0);
                const double* vu = S.bval + (int64_t)o * 32 + sh;
                const double2* v2 = reinterpret_cast<const double2*>(vu);
                const double x0 = __ldg(xs), x1 = __ldg(xs + 1), x2 = __ldg(xs + 2);
                const double2 a = __ldg(v2), b = __ldg(v2 + 1), cc = __ldg(v2 + 2), d = __ldg(v2 + 3);
                const double v8 = __ldg(vu + 8);
                acc[0] = fma(a.x, x0, acc[0]); acc[0] = fma(a.y, x1, acc[0]); acc[0] = fma(b.x, x2, acc[0]);
                acc[1] = fma(b.y, x0, acc[1]); acc[1] = fma(cc.x, x1, acc[1]); acc[1] = fma(cc.y, x2, acc[1]);
                acc[2] = fma(d.x, x0, acc[2]); acc[2] = fma(d.y, x1, acc[2]); acc[2] = fma(v8, x2, acc[2]);
              }
              sell_epilogue<BR, ZERO, MODE>(e, p, acc);
              continue;
            }
            if (us) {
              const int32_t c0 = (int32_t)((uint32_t)(m0 >> 36) & 0xFFFFFFu) - 1;  // slot `lane`: first column
              sell_epilogue_prefetch<BR, MODE>(e, p);
#pragma unroll kUsUnroll
              for (int k = 0; k < width; ++k) {
                const int32_t c = __shfl_sync(0xffffffffu, c0, k);
                const uint32_t o = __shfl_sync(0xffffffffu, o0, k);
                CAMG_DCHECK(c >= 0 && (S.ncb == 0 || (int64_t)c + lane < S.ncb) &&
                                (S.ngroups == 0 || (int64_t)o < S.ngroups),
                            "uniform slice: column or value group out of range");
                const double* xs = xu + (int64_t)(c + lane) * 3;
                const double2* v2 = reinterpret_cast<const double2*>(S.bval + (int64_t)o * 32);
                const double x0 = __ldg(xs), x1 = __ldg(xs + 1), x2 = __ldg(xs + 2);
                const double2 a = __ldg(v2), b = __ldg(v2 + 1), cc = __ldg(v2 + 2), d = __ldg(v2 + 3);
                const double v8 = __ldg(reinterpret_cast<const double*>(v2) + 8);
                acc[0] = fma(a.x, x0, acc[0]); acc[0] = fma(a.y, x1, acc[0]); acc[0] = fma(b.x, x2, acc[0]);
                acc[1] = fma(b.y, x0, acc[1]); acc[1] = fma(cc.x, x1, acc[1]); acc[1] = fma(cc.y, x2, acc[1]);
                acc[2] = fma(d.x, x0, acc[2]); acc[2] = fma(d.y, x1, acc[2]); acc[2] = fma(v8, x2, acc[2]);
              }
              sell_epilogue<BR, ZERO, MODE>(e, p, acc);
              continue;
            }
          }
          const uint32_t o1 = lane + 32 < width ? __ldg(S.vo + base + 32 + lane) : 0u;
#if CAMG_US_PREFETCH
          // other slices (mesh-row ends, boundaries, interface rows): the column indices of the non-linear
          // slots -- one 128-byte line per slot, a compulsory DRAM read ahead of every x gather -- and the
          // epilogue's vectors are prefetched now, all at once, instead of one DRAM round trip per slot
          if (lane < width && !((uint32_t)(m0 >> 36) & 0xFFFFFFu))
            asm volatile(CAMG_BCOL_PF " [%0];" ::"l"(S.bcol + (base + lane) * 32));
          if (lane + 32 < width && !((uint32_t)(m1 >> 36) & 0xFFFFFFu))
            asm volatile(CAMG_BCOL_PF " [%0];" ::"l"(S.bcol + (base + 32 + lane) * 32));
          if (active) sell_epilogue_prefetch<BR, MODE>(e, p);
#endif
          // x of slot k (a linear slot has a block in every lane: k < n for all 32)
          auto fetch_x = [&](int k, uint64_t mk, double* xo) {
            const uint32_t lin = (uint32_t)(mk >> 36) & 0xFFFFFFu;
            if (lin && (!SPLIT || (int64_t)lin + 30 < split_blocks)) {
              const double* xs = xu + ((int64_t)(lin - 1) + lane) * BC;
#pragma unroll
              for (int c = 0; c < BC; ++c) xo[c] = __ldg(xs + c);
            } else if (lin || k < n) {
              load_x(base + k, xo, lin);
            }
          };
          for (int k = 0; k < width; ++k) {
            const uint32_t o = k < 32 ? __shfl_sync(0xffffffffu, o0, k)
                                      : (k < 64 ? __shfl_sync(0xffffffffu, o1, k - 32) : __ldg(S.vo + base + k));
            double xv[BC];
            const uint64_t m = slot_desc(k);
            if (!((uint32_t)(m >> 36) & 0xFFFFFFu) && k >= n) continue;
            fetch_x(k, m, xv);
            CAMG_DCHECK(S.ngroups == 0 || (int64_t)o < S.ngroups,
                        "sell value group out of range");
            double val[BE];
            const unsigned kind = (unsigned)(m >> 60) & 3u;
            if (kind) {
              // kind 1: one dense block for all lanes (broadcast loads); kind 2:
              // the same with one or two exception lanes, whose blocks follow
              // in the group (entry 9 names the lanes)
              const double* vu = S.bval + (int64_t)o * 32;
              if (kind == 2)  // exception lanes: descriptor bits 0-7 and 8-15 (0xFF: none)
                vu += lane == (int)(m & 0xFF) ? 10 : (lane == (int)((m >> 8) & 0xFF) ? 20 : 0);
              if constexpr (BE == 9) {
                const double2* v2 = reinterpret_cast<const double2*>(vu);
                const double2 a = __ldg(v2), b = __ldg(v2 + 1), c = __ldg(v2 + 2), d = __ldg(v2 + 3);
                val[0] = a.x; val[1] = a.y; val[2] = b.x; val[3] = b.y;
                val[4] = c.x; val[5] = c.y; val[6] = d.x; val[7] = d.y;
                val[8] = __ldg(vu + 8);
              } else {
#pragma unroll
                for (int q = 0; q < BE; ++q) val[q] = __ldg(vu + q);
              }
            } else {
              const double* v = S.bval + (int64_t)o * 32 + lane;
#if CAMG_DEDUP_NUDENSE
#pragma unroll
              for (int q = 0; q < BE; ++q) val[q] = __ldg(v + q * 32);
#else
              // only the slot's union pattern is stored (nibble q of the
              // descriptor = 1 + rank of position q; 0 = absent: the zero group)
#pragma unroll
              for (int q = 0; q < BE; ++q) {
                const int g = (int)((m >> (4 * q)) & 15u);
                val[q] = __ldg(g ? v + (g - 1) * 32 : S.zero + lane);
              }
#endif
            }
#pragma unroll
            for (int q = 0; q < BE; ++q) acc[q / BC] = fma(val[q], xv[q % BC], acc[q / BC]);
          }
        } else {
          // the slice's values start at group voff[base]; slots follow in order
          const double* v = S.bval + __ldg(S.voff + base) * 32 + lane;
          for (int k = 0; k < width; ++k) {
            const uint64_t m = slot_desc(k);
            if (k < n) {
              double xv[BC];
              load_x(base + k, xv, (uint32_t)(m >> 36) & 0xFFFFFFu);
              // absent positions load the zero group (L1/L2-resident): all BE
              // loads are unconditional and independent, nothing but the loaded
              // values stays live across them, and an absent position enters as
              // fma(0, x, acc) -- the same operations (and results) as the
              // full-block kernel on its stored zeros
              double val[BE];
#pragma unroll
              for (int q = 0; q < BE; ++q) {
                const int g = (int)((m >> (4 * q)) & 15u);
                CAMG_DCHECK(!g || S.ngroups == 0 || (v - S.bval) / 32 + g - 1 < S.ngroups,
                            "sell value group out of range");
                val[q] = __ldcs(g ? v + (g - 1) * 32 : S.zero + lane);
              }
#pragma unroll
              for (int q = 0; q < BE; ++q) acc[q / BC] = fma(val[q], xv[q % BC], acc[q / BC]);
            }
            v += (int)(m >> 60) * 32;
          }
        }
      }
    }
    if (!active) continue;
    sell_epilogue<BR, ZERO, MODE>(e, p, acc);
  }
}

// Small matrices (few slices) lose a quarter of the time to wave
// quantisation with one warp per slice; this variant gives each block row to
// a lane pair (even lane: first half of its slots, odd lane: second half,
// deterministic pair reduction), i.e. two work units per slice.
template <int BR, int BC, bool ZERO, bool SPLIT, int MODE, int LPR>
__global__ void __launch_bounds__(256, BR * BC >= 18 ? CAMG_BIG_MINB : 0) k_sell_row2(SellView S, const double* __restrict__ xu,
                                                   const double* __restrict__ xl, int64_t split_blocks,
                                                   SellEpi e) {
  CAMG_PDL_ENTRY();
  constexpr int BE = BR * BC;
  const int lane = threadIdx.x & 31;
  const int part = lane & (LPR - 1);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t hs = warp; hs < LPR * S.nwork; hs += nwarps) {
    const int64_t s = S.slist ? (int64_t)S.slist[hs / LPR] : hs / LPR;
    const int pl = (int)(hs % LPR) * (32 / LPR) + lane / LPR;
    const int64_t p = s * 32 + pl;
    const bool active = p < S.nbr;
    double acc[BR];
#pragma unroll
    for (int r = 0; r < BR; ++r) acc[r] = 0.0;
    if (!ZERO) {
      const int n = active ? S.len[p] : 0;
      const int chunk = (n + LPR - 1) / LPR;
      const int k0 = min(n, part * chunk), k1 = min(n, k0 + chunk);
      const int64_t base = S.slice_ptr[s];
      for (int k = k0; k < k1; ++k) {
        const int64_t slot = base + k;
        const int32_t bc = __ldcs(S.bcol + slot * 32 + pl);
        const double* xs;
        if (!SPLIT || bc < split_blocks) xs = xu + (int64_t)bc * BC;
        else xs = xl ? xl + ((int64_t)bc - split_blocks) * BC : nullptr;
        double xv[BC];
#pragma unroll
        for (int c = 0; c < BC; ++c) xv[c] = xs ? __ldg(xs + c) : 0.0;
        const double* v = S.bval + slot * (BE * 32) + pl;
#pragma unroll
        for (int q = 0; q < BE; ++q) acc[q / BC] = fma(__ldcs(v + q * 32), xv[q % BC], acc[q / BC]);
      }
    }
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1)
#pragma unroll
      for (int r = 0; r < BR; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    if (!active || part) continue;
    sell_epilogue<BR, ZERO, MODE>(e, p, acc);
  }
}

// below this many slices four lanes share a block row (CAMG_SELL_QUAD sets it)
static int64_t quad_slices() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("CAMG_SELL_QUAD");
    v = e ? atoll(e) : kSellQuadSlices;
  }
  return v;
}

// grid cap of the one-lane-per-row kernels in CTAs per SM (CAMG_SELL_CTAS):
// 64 (~3 slices per warp on the C5 fine level, short CTAs that rebalance
// the per-SM load) beats 16 (~13 slices per warp): fine predictor pass
// 2.154 -> 2.113 ms, V-cycle 20.0 -> 19.8 ms; 4 (persistent), 8, 32, 48, 96,
// 128 measured in between or slower
static int64_t sell_ctas_per_sm() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("CAMG_SELL_CTAS");
    v = e ? atoll(e) : 64;
  }
  return v;
}

// read per call (build and capture time only): tests switch it per case
static int64_t pair_slices() {
  const char* e = getenv("CAMG_SELL_PAIR");
  return e ? atoll(e) : kSellPairSlices;
}

static int64_t quad_min_blocks() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("CAMG_SELL_QUAD_BLOCKS");
    v = e ? atoll(e) : kSellQuadBlocks;
  }
  return v;
}

template <int BR, int BC>
static void launch_blk(const Sell* S, int mode, bool zero, const double* xu, const double* xl, int64_t split,
                       const SellEpi& e, cudaStream_t st, const int32_t* slist, int64_t nlist, const uint8_t* lmode,
                       const int32_t* ldist) {
  SellView v{S->slice_ptr, S->len, S->bcol, S->bval, S->mask, S->voff, S->desc, S->zero, S->nbr, S->nslices};
  v.ncb = S->ncb;
  v.ngroups = S->masked ? S->ngroups : 0;
  v.vo = S->vo;
  // uniform slices read xu only: their columns lie below nbr, so any split at or above it is safe
  v.uslice = (split < 0 || split / BC >= S->nbr) ? S->uslice : nullptr;
  v.slist = slist;
  v.nwork = slist ? nlist : S->nslices;
  if (v.uslice && !zero) {
    if (!slist && S->witems) {
      v.slist = S->witems;
      v.nwork = S->n_witems;
      v.wmode = S->wmode;
      v.wdist = S->wdist;
    } else if (slist) {
      v.wmode = lmode;
      v.wdist = ldist;
    }
  }
  CAMG_CHECK(!(slist && lmode && !v.wmode) && !(v.wmode && !v.wdist), CAMG_ERR_NATIVE,
             "work-item list passed to a pass that cannot run uniform-slice groups");
  if (v.nwork <= 0) return;
  const int64_t nw = v.nwork;
  // rows with many blocks (R = P^T: ~117 6x3 blocks per coarse node) split
  // over four lanes, short ones over two
  const bool long_rows = S->nbr > 0 && S->used_blocks >= quad_min_blocks() * S->nbr;
  const unsigned grid = grid_for(nw * 32, kSellThreads, int64_t(kNumSMs) * sell_ctas_per_sm() * 256 / kSellThreads);
  const bool sp = split >= 0;
  const int64_t sb = sp ? split / BC : 0;
  note_launch();
#define CAMG_SELL_LAUNCH(Z, SP, M)                                                           \
  do {                                                                                       \
    if (S->masked && S->dedup) launch_k(k_sell_row<BR, BC, Z, SP, M, true, true>, grid, kSellThreads, 0, st, v, xu, xl, sb, e); \
    else if (S->masked) launch_k(k_sell_row<BR, BC, Z, SP, M, true>, grid, kSellThreads, 0, st, v, xu, xl, sb, e);         \
    else if (nw < quad_slices() || (nw < pair_slices() && long_rows))                       \
      launch_k(k_sell_row2<BR, BC, Z, SP, M, 4>, grid_for(nw * 128, 256, int64_t(kNumSMs) * 16), 256, 0, st, \
               v, xu, xl, sb, e);                                                            \
    else if (nw < pair_slices())                                                             \
      launch_k(k_sell_row2<BR, BC, Z, SP, M, 2>, grid_for(nw * 64, 256, int64_t(kNumSMs) * 16), 256, 0, st, \
               v, xu, xl, sb, e);                                                            \
    else launch_k(k_sell_row<BR, BC, Z, SP, M, false>, grid, kSellThreads, 0, st, v, xu, xl, sb, e);                  \
  } while (0)
  if (mode == 0) {
    if (sp) CAMG_SELL_LAUNCH(false, true, 0); else CAMG_SELL_LAUNCH(false, false, 0);
  } else {
    if constexpr (BR == BC) {
      if (mode == 1) {
        if (zero) CAMG_SELL_LAUNCH(true, false, 1);
        else if (sp) CAMG_SELL_LAUNCH(false, true, 1);
        else CAMG_SELL_LAUNCH(false, false, 1);
      } else {
        if (sp) CAMG_SELL_LAUNCH(false, true, 2); else CAMG_SELL_LAUNCH(false, false, 2);
      }
    } else {
      throw Error(CAMG_ERR_NATIVE, "smoother modes need square blocks");
    }
  }
#undef CAMG_SELL_LAUNCH
  CAMG_LAUNCH_CHECK();
}

void sell_compact_list(const Sell* S, std::vector<int32_t>& list, std::vector<uint8_t>& mode,
                       std::vector<int32_t>& dist) {
  mode.assign(list.size(), 0);
  dist.assign(list.size(), 1);
  if (!S->uslice || S->n_upairs == 0) return;
  if (S->h_uslice.empty()) {
    Sell* M = const_cast<Sell*>(S);
    M->h_uslice.resize(S->nslices);
    CAMG_CUDA(cudaMemcpy(M->h_uslice.data(), S->uslice, S->nslices, cudaMemcpyDeviceToHost));
  }
  const std::vector<uint8_t>& us = S->h_uslice;
  const std::vector<int32_t>& xp = S->h_xpart;
  // slices with exception lanes: chains s, s + d, s + 2d, ... (d = xp[s]) cut into threes and twos, a group
  // formed only of members that are all in the list; taken[s] = 1: s runs inside an earlier entry's group
  std::vector<uint8_t> in_list, taken;
  if (!xp.empty()) {
    in_list.assign(S->nslices, 0);
    taken.assign(S->nslices, 0);
    for (int32_t s : list) in_list[s] = 1;
  }
  std::vector<int32_t> out, od;
  std::vector<uint8_t> om;
  out.reserve(list.size());
  om.reserve(list.size());
  od.reserve(list.size());
  const size_t n = list.size();
  for (size_t w = 0; w < n;) {
    const int32_t s = list[w];
    const int u = us[s];
    if (u == 2 && !xp.empty()) {
      if (taken[s]) { ++w; continue; }
      const int64_t d = xp[s];
      int g = 1;
      if (d > 0) {
        // members available after s: in the list, not yet taken, and linked by the same period
        int64_t t = s;
        // (pairs: three rows per lane with the per-lane value pointer do not fit the pass's 64 registers)
        while (g < 2 && xp[t] == d && t + d < S->nslices && in_list[t + d] && !taken[t + d] && us[t + d] == 2) {
          t += d;
          ++g;
        }
      }
      if (g >= 2) {
        for (int j = 1; j < g; ++j) taken[s + j * d] = 1;
        out.push_back(s);
        om.push_back((uint8_t)(g | 4));
        od.push_back((int32_t)d);
      } else {
        out.push_back(s);
        om.push_back(0);
        od.push_back(1);
      }
      ++w;
      continue;
    }
    const int g = u == 3 ? 2 : (u == 5 ? 3 : 0);
    bool whole = g && w + g <= n;
    for (int j = 1; whole && j < g; ++j) whole = list[w + j] == s + j;
    out.push_back(s);
    om.push_back(whole ? (uint8_t)g : 0);
    od.push_back(1);
    w += whole ? g : 1;  // a follower without its leader in front stays an entry of its own
  }
  list.swap(out);
  mode.swap(om);
  dist.swap(od);
}

void sell_launch(const Sell* S, int mode, bool zero, const double* xu, const double* xl, int64_t split,
                 const SellEpi& e, cudaStream_t st, const int32_t* slist, int64_t nlist, const uint8_t* lmode,
                 const int32_t* ldist) {
#define CAMG_SELL_CASE(R_, C_) \
  if (S->br == R_ && S->bc == C_) \
    return launch_blk<R_, C_>(S, mode, zero, xu, xl, split, e, st, slist, nlist, lmode, ldist);
  CAMG_SELL_CASE(2, 2) CAMG_SELL_CASE(3, 3) CAMG_SELL_CASE(6, 6)
  CAMG_SELL_CASE(3, 6) CAMG_SELL_CASE(6, 3) CAMG_SELL_CASE(2, 3) CAMG_SELL_CASE(3, 2)
#undef CAMG_SELL_CASE
  throw Error(CAMG_ERR_NATIVE, "bad SELL block shape");
}

double sell_pass_bytes(const Sell* S) { return S->pass_bytes; }

// lanes per block row of a full pass (the choice launch_blk makes for
// nwork = nslices): 1 = one lane per block row, 2 = lane pairs, 4 = quads
int sell_lanes(const Sell* S) {
  const int64_t nw = S->nslices;
  const bool long_rows = S->nbr > 0 && S->used_blocks >= quad_min_blocks() * S->nbr;
  if (S->masked) return 1;
  if (nw < quad_slices() || (nw < pair_slices() && long_rows)) return 4;
  if (nw < pair_slices()) return 2;
  return 1;
}

// ---------------------------------------------------------------------------
// Multicolour Gauss-Seidel on a colour-ordered SELL (slices [s0, s1) hold the
// block rows of one colour; rows of one colour share no entries, so each lane
// updates its node in place).  Within a node the BR DOFs are visited in order
// (backward: reverse order): every off-node product and the node's own block
// use the values from before this pass (acc), and the DOFs already updated
// in this pass enter through the stored diagonal block:
//   dv_d = dinv_d * (b_d - acc_d - sum_{e before d} K_de dv_e),  y_d += dv_d
// which is the sequential Gauss-Seidel update of SSOR (smoothers.py:155-164)
// on the colour-permuted matrix.  Columns >= split read xl (lambda; null = 0).
template <int BR, bool FWD, bool ZERO>
__global__ void __launch_bounds__(256) k_sell_gs(SellView S, const int32_t* __restrict__ perm,
                                                 const double* __restrict__ dblk, int64_t s0, int64_t s1,
                                                 const double* __restrict__ xl, int64_t split_blocks,
                                                 const double* __restrict__ b, const double* __restrict__ dinv,
                                                 double* y) {
  CAMG_PDL_ENTRY();
  constexpr int BE = BR * BR;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // no address this kernel writes is read by another lane (same-colour rows
  // are uncoupled), so the read-only path is safe for y
  const double* __restrict__ yr = y;
  for (int64_t s = s0 + warp; s < s1; s += nwarps) {
    const int64_t t = s * 32 + lane;
    const int32_t p = perm[t];
    double acc[BR];
#pragma unroll
    for (int r = 0; r < BR; ++r) acc[r] = 0.0;
    if (!ZERO) {
      const int n = S.len[t];
      const int64_t base = S.slice_ptr[s];
      for (int k = 0; k < n; ++k) {
        const int64_t slot = base + k;
        const int32_t bc = __ldcs(S.bcol + slot * 32 + lane);
        const double* xs;
        if (bc < split_blocks) xs = yr + (int64_t)bc * BR;
        else xs = xl ? xl + ((int64_t)bc - split_blocks) * BR : nullptr;
        double xv[BR];
#pragma unroll
        for (int c = 0; c < BR; ++c) xv[c] = xs ? __ldg(xs + c) : 0.0;
        const double* v = S.bval + slot * (BE * 32) + lane;
#pragma unroll
        for (int q = 0; q < BE; ++q) acc[q / BR] = fma(__ldcs(v + q * 32), xv[q % BR], acc[q / BR]);
      }
    }
    if (p < 0) continue;
    const double* db = dblk + s * (BE * 32) + lane;
    double dv[BR];
#pragma unroll
    for (int dd = 0; dd < BR; ++dd) {
      const int d = FWD ? dd : BR - 1 - dd;
      double corr = 0.0;
#pragma unroll
      for (int ee = 0; ee < dd; ++ee) {
        const int e = FWD ? ee : BR - 1 - ee;
        corr = fma(__ldg(db + (d * BR + e) * 32), dv[e], corr);
      }
      const int64_t i = (int64_t)p * BR + d;
      dv[d] = __ldg(dinv + i) * ((__ldg(b + i) - acc[d]) - corr);
    }
#pragma unroll
    for (int d = 0; d < BR; ++d) {
      const int64_t i = (int64_t)p * BR + d;
      y[i] = (ZERO ? 0.0 : y[i]) + dv[d];
    }
  }
}

template <int BR>
static void launch_gs(const Sell* S, int64_t s0, int64_t s1, bool fwd, bool zero, const double* xl, int64_t split,
                      const double* b, const double* dinv, double* y, cudaStream_t st) {
  SellView v{S->slice_ptr, S->len, S->bcol, S->bval, S->mask, S->voff, S->desc, S->zero, S->nbr, S->nslices};
  const unsigned grid = grid_for((s1 - s0) * 32, 256, int64_t(kNumSMs) * 16);
  const int64_t sb = split / BR;
  note_launch();
  if (zero) {
    if (fwd) launch_k(k_sell_gs<BR, true, true>, grid, 256, 0, st, v, S->perm, S->dblk, s0, s1, xl, sb, b, dinv, y);
    else launch_k(k_sell_gs<BR, false, true>, grid, 256, 0, st, v, S->perm, S->dblk, s0, s1, xl, sb, b, dinv, y);
  } else {
    if (fwd) launch_k(k_sell_gs<BR, true, false>, grid, 256, 0, st, v, S->perm, S->dblk, s0, s1, xl, sb, b, dinv, y);
    else launch_k(k_sell_gs<BR, false, false>, grid, 256, 0, st, v, S->perm, S->dblk, s0, s1, xl, sb, b, dinv, y);
  }
  CAMG_LAUNCH_CHECK();
}

void sell_gs_launch(const Sell* S, int64_t s0, int64_t s1, bool fwd, bool zero, const double* xl, int64_t split,
                    const double* b, const double* dinv, double* y, cudaStream_t st) {
  if (s1 <= s0) return;
  CAMG_CHECK(S->perm && S->dblk && S->br == S->bc, CAMG_ERR_NATIVE, "not a colour-ordered SELL");
  switch (S->br) {
    case 1: return launch_gs<1>(S, s0, s1, fwd, zero, xl, split, b, dinv, y, st);
    case 2: return launch_gs<2>(S, s0, s1, fwd, zero, xl, split, b, dinv, y, st);
    case 3: return launch_gs<3>(S, s0, s1, fwd, zero, xl, split, b, dinv, y, st);
    case 6: return launch_gs<6>(S, s0, s1, fwd, zero, xl, split, b, dinv, y, st);
    default: throw Error(CAMG_ERR_NATIVE, "bad SELL block size");
  }
}

}  // namespace camg

using namespace camg;

extern "C" int camg_csr_attach_blocks(camg_csr* A, int bs, int64_t nrows) {
  return guarded([&] {
    Csr* M = A->m;
    delete M->sell;
    M->sell = nullptr;
    if (bs <= 1 || nrows <= 0) return;
    const char* env = getenv("CAMG_SELL_MASKED");
    // masked slots (3x3 / 2x2 blocks) stream 16% fewer bytes on hex8
    // stencils: C5 merged SpMV 2.58 -> 2.23 ms, V-cycle 23.3 -> 22.1 ms
    // (scripts/sell_ab.py); CAMG_SELL_MASKED=0 keeps full blocks
    // (only where the one-lane-per-row kernel runs: smaller mirrors split
    // rows over lane pairs, which need the full-block layout)
    const bool masked = !(env && env[0] == '0') && (nrows / bs + 31) / 32 >= pair_slices();
    M->sell = sell_build(M, bs, bs, nrows, M->n_cols - M->n_cols % bs, 0, masked);
  });
}

extern "C" int camg_csr_attach_rect_blocks(camg_csr* A, int br, int bc, int64_t nrows, int64_t ncols_blocked) {
  return guarded([&] {
    Csr* M = A->m;
    delete M->sell;
    M->sell = nullptr;
    if (br <= 0 || bc <= 0 || nrows <= 0) return;
    M->sell = sell_build(M, br, bc, nrows, ncols_blocked, 0, false);
  });
}

__global__ void k_slot_stats(const unsigned long long* __restrict__ desc, int64_t slots, unsigned long long* __restrict__ out) {
  unsigned long long u = 0, l = 0, ul = 0, x = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < slots; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = desc[i];
    const unsigned kind = (unsigned)(d >> 60) & 3u;
    const bool li = ((d >> 36) & 0xFFFFFFull) != 0;
    u += kind == 1; l += li; ul += kind == 1 && li; x += kind == 2;
  }
  for (int o = 16; o > 0; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    l += __shfl_xor_sync(0xffffffffu, l, o);
    ul += __shfl_xor_sync(0xffffffffu, ul, o);
    x += __shfl_xor_sync(0xffffffffu, x, o);
  }
  if ((threadIdx.x & 31) == 0) { atomicAdd(out, u); atomicAdd(out + 1, l); atomicAdd(out + 2, ul); atomicAdd(out + 3, x); }
}

// slots of a masked mirror: out[5] = {slots, lane-uniform, linear, both, uniform with one or two exception lanes}
extern "C" int camg_csr_slot_stats(const camg_csr* A, int64_t* out) {
  return guarded([&] {
    const Sell* S = A->m->sell;
    for (int i = 0; i < 5; ++i) out[i] = 0;
    if (!S || !S->desc) return;
    DBuf<unsigned long long> acc(4);
    CAMG_CUDA(cudaMemset(acc.p, 0, 4 * sizeof(unsigned long long)));
    k_slot_stats<<<grid_for(S->slots, 256), 256>>>(S->desc, S->slots, acc.p);
    unsigned long long h[4];
    CAMG_CUDA(cudaMemcpy(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost));
    out[0] = S->slots;
    out[2] = (int64_t)h[1];
    if (S->dedup) { out[1] = (int64_t)h[0]; out[3] = (int64_t)h[2]; out[4] = (int64_t)h[3]; }
  });
}

// slices of the block mirror and how many of them run the uniform-slice loop
extern "C" int camg_csr_uniform_slices(const camg_csr* A, int64_t* out) {
  return guarded([&] {
    const Sell* S = A->m->sell;
    out[0] = S ? S->nslices : 0;
    out[1] = S ? S->n_uslices : 0;
    out[2] = S ? S->n_upairs : 0;
    out[3] = S ? S->n_aligned : 0;
    out[4] = S ? S->n_xgroups : 0;
  });
}

extern "C" int camg_csr_value_groups(const camg_csr* A, int64_t* kept, int64_t* full) {
  return guarded([&] {
    const Sell* S = A->m->sell;
    *kept = S ? S->ngroups : 0;
    *full = S ? (S->dedup ? S->ngroups_full : S->ngroups) : 0;
  });
}

extern "C" int camg_csr_stream_bytes(const camg_csr* A, double* bytes) {
  return guarded([&] {
    const Csr* M = A->m;
    double b = 0.0;
    int64_t row0 = 0;
    if (M->sell) {
      b += sell_pass_bytes(M->sell);
      row0 = M->sell->rows();
    }
    const int64_t tail_nnz = M->nnz - (row0 ? read_i64(M->rowptr + row0) : 0);
    b += 12.0 * (double)tail_nnz + 8.0 * (double)(M->n_rows - row0 + 1);
    b += 8.0 * (double)M->n_cols + 8.0 * (double)M->n_rows;  // x read, y written
    *bytes = b;
  });
}

// Block SELL-32 acceleration mirror (see sell.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace camg {

struct Sell {
  int br = 0, bc = 0;                 // block rows x block columns
  bool masked = false;                // per-slot union masks (else full blocks)
  int64_t nbr = 0, nslices = 0, slots = 0, used_blocks = 0;
  int64_t ncb = 0;                    // block columns of the vector read (checked build)
  int64_t ngroups = 0;                // 32-double value groups stored (checked build)
  double pass_bytes = 0.0;            // compulsory bytes of one pass over the blocks
  int64_t* slice_ptr = nullptr;       // slot offset of each slice (nslices+1)
  uint8_t* len = nullptr;             // blocks per block row
  int32_t* bcol = nullptr;            // [slot][lane]
  double* bval = nullptr;             // [voff[slot] + rank in mask][lane]
  unsigned long long* mask = nullptr; // per slot: union of the block patterns of its lanes
  int64_t* voff = nullptr;            // per slot: offset of its value groups (32 doubles each)
  unsigned long long* desc = nullptr; // per slot (BR*BC <= 15): nibble q = 1 + rank of position q (0: absent),
                                      // bits 36-59 = 1 + first column of a linear slot (0: load bcol), bits 60-63 = count
  double* zero = nullptr;             // masked: one zero value group (absent positions load it)
  // shared value groups (masked mirrors): slots whose stored values are bit-identical (the interior stencil
  // of a structured mesh repeats from slice to slice) keep ONE copy; vo[slot] = first value group of the
  // slot's copy, desc bit 60 = every group of the slot is lane-uniform (loaded as a broadcast)
  bool dedup = false;
  uint32_t* vo = nullptr;
  int64_t ngroups_full = 0;           // value groups before sharing
  // uniform slices (shared value groups, 3x3): every slot of the slice is linear and lane-uniform (a slice
  // inside one mesh row of the structured interior) and reads columns of the square part only: the pass runs
  // them through a loop without descriptor decoding (uslice[slice] = 1)
  uint8_t* uslice = nullptr;
  // work items of a full pass: the slices without the followers of the groups (a follower's warp would only
  // skip), wmode[w] = block rows per lane of item w's group (2 / 3) or 0 (run the slice by itself)
  int32_t* witems = nullptr;
  uint8_t* wmode = nullptr;
  int32_t* wdist = nullptr;           // slices between the members of item w's group (1: neighbours)
  int64_t n_witems = 0;
  std::vector<uint8_t> h_uslice;      // host copy of uslice (sell_compact_list)
  // slices with exception lanes (uslice 2) repeat with a period: the slice `xpart[s]` slices further on has
  // the same value groups, the same exception lanes and columns 32 * xpart[s] apart (0: none) -- on a
  // structured mesh the slice across the end of mesh row j and the one across row j + 32.  Such slices run
  // in groups too (work items only)
  int32_t* xpart = nullptr;
  std::vector<int32_t> h_xpart;
  int64_t n_xgroups = 0;
  int64_t n_aligned = 0;  // slices with offset-aligned slots (sell.cu)
  int64_t n_uslices = 0, n_upairs = 0;  // n_upairs: pairs of neighbouring uniform slices run as one work item (uslice 3 / 4)
  int32_t* perm = nullptr;            // ordered SELL: block row at each position (-1 = padding)
  double* dblk = nullptr;             // ordered SELL: diagonal node block per position [slice][e][lane]
  ~Sell();
  int64_t rows() const { return nbr * br; }
};

struct SellView {
  const int64_t* __restrict__ slice_ptr;
  const uint8_t* __restrict__ len;
  const int32_t* __restrict__ bcol;
  const double* __restrict__ bval;
  const unsigned long long* __restrict__ mask;
  const int64_t* __restrict__ voff;
  const unsigned long long* __restrict__ desc;
  const double* __restrict__ zero;
  int64_t nbr, nslices;
  const int32_t* __restrict__ slist = nullptr;  // optional subset of slices to process
  int64_t nwork = 0;                            // slices to process (slist length, or nslices)
  int64_t ncb = 0, ngroups = 0;                 // bounds for the checked build (0: unknown)
  const uint32_t* __restrict__ vo = nullptr;    // shared value groups: first group of each slot
  const uint8_t* __restrict__ uslice = nullptr; // uniform slices (null: none / columns may cross the split)
  const uint8_t* __restrict__ wmode = nullptr;  // per work item: group size decided on the host (null: the kernel
                                                // checks the group's members in the list itself); bit 2: a
                                                // group of slices with exception lanes
  const int32_t* __restrict__ wdist = nullptr;  // per work item: slices between the group's members
};

// epilogue arguments of the three SELL row kernels (modes 0/1/2)
struct SellEpi {
  double* y = nullptr;
  double alpha = 1.0, beta = 0.0;
  const double* b = nullptr;
  const double* x = nullptr;
  double* out_r = nullptr;
  const double* dscale = nullptr;
  double* out_d = nullptr;
  double* out_x = nullptr;
  double coef = 0.0;
  const double* d = nullptr;
  const double* r = nullptr;
  const double* x0 = nullptr;  // mode 1, xmode 1: out_x = x0 + coef*((x + d) - x0)
  int xmode = 0;
  double* out_y = nullptr;     // mode 1: Jacobi iterate y = x + d
  const double* dprev = nullptr;  // mode 1 (Chebyshev): d = c1*dprev + c2*dscale*res
  double c1 = 0.0, c2 = 1.0;
};

Sell* sell_build(const Csr* A, int br, int bc, int64_t nrows, int64_t ncols_blocked, cudaStream_t s,
                 bool masked = false);
// shared value groups of the masked mirrors built next: 1 on, 0 off, -1 as CAMG_SELL_DEDUP says (default on)
void sell_share_override(int v);
// mode 0: spmv, 1: residual (+ fused Jacobi epilogue), 2: extra Jacobi sweep
// (modes 1/2 need square blocks).  split < 0: x is one vector (xu); else
// columns >= split read xl (null = 0).
void sell_launch(const Sell* S, int mode, bool zero, const double* xu, const double* xl, int64_t split,
                 const SellEpi& e, cudaStream_t st, const int32_t* slist = nullptr, int64_t nlist = -1,
                 const uint8_t* lmode = nullptr, const int32_t* ldist = nullptr);
// Turn an ascending slice list into work items for passes with x != 0: followers of uniform-slice groups
// whose whole group is in the list are dropped, mode[w] = 2 / 3 for an entry that leads such a group, 0 for an
// entry that runs by itself.  Pass the result as (slist, nlist, lmode); zero-start passes keep the slice list.
// dist[w] = slices between the members of entry w's group (1 for neighbours; mode bit 2 marks a group of slices
// with exception lanes, whose members lie a mesh-row period apart).  Pass (slist, nlist, lmode, ldist).
void sell_compact_list(const Sell* S, std::vector<int32_t>& list, std::vector<uint8_t>& mode,
                       std::vector<int32_t>& dist);
double sell_pass_bytes(const Sell* S);
int sell_lanes(const Sell* S);
// colour-ordered SELL (square bs x bs blocks, full): position t of the
// mirror holds block row order[t] (-1 = padding), order.size() % 32 == 0
Sell* sell_build_ordered(const Csr* A, int bs, int64_t nrows, int64_t ncols_blocked, const std::vector<int32_t>& order,
                         cudaStream_t s);
// one colour pass of multicolour Gauss-Seidel over slices [s0, s1)
void sell_gs_launch(const Sell* S, int64_t s0, int64_t s1, bool fwd, bool zero, const double* xl, int64_t split,
                    const double* b, const double* dinv, double* y, cudaStream_t st);

}  // namespace camg

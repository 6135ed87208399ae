// Point smoothers with the reference's exact (lexicographic) semantics on the
// device (smoothers.py:141-199): jacobi, sgs (residual-form SSOR(omega) with
// the forward / backward triangular solves of tril(A)+D/omega and
// triu(A)+D/omega), ilu0 (the reference's IKJ factorization, unit-lower L and
// upper U solves), direct (dense LU).  The triangular solves are sync-free:
// one warp per row, rows handed out in dependency order by a global ticket,
// each row waiting (acquire) on the completion flags of the rows it reads.
#pragma once

#include "kernels.cuh"

namespace camg {

// reference ILU(0) in IKJ order on host CSR arrays (in place); returns the
// diagonal positions (hierarchy.cu)
std::vector<int64_t> ilu0_ikj(int64_t n, const int64_t* rp, const int32_t* ci, double* va, const int32_t* name);
// dense LU solve with LAPACK factors (column-major) on one CTA (hierarchy.cu)
void lu_solve(int n, const double* LU, const int32_t* piv, const double* b, double* x, cudaStream_t s);

// y = T^-1 r for a triangular T given by its strict part Toff and diagonal
// diag (null: unit); lower = rows in increasing order.  `sync` holds the
// ticket and the n completion flags (8 + 4 n bytes, zeroed here).
void sptrsv(const Csr* Toff, const double* diag, bool lower, const double* r, double* y, void* sync, int* err,
            cudaStream_t s);
size_t sptrsv_sync_bytes(int64_t n);

struct PointSolver {
  int kind = CAMG_PT_JACOBI;
  int sweeps = 1;
  double damping = 1.0;
  const Csr* A = nullptr;  // borrowed
  int64_t n = 0;
  DBuf<double> dinv;                  // jacobi: damping / diag(A)
  std::unique_ptr<Csr> Lo, Uo;        // strict lower / upper triangles (sgs: of A, ilu0: of the factors)
  DBuf<double> dsgs, udiag;           // sgs: diag(A) / damping; ilu0: diagonal of U
  DBuf<double> lu;                    // direct: LAPACK factors, column-major
  DBuf<int32_t> piv;
  DBuf<int> err;                      // sync-free solve watchdog
  // per-application work vectors (re-entrant V-cycle workspaces swap them)
  DBuf<double> w_r, w_d, w_sync;

  void setup(const Csr* A_, int kind_, int sweeps_, double damping_);
  void set_lu(int64_t n_, const double* lu_colmajor, const int32_t* piv_);
  // out = `sweeps` sweeps from x (null: zero) on A out = b; direct: out = A^-1 b
  void smooth(const double* x, const double* b, double* out, cudaStream_t s);
  void check_watchdog();
  void work_slots(std::vector<DBuf<double>*>& v) {
    v.push_back(&w_r);
    v.push_back(&w_d);
    v.push_back(&w_sync);
  }
  bool active() const { return A != nullptr; }
};

}  // namespace camg

// Shared definitions for libcamg (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>
#include <stdexcept>

#include "../../include/camg.h"

namespace camg {

struct Sell;

// ---------------------------------------------------------------------------
// error handling: every C entry point catches camg::Error and returns its code

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define CAMG_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      throw ::camg::Error(CAMG_ERR_CUDA, std::string(#call " failed: ") +        \
                                             cudaGetErrorString(e_) + " at " +   \
                                             __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define CAMG_CHECK(cond, code, msg)                       \
  do {                                                    \
    if (!(cond)) throw ::camg::Error((code), (msg));      \
  } while (0)

#define CAMG_LAUNCH_CHECK() CAMG_CUDA(cudaGetLastError())

// Device-side bounds / invariant checks of the checked build (`make checked`
// -> libcamg_checked.so, -DCAMG_CHECKED; load it with CAMG_LIB): a failed
// check prints its site and traps (the launch fails with an error).  The
// substitute for compute-sanitizer, which this GPU pool does not allow.
#ifdef CAMG_CHECKED
#define CAMG_DCHECK(cond, what)                                                          \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("camg device check failed: %s (%s:%d)\n", what, __FILE__, __LINE__);        \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define CAMG_DCHECK(cond, what) \
  do {                          \
  } while (0)
#endif

// Run `body` and translate exceptions into status codes.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return CAMG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return CAMG_ERR_NATIVE;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CAMG_ERR_NATIVE;
  }
}

// ---------------------------------------------------------------------------
// device memory

template <class T>
T* dalloc(size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
  CAMG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}

inline void dfree(void* p) {
  if (p) cudaFree(p);
}

// RAII device buffer used for temporaries
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t n_) : p(dalloc<T>(n_)), n(n_) {}
  ~DBuf() { dfree(p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { dfree(p); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  T* release() { T* q = p; p = nullptr; n = 0; return q; }
  void resize(size_t n_) { if (n_ > n) { dfree(p); p = dalloc<T>(n_); n = n_; } }
};

// ---------------------------------------------------------------------------
// device CSR: int64 row offsets, int32 columns, fp64 values

struct Csr {
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double avg_row = 0.0;
  Sell* sell = nullptr;  // optional block SELL-32 mirror of the leading rows
  ~Csr();
};

struct CsrView {
  const int64_t* __restrict__ rowptr;
  const int32_t* __restrict__ col;
  const double* __restrict__ val;
  int64_t n_rows, n_cols;
};

inline CsrView view(const Csr* A) {
  return CsrView{A->rowptr, A->col, A->val, A->n_rows, A->n_cols};
}

Csr* csr_alloc(int64_t n_rows, int64_t n_cols, int64_t nnz);

// helpers implemented in csr.cu / vec.cu
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);  // out has n+1 entries
int64_t read_i64(const int64_t* dptr);
void spmv(const Csr* A, double alpha, const double* x, double beta, double* y, cudaStream_t s);
void spmv_rows(const Csr* A, int64_t row0, int64_t nrows, double alpha, const double* xu,
               const double* xl, int64_t split, double beta, double* y, cudaStream_t s);
Csr* csr_transpose(const Csr* A, cudaStream_t s);
void csr_diagonal(const Csr* A, int mode, double* d, cudaStream_t s);
Csr* csr_copy(const Csr* A, cudaStream_t s);

inline unsigned grid_for(int64_t work, int block, int64_t cap = 148LL * 64) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

constexpr int kNumSMs = 148;

}  // namespace camg

// opaque handle types exposed through the C ABI
namespace camg { struct Level; struct Hierarchy; struct ScalarHier; struct VcycleWs; struct Gmres; }
struct camg_csr { camg::Csr* m; };
struct camg_level { camg::Level* L; };
struct camg_hierarchy { camg::Hierarchy* H; };
struct camg_scalar_hierarchy { camg::ScalarHier* H; };
struct camg_vcycle_workspace { camg::VcycleWs* W; camg::Hierarchy* H; };
struct camg_gmres_workspace { camg::Gmres* G; };

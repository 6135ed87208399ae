"""Sparse matrices and block vectors backed by device CSR (libcamg).

Mirrors `pkg/src/contactamg/sparse.py`: `SparseMatrix` keeps the reference
constructor, canonical form (sorted columns, duplicates summed, |v| < 1e-300
dropped, sparse.py:50-66) and immutability, but its storage of record is a
device CSR handle.  Host arrays are downloaded lazily, only when a caller
asks for `row_offsets` / `col_indices` / `values` / `to_scipy()`.

Vectors: functions accept numpy arrays (copied to and from the device) or
float64 CUDA torch tensors (zero copy); results come back in the caller's
kind.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.io
import scipy.linalg
import scipy.sparse

from . import _native as N
from .errors import DimensionError, SingularMatrixError

DROP_TOL = 1e-300


# ---------------------------------------------------------------------------
# device vector helpers (torch is used for device memory only)


def _torch():
    import torch

    return torch


def stream_ptr():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def is_device(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, n=None):
    """float64 contiguous CUDA tensor for numpy / torch input."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=torch.float64)
        t = t.contiguous()
    else:
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        t = torch.from_numpy(a).to("cuda")
    if n is not None and t.numel() != n:
        raise DimensionError(f"vector has length {t.numel()}, expected {n}")
    return t


def empty(n):
    torch = _torch()
    return torch.empty(int(n), dtype=torch.float64, device="cuda")


def zeros(n):
    torch = _torch()
    return torch.zeros(int(n), dtype=torch.float64, device="cuda")


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def like_input(t, ref):
    """Return device tensor `t` in the kind of `ref` (numpy or torch)."""
    if is_device(ref):
        return t
    return t.cpu().numpy()


# ---------------------------------------------------------------------------


def _canonical_scipy(mat) -> scipy.sparse.csr_matrix:
    csr = scipy.sparse.csr_matrix(mat)
    csr.sum_duplicates()
    csr.sort_indices()
    keep = np.abs(csr.data) >= DROP_TOL
    if not keep.all():
        coo = csr.tocoo()
        csr = scipy.sparse.csr_matrix((coo.data[keep], (coo.row[keep], coo.col[keep])), shape=csr.shape)
        csr.sum_duplicates()
        csr.sort_indices()
    return csr


class _Handle:
    """Owns one camg_csr*."""

    __slots__ = ("h",)

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h and N._lib is not None:
            N._lib.camg_csr_destroy(self.h)
            self.h = None


class SparseMatrix:
    """Immutable CSR matrix (sparse.py:24-115), stored on the device."""

    __slots__ = ("num_rows", "num_cols", "_host", "_dev", "_nnz", "__weakref__")

    def __init__(self, num_rows, num_cols, row_offsets, col_indices, values):
        self.num_rows = int(num_rows)
        self.num_cols = int(num_cols)
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(col_indices, dtype=np.int64)
        va = np.ascontiguousarray(values, dtype=np.float64)
        if ro.shape != (self.num_rows + 1,):
            raise DimensionError("row_offsets length must be num_rows + 1")
        if ro[0] != 0 or ro[-1] != len(va):
            raise DimensionError("row_offsets must start at 0 and end at nnz")
        if len(ci) != len(va):
            raise DimensionError("col_indices and values length mismatch")
        for a in (ro, ci, va):
            a.flags.writeable = False
        self._host = (ro, ci, va)
        self._dev = None
        self._nnz = len(va)

    # -- constructors ---------------------------------------------------------

    @staticmethod
    def from_scipy(mat) -> "SparseMatrix":
        c = _canonical_scipy(mat)
        return SparseMatrix(c.shape[0], c.shape[1], c.indptr, c.indices, c.data)

    @staticmethod
    def from_coo(rows, cols, vals, shape) -> "SparseMatrix":
        return SparseMatrix.from_scipy(
            scipy.sparse.coo_matrix((np.asarray(vals, dtype=np.float64), (rows, cols)), shape=shape))

    @staticmethod
    def from_dense(arr) -> "SparseMatrix":
        return SparseMatrix.from_scipy(scipy.sparse.csr_matrix(np.asarray(arr, dtype=np.float64)))

    @staticmethod
    def identity(n) -> "SparseMatrix":
        return SparseMatrix.from_scipy(scipy.sparse.identity(n, format="csr"))

    @staticmethod
    def zeros(num_rows, num_cols) -> "SparseMatrix":
        return SparseMatrix(num_rows, num_cols, np.zeros(num_rows + 1, dtype=np.int64), [], [])

    @staticmethod
    def diagonal(d) -> "SparseMatrix":
        return SparseMatrix.from_scipy(scipy.sparse.diags(np.asarray(d, dtype=np.float64), format="csr"))

    @staticmethod
    def _wrap(handle) -> "SparseMatrix":
        """Adopt a device matrix produced by libcamg."""
        m = SparseMatrix.__new__(SparseMatrix)
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        N.call("camg_csr_shape", handle, C.byref(r), C.byref(c), C.byref(z))
        m.num_rows, m.num_cols, m._nnz = r.value, c.value, z.value
        m._host = None
        m._dev = _Handle(handle)
        return m

    # -- device / host views ----------------------------------------------------

    @property
    def device(self):
        """camg_csr* handle (uploads on first use)."""
        if self._dev is None:
            ro, ci, va = self._host
            h = C.c_void_p()
            N.call("camg_csr_from_host", self.num_rows, self.num_cols, len(va),
                   ro.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p),
                   va.ctypes.data_as(C.c_void_p), C.byref(h))
            self._dev = _Handle(h)
        return self._dev.h

    def _host_arrays(self):
        if self._host is None:
            ro = np.empty(self.num_rows + 1, dtype=np.int64)
            ci = np.empty(self._nnz, dtype=np.int64)
            va = np.empty(self._nnz, dtype=np.float64)
            N.call("camg_csr_to_host", self._dev.h, ro.ctypes.data_as(C.c_void_p),
                   ci.ctypes.data_as(C.c_void_p), va.ctypes.data_as(C.c_void_p))
            for a in (ro, ci, va):
                a.flags.writeable = False
            self._host = (ro, ci, va)
        return self._host

    @property
    def row_offsets(self):
        return self._host_arrays()[0]

    @property
    def col_indices(self):
        return self._host_arrays()[1]

    @property
    def values(self):
        return self._host_arrays()[2]

    def drop_host(self):
        """Forget the host copy (large matrices live on the device only)."""
        _ = self.device
        self._host = None

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        ro, ci, va = self._host_arrays()
        return scipy.sparse.csr_matrix((va, ci, ro), shape=(self.num_rows, self.num_cols))

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    @property
    def nnz(self) -> int:
        return self._nnz

    @property
    def shape(self):
        return (self.num_rows, self.num_cols)

    def __repr__(self):
        return f"SparseMatrix({self.num_rows}x{self.num_cols}, nnz={self.nnz})"


class BlockVector:
    """Displacement / multiplier pair [u, lam] (sparse.py:118-143).

    Holds numpy arrays or CUDA tensors; the constructor copies.
    """

    __slots__ = ("u", "lam")

    def __init__(self, u, lam):
        if is_device(u):
            self.u = u.clone().to(dtype=_torch().float64)
            self.lam = to_device(lam).clone()
        else:
            self.u = np.array(u, dtype=np.float64)
            self.lam = np.array(lam, dtype=np.float64)

    @staticmethod
    def zeros(n_u, n_lam) -> "BlockVector":
        return BlockVector(np.zeros(n_u), np.zeros(n_lam))

    @staticmethod
    def from_merged(x, n_u) -> "BlockVector":
        if is_device(x):
            return BlockVector(x[:n_u], x[n_u:])
        x = np.asarray(x, dtype=np.float64)
        return BlockVector(x[:n_u], x[n_u:])

    def merged(self):
        if is_device(self.u):
            return _torch().cat([self.u, self.lam])
        return np.concatenate([self.u, self.lam])

    def copy(self) -> "BlockVector":
        return BlockVector(self.u, self.lam)

    def __len__(self):
        return len(self.u) + len(self.lam)


# ---------------------------------------------------------------------------
# operations (device)


def spmv(A: SparseMatrix, x):
    """y = A @ x on the device (sparse.py:149-154)."""
    n = x.numel() if is_device(x) else np.asarray(x).shape[0]
    if (not is_device(x) and np.asarray(x).shape != (A.num_cols,)) or n != A.num_cols:
        raise DimensionError(f"spmv: x has length {n}, expected ({A.num_cols},)")
    xd = to_device(x)
    y = empty(A.num_rows)
    N.call("camg_spmv", A.device, 1.0, ptr(xd), 0.0, ptr(y), stream_ptr())
    return like_input(y, x)


def sp_transpose(A: SparseMatrix) -> SparseMatrix:        # sparse.py:157-158
    h = C.c_void_p()
    N.call("camg_transpose", A.device, C.byref(h))
    return SparseMatrix._wrap(h)


def sp_matmul(A: SparseMatrix, B: SparseMatrix) -> SparseMatrix:   # sparse.py:161-166
    if A.num_cols != B.num_rows:
        raise DimensionError(f"sp_matmul: inner dimensions {A.num_cols} != {B.num_rows}")
    h = C.c_void_p()
    N.call("camg_spgemm", A.device, B.device, C.byref(h))
    return SparseMatrix._wrap(h)


def galerkin_triple(R: SparseMatrix, A: SparseMatrix, P: SparseMatrix) -> SparseMatrix:  # :169-173
    if R.num_cols != A.num_rows or A.num_cols != P.num_rows:
        raise DimensionError("galerkin_triple: dimension mismatch")
    h = C.c_void_p()
    N.call("camg_galerkin", R.device, A.device, P.device, C.byref(h))
    return SparseMatrix._wrap(h)


def diagonal_device(A: SparseMatrix, mode: str = "plain"):
    if A.num_rows != A.num_cols:
        raise DimensionError("extract_diagonal: matrix must be square")
    m = {"plain": 0, "abs_rowsum": 1}.get(mode)
    if m is None:
        raise ValueError(f"unknown diagonal mode: {mode!r}")
    d = empty(A.num_rows)
    N.call("camg_diagonal", A.device, m, ptr(d))
    return d


def extract_diagonal(A: SparseMatrix, mode: str = "plain") -> np.ndarray:   # sparse.py:176-188
    d = diagonal_device(A, mode).cpu().numpy()
    if mode == "abs_rowsum" and np.any(d == 0.0):
        row = int(np.argmax(d == 0.0))
        raise SingularMatrixError(f"abs_rowsum lumping: row {row} is entirely zero")
    return d


def dense_lu_solve(A, b) -> np.ndarray:                    # sparse.py:191-208
    """Dense LU with partial pivoting (host LAPACK; small dense systems)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise DimensionError("dense_lu_solve: A must be square")
    if b.shape[0] != A.shape[0]:
        raise DimensionError("dense_lu_solve: rhs length mismatch")
    if A.shape[0] == 0:
        return np.zeros(0)
    lu, piv = lu_factor_quiet(A)
    if np.any(np.diag(lu) == 0.0):
        raise SingularMatrixError("dense_lu_solve: zero pivot after pivoting")
    return scipy.linalg.lu_solve((lu, piv), b)


def lu_factor_quiet(A):
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", scipy.linalg.LinAlgWarning)
        return scipy.linalg.lu_factor(A)


def dot(x, y) -> float:
    if is_device(x) or is_device(y):
        xd, yd = to_device(x), to_device(y)
        if xd.numel() != yd.numel():
            raise DimensionError("dot: length mismatch")
        r = C.c_double()
        N.call("camg_dot", xd.numel(), ptr(xd), ptr(yd), C.byref(r), stream_ptr())
        return r.value
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise DimensionError("dot: length mismatch")
    return float(np.dot(x, y))


def axpy(alpha, x, y):
    """alpha * x + y (new array)."""
    if is_device(x) or is_device(y):
        xd, yd = to_device(x), to_device(y).clone()
        if xd.numel() != yd.numel():
            raise DimensionError("axpy: length mismatch")
        N.call("camg_axpy", xd.numel(), float(alpha), ptr(xd), ptr(yd), stream_ptr())
        return yd
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise DimensionError("axpy: length mismatch")
    return alpha * x + y


def norm2(x) -> float:
    if is_device(x):
        return float(np.sqrt(max(dot(x, x), 0.0)))
    x = np.asarray(x, dtype=np.float64)
    return 0.0 if x.size == 0 else float(np.linalg.norm(x))


# -- MatrixMarket I/O (sparse.py:238-261) ------------------------------------


def write_matrix_market(path, A: SparseMatrix) -> None:
    with open(path, "wb") as fh:
        scipy.io.mmwrite(fh, A.to_scipy().tocoo(), field="real", symmetry="general")


def read_matrix_market(path) -> SparseMatrix:
    with open(path, "rb") as fh:
        return SparseMatrix.from_scipy(scipy.io.mmread(fh))


def write_vector(path, v) -> None:
    with open(path, "wb") as fh:
        scipy.io.mmwrite(fh, np.asarray(v, dtype=np.float64).reshape(-1, 1))


def read_vector(path) -> np.ndarray:
    with open(path, "rb") as fh:
        return np.asarray(scipy.io.mmread(fh)).ravel()

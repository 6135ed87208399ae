"""Saddle-point block smoothers on the device (smoothers.py:1-384).

`BlockSmoother` binds a configuration to one saddle operator and owns a
native level (`camg_level`): merged operator, S~, inverse diagonals and the
fused step kernels of `csrc/hierarchy.cu`.  Configuration classes keep the
reference names, defaults and validation (smoothers.py:29-70).

Inner solves on the GPU keep the reference's semantics: `jacobi` (fused into
the row passes), `direct` (dense LU solve; LAPACK factors from the host),
and the lexicographic `sgs` / `ilu0` (smoothers.py:141-199) as sync-free
triangular solves in the reference's row order (`csrc/pointsolve.cu`), so the
reference default `BlockSmootherConfig()` (sgs predictor, ilu0 corrector)
runs the reference's algorithm and matches it elementwise.  Their
dependency chains make them latency-bound on large levels; the GPU variants
below are the fast choices (compared with the lexicographic reference by
convergence: profiles/r02_convergence_table.md).  `a_hat_mode="exact"`
(test-scale, smoothers.py:233-236) builds S~ densely on the host from K's LU
factors and applies A^-1 = K^-1 by dense LU solves on the device.
The GPU variant
`mcgs` is the reference's residual-form SSOR applied with rows renumbered by
a greedy colouring: multicolour symmetric Gauss-Seidel, compared with the
reference SGS by convergence, and elementwise with the oracle's emulation of
the same colouring.  As corrector it colours the rows of S~; as predictor it
colours the nodes of K (`node_block` consecutive DOFs per node, visited in
order within a node), which is the block Gauss-Seidel the paper's Uzawa / BGS
configurations use on the GPU.  `mcilu0` (corrector) is the reference's
ILU(0) (smoothers.py:82-123, 195-197) on S~ with rows and columns renumbered
by the same greedy point colouring: both triangular solves then run one
colour per pass.  `gpu_chebyshev` (predictor, GPU-only like
`mcgs`; the reference rejects the name "chebyshev", and so does this
package) is the Chebyshev polynomial of D^-1 K of degree `sweeps` on
[lmax/30, 1.1 lmax] with lmax from the smoothed-aggregation power
iteration; `damping` is not used by it.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ConfigError, SingularMatrixError
from .saddle import SaddleOperator, SaddleSystem
from .sparse import (
    BlockVector,
    SparseMatrix,
    diagonal_device,
    extract_diagonal,
    empty,
    is_device,
    lu_factor_quiet,
    ptr,
    stream_ptr,
    to_device,
)

POINT_KINDS = ("jacobi", "sgs", "ilu0", "direct", "mcgs", "mcilu0", "gpu_chebyshev")
BLOCK_KINDS = ("uzawa", "braess_sarazin", "simple", "simplec")
A_HAT_MODES = ("plain_diag", "abs_rowsum", "exact")
GPU_POINT_KINDS = ("jacobi", "sgs", "ilu0", "direct")
GPU_PREDICTOR_KINDS = ("jacobi", "sgs", "ilu0", "direct", "gpu_chebyshev", "mcgs")
GPU_CORRECTOR_KINDS = ("jacobi", "sgs", "ilu0", "direct", "mcgs", "mcilu0")

# multicolour GPU variants of the reference's sequential inner solves
GPU_VARIANT = {"sgs": "mcgs", "ilu0": "mcilu0"}

_BLOCK_CODE = {"uzawa": 0, "braess_sarazin": 1, "simple": 2, "simplec": 3}
_POINT_CODE = {"jacobi": 0, "sgs": 1, "ilu0": 2, "direct": 3, "gpu_chebyshev": 4, "mcgs": 5, "mcilu0": 6}
_AHAT_CODE = {"plain_diag": 0, "abs_rowsum": 1, "exact": 2}


@dataclass(frozen=True)
class PointSmootherConfig:                       # smoothers.py:29-41
    kind: str = "sgs"
    sweeps: int = 1
    damping: float = 1.0

    def __post_init__(self):
        if self.kind not in POINT_KINDS:
            raise ConfigError(f"unknown point smoother kind: {self.kind!r}")
        if self.sweeps < 1:
            raise ConfigError("point smoother sweeps must be >= 1")
        if not (0.0 < self.damping < 2.0):
            raise ConfigError("point smoother damping must lie in (0, 2)")


@dataclass(frozen=True)
class BlockSmootherConfig:                       # smoothers.py:44-70
    kind: str = "simplec"
    alpha: float = 0.7
    outer_sweeps: int = 1
    predictor: PointSmootherConfig = field(default_factory=PointSmootherConfig)
    corrector: PointSmootherConfig = field(default_factory=lambda: PointSmootherConfig(kind="ilu0"))
    a_hat_mode: str = "plain_diag"

    def __post_init__(self):
        if self.kind not in BLOCK_KINDS:
            raise ConfigError(f"unknown block smoother kind: {self.kind!r}")
        if self.alpha <= 0.0:
            raise ConfigError("alpha must be positive")
        if self.outer_sweeps < 1:
            raise ConfigError("outer_sweeps must be >= 1")
        if self.a_hat_mode not in A_HAT_MODES:
            raise ConfigError(f"unknown a_hat_mode: {self.a_hat_mode!r}")
        if self.kind == "braess_sarazin" and self.a_hat_mode != "plain_diag":
            raise ConfigError("braess_sarazin hard-codes the plain-diagonal predictor")

    def effective_a_hat_mode(self) -> str:
        if self.kind == "simplec":
            return "abs_rowsum"
        if self.kind == "braess_sarazin":
            return "plain_diag"
        return self.a_hat_mode


@dataclass
class SchurOperator:
    S_tilde: SparseMatrix
    a_hat_inv_diag: np.ndarray | None


def multicolour_cfg(cfg: BlockSmootherConfig):
    """`cfg` with the sequential `sgs` / `ilu0` inner solves replaced by their
    multicolour GPU variants (same damping; ILU(0) has none) -- the fast
    choice on large levels.  Returns (config, list of substitutions made)."""
    from dataclasses import replace

    subs = []
    pred, corr = cfg.predictor, cfg.corrector
    if cfg.kind != "braess_sarazin" and pred.kind in GPU_VARIANT:
        subs.append(f"predictor {pred.kind} -> {GPU_VARIANT[pred.kind]}")
        pred = replace(pred, kind=GPU_VARIANT[pred.kind])
    if corr.kind in GPU_VARIANT:
        subs.append(f"corrector {corr.kind} -> {GPU_VARIANT[corr.kind]}")
        corr = replace(corr, kind=GPU_VARIANT[corr.kind])
    if not subs:
        return cfg, subs
    return replace(cfg, predictor=pred, corrector=corr), subs


def native_cfg(cfg: BlockSmootherConfig, node_block: int = 1) -> N.SmootherCfg:
    mode = cfg.effective_a_hat_mode()
    if cfg.kind != "braess_sarazin" and cfg.predictor.kind not in GPU_PREDICTOR_KINDS:
        raise ConfigError(f"GPU predictor supports {GPU_PREDICTOR_KINDS}, got {cfg.predictor.kind!r}")
    if cfg.corrector.kind not in GPU_CORRECTOR_KINDS:
        raise ConfigError(f"GPU corrector supports {GPU_CORRECTOR_KINDS}, got {cfg.corrector.kind!r}")
    return N.SmootherCfg(
        kind=_BLOCK_CODE[cfg.kind], alpha=float(cfg.alpha), outer_sweeps=int(cfg.outer_sweeps),
        a_hat_mode=_AHAT_CODE[mode],
        pred_kind=_POINT_CODE.get(cfg.predictor.kind, 0), pred_sweeps=int(cfg.predictor.sweeps),
        pred_damping=float(cfg.predictor.damping),
        corr_kind=_POINT_CODE[cfg.corrector.kind], corr_sweeps=int(cfg.corrector.sweeps),
        corr_damping=float(cfg.corrector.damping), node_block=max(1, int(node_block)),
    )


class _LevelHandle:
    __slots__ = ("h",)

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h and N._lib is not None:
            N._lib.camg_level_destroy(self.h)
            self.h = None


class _PointHandle:
    __slots__ = ("h",)

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h and N._lib is not None:
            N._lib.camg_point_destroy(self.h)
            self.h = None


def _lu_factors(A_dense):
    """LAPACK LU (scipy.linalg.lu_factor) as (column-major factors, int32
    pivots); a zero pivot raises like the reference (smoothers.py:176-181)."""
    lu, piv = lu_factor_quiet(A_dense)
    if np.any(np.diag(lu) == 0.0):
        raise SingularMatrixError("direct smoother: singular matrix")
    return np.asfortranarray(lu), np.ascontiguousarray(piv, dtype=np.int32)


class PointSmoother:
    """Point smoother bound to one matrix (smoothers.py:141-199), executed by
    libcamg (`camg_point_*`): jacobi, the lexicographic sgs / ilu0 sweeps
    (sync-free triangular solves in the reference's order; ilu0 factored in
    the reference's IKJ order), direct (dense LU solve on the device)."""

    def __init__(self, cfg: PointSmootherConfig, A: SparseMatrix):
        if cfg.kind not in GPU_POINT_KINDS:
            raise ConfigError(f"GPU point smoother supports {GPU_POINT_KINDS}, got {cfg.kind!r}")
        self.cfg, self.A = cfg, A
        h = C.c_void_p()
        N.call("camg_point_create", A.device, _POINT_CODE[cfg.kind], int(cfg.sweeps), float(cfg.damping),
               C.byref(h))
        self._h = _PointHandle(h)
        if cfg.kind == "direct" and A.num_rows:
            lu, piv = _lu_factors(A.to_dense())
            N.call("camg_point_set_lu", h, A.num_rows, lu.ctypes.data_as(C.c_void_p), piv.ctypes.data_as(C.c_void_p))

    def _run(self, x, b):
        n = self.A.num_rows
        bd = to_device(b, n)
        xd = None if x is None else to_device(x, n)
        out = empty(n)
        N.call("camg_point_smooth", self._h.h, C.c_void_p(0) if xd is None else ptr(xd), ptr(bd), ptr(out),
               stream_ptr())
        return out if is_device(b) else out.cpu().numpy()

    def smooth(self, x, b):
        return self._run(x, b)

    def apply(self, b):
        """Approximate A^-1 b from the zero vector (linear in b)."""
        return self._run(None, b)


def build_schur(op, a_hat_mode: str = "plain_diag", alpha: float = 1.0, scale_with_alpha: bool = False,
                a_hat_scale: float = 1.0) -> SchurOperator:
    """S~ = scale*Cz + scale*B2 diag(1/(a_hat_scale*A^)) B1 on the device
    (smoothers.py:220-239)."""
    if isinstance(op, SaddleSystem):
        op = op.op
    scale = alpha if scale_with_alpha else 1.0
    if a_hat_mode == "exact":
        # test-scale (smoothers.py:233-236): dense K inverse, as the reference
        Kinv = np.linalg.inv(op.K.to_dense())
        S = scale * (op.Cz.to_dense() + op.B2.to_dense() @ Kinv @ op.B1.to_dense())
        return SchurOperator(SparseMatrix.from_dense(S), None)
    d = diagonal_device(op.K, "plain" if a_hat_mode == "plain_diag" else "abs_rowsum")
    if bool((d == 0).any()):
        from .errors import SingularMatrixError
        raise SingularMatrixError("a_hat: zero diagonal entry")
    ainv = 1.0 / (a_hat_scale * d)
    h = C.c_void_p()
    N.call("camg_schur", op.B2.device, op.Cz.device, op.B1.device, ptr(ainv), float(scale), C.byref(h))
    return SchurOperator(SparseMatrix._wrap(h), ainv.cpu().numpy())


class BlockSmoother:
    """Bound block smoother (smoothers.py:245-329), executed by libcamg.

    `node_block` (extension): DOFs per displacement node of the level when
    every node owns that many consecutive DOFs; it sets the node colouring of
    an `mcgs` predictor (1 = colour single DOFs).  An `mcgs` corrector colours
    the rows of S~."""

    def __init__(self, cfg: BlockSmootherConfig, op, predictor_solver=None, pre_sweeps: int = 1,
                 post_sweeps: int = 1, node_block: int = 1):
        if isinstance(op, SaddleSystem):
            op = op.op
        user_cfg = cfg
        self.substitutions = []
        inner = None
        if predictor_solver is not None:
            # smoothers.py:277-278: any object with apply(rhs); on the GPU path it
            # must be a native solver (the nested preconditioner's ScalarHierarchy)
            if not hasattr(predictor_solver, "handle") or not hasattr(predictor_solver, "smoother_cfg"):
                raise ConfigError("GPU predictor_solver must be a ScalarHierarchy (build_scalar_hierarchy)")
            inner = predictor_solver
            if cfg.kind != "braess_sarazin":
                # the configured predictor is unused (reference: overridden)
                cfg_native = BlockSmootherConfig(kind=cfg.kind, alpha=cfg.alpha, outer_sweeps=cfg.outer_sweeps,
                                                 predictor=PointSmootherConfig("jacobi", 1, 1.0),
                                                 corrector=cfg.corrector, a_hat_mode=cfg.a_hat_mode)
            else:
                cfg_native = cfg
        else:
            cfg_native = cfg
        self.cfg = user_cfg
        self.gpu_cfg = cfg
        self.op = op
        ncfg = native_cfg(cfg_native, node_block)
        h = C.c_void_p()
        # the level borrows the operator's merged matrix (one device copy shared
        # with GMRES); self.op keeps it alive
        N.call("camg_level_create_shared", op.merged().device, op.K.device, op.B1.device, op.B2.device,
               op.Cz.device, C.byref(ncfg), int(pre_sweeps), int(post_sweeps), C.byref(h))
        self._level = _LevelHandle(h)
        self._schur = None
        self.predictor_solver = inner
        if inner is not None and cfg.kind != "braess_sarazin":
            N.call("camg_level_set_predictor_solver", h, inner.handle)
        exact = cfg.effective_a_hat_mode() == "exact"
        pred_direct = cfg.kind != "braess_sarazin" and inner is None and cfg.predictor.kind == "direct"
        if exact or pred_direct:
            # dense LU of K (smoothers.py:176, 272-273): the direct predictor and A^-1
            Kd = op.K.to_dense()
            lu, piv = _lu_factors(Kd)
            N.call("camg_level_set_k_lu", h, op.n_u, lu.ctypes.data_as(C.c_void_p), piv.ctypes.data_as(C.c_void_p))
        if exact:
            # S~ = scale (Cz + B2 K^-1 B1) (smoothers.py:233-236), dense, test-scale
            import scipy.linalg
            scale = cfg.alpha if cfg.kind in ("simple", "simplec") else 1.0
            KinvB1 = scipy.linalg.lu_solve((np.asarray(lu), piv), op.B1.to_dense())
            S = scale * (op.Cz.to_dense() + op.B2.to_dense() @ KinvB1)
            Ssm = SparseMatrix.from_dense(S)
            N.call("camg_level_set_schur", h, Ssm.device)
        if cfg.corrector.kind == "direct" and op.n_lam > 0:
            lu_f, piv32 = _lu_factors(self.schur.S_tilde.to_dense())
            N.call("camg_level_set_corrector_lu", self._level.h, op.n_lam,
                   lu_f.ctypes.data_as(C.c_void_p), piv32.ctypes.data_as(C.c_void_p))

    @property
    def handle(self):
        return self._level.h

    @property
    def schur(self) -> SchurOperator:
        if self._schur is None:
            h = C.c_void_p()
            N.call("camg_level_schur", self._level.h, C.byref(h))
            self._schur = SchurOperator(SparseMatrix._wrap(h), None)
        return self._schur

    def sweep_merged(self, x, b):
        """sweep on merged device vectors (x None = zero start)."""
        n = self.op.total_rows
        xd = None if x is None else to_device(x, n)
        bd = to_device(b, n)
        out = empty(n)
        N.call("camg_level_sweep", self._level.h, None if xd is None else ptr(xd), ptr(bd), ptr(out),
               stream_ptr())
        return out

    def sweep(self, x: BlockVector, b: BlockVector) -> BlockVector:
        out = self.sweep_merged(x.merged(), b.merged())
        if not is_device(x.u):
            out = out.cpu().numpy()
        return BlockVector.from_merged(out, self.op.n_u)

    def apply(self, b: BlockVector) -> BlockVector:
        n = self.op.total_rows
        bd = to_device(b.merged(), n)
        out = empty(n)
        N.call("camg_level_sweep", self._level.h, C.c_void_p(0), ptr(bd), ptr(out), stream_ptr())
        if not is_device(b.u):
            out = out.cpu().numpy()
        return BlockVector.from_merged(out, self.op.n_u)


def uzawa_sweep(sys, cfg: BlockSmootherConfig, x: BlockVector, b: BlockVector) -> BlockVector:
    return BlockSmoother(cfg, sys).sweep(x, b)


def braess_sarazin_sweep(sys, cfg: BlockSmootherConfig, x: BlockVector, b: BlockVector) -> BlockVector:
    return BlockSmoother(cfg, sys).sweep(x, b)


def simple_sweep(sys, cfg: BlockSmootherConfig, x: BlockVector, b: BlockVector) -> BlockVector:
    return BlockSmoother(cfg, sys).sweep(x, b)


def point_smooth(cfg: PointSmootherConfig, A: SparseMatrix, x, b):
    return PointSmoother(cfg, A).smooth(x, b)


# -- host helpers of the reference API (smoothers.py:80-123, 209-217, 347-384) --


def ilu0_factor(A: SparseMatrix) -> np.ndarray:
    """ILU(0) factor values on A's exact pattern, unit lower diagonal implicit
    (smoothers.py:80-123): libcamg's host factorization (camg_ilu0_factor),
    the one the multicolour ILU(0) corrector applies to the permuted S~.  A
    missing diagonal or a zero pivot raises SingularMatrixError naming the
    row."""
    ro, ci, va = A._host_arrays()
    ro = np.ascontiguousarray(ro, dtype=np.int64)
    ci32 = np.ascontiguousarray(ci, dtype=np.int32)
    out = np.array(va, dtype=np.float64)
    N.call("camg_ilu0_factor", A.num_rows, ro.ctypes.data_as(C.c_void_p), ci32.ctypes.data_as(C.c_void_p),
           out.ctypes.data_as(C.c_void_p))
    return out


def a_hat_diagonal(K: SparseMatrix, mode: str) -> np.ndarray:
    """Diagonal approximation of K used in S~ (smoothers.py:209-217)."""
    if mode == "plain_diag":
        d = extract_diagonal(K, "plain")
        if np.any(d == 0.0):
            raise SingularMatrixError("a_hat: zero diagonal entry")
        return d
    if mode == "abs_rowsum":
        return extract_diagonal(K, "abs_rowsum")
    raise ValueError(f"a_hat_diagonal: unsupported mode {mode!r}")


def preconditioning_matrix(sys, cfg: BlockSmootherConfig) -> np.ndarray:
    """Dense block preconditioner M of one smoother step with exact inner
    solves, x <- x + M^-1 (b - A x) (smoothers.py:347-378; paper Algs. 2-4):
    Uzawa  M = [[K, 0], [B2, -S]] / alpha,            S = Cz + B2 A^-1 B1
    BS     M = [[alpha A^, B1], [B2, -Cz]]
    SIMPLE M = [[K, 0], [B2, -S]] [[I, A^-1 B1], [0, I / alpha]],  S = alpha (Cz + B2 A^-1 B1)
    with A^ = K for a_hat_mode "exact", else diag(a_hat_diagonal).  Test-scale
    (dense) helper."""
    op = sys.op if isinstance(sys, SaddleSystem) else sys
    K, B1, B2, Cz = (m.to_dense() for m in (op.K, op.B1, op.B2, op.Cz))
    nu, nl = op.n_u, op.n_lam
    a = cfg.alpha
    mode = cfg.effective_a_hat_mode()
    ahat = K if mode == "exact" else np.diag(a_hat_diagonal(op.K, mode))
    ahat_inv = np.linalg.inv(ahat)
    zero_ul = np.zeros((nu, nl))
    if cfg.kind == "uzawa":
        S = Cz + B2 @ ahat_inv @ B1
        return np.block([[K, zero_ul], [B2, -S]]) / a
    if cfg.kind == "braess_sarazin":
        return np.block([[a * ahat, B1], [B2, -Cz]])
    S = a * (Cz + B2 @ ahat_inv @ B1)
    lower = np.block([[K, zero_ul], [B2, -S]])
    upper = np.block([[np.eye(nu), ahat_inv @ B1], [np.zeros((nl, nu)), np.eye(nl) / a]])
    return lower @ upper


def error_matrix(sys, cfg: BlockSmootherConfig) -> np.ndarray:
    """E = A - M of the configured smoother (smoothers.py:381-384)."""
    op = sys.op if isinstance(sys, SaddleSystem) else sys
    return op.merged_dense() - preconditioning_matrix(sys, cfg)

"""CPU tests of the host logic: configuration validation (mirrors the
reference's tests), generator invariants, host aggregation vs the oracle."""

import sys

import numpy as np
import pytest
import scipy.sparse

import camg_oracle as O
from _golden import GOLDEN, cases, load

from paper_1912_09056_b200.aggregation import NodeGraph, aggregate_greedy, aggregate_lagrange, LagrangeMap
from paper_1912_09056_b200.errors import ConfigError
from paper_1912_09056_b200.hierarchy import HierarchyConfig
from paper_1912_09056_b200.krylov import GmresConfig
from paper_1912_09056_b200.problem import config_spec, element_stiffness, generate, mortar_1d
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig
from paper_1912_09056_b200.sparse import SparseMatrix

sys.path.insert(0, GOLDEN)
from cases import BY_NAME  # noqa: E402


def test_point_config_validation():                 # reference tests/test_smoothers.py:118-124
    with pytest.raises(ConfigError):
        PointSmootherConfig(kind="chebyshev")
    with pytest.raises(ConfigError):
        PointSmootherConfig(sweeps=0)
    with pytest.raises(ConfigError):
        PointSmootherConfig(damping=2.0)


def test_block_config_validation():
    with pytest.raises(ConfigError):
        BlockSmootherConfig(kind="nope")
    with pytest.raises(ConfigError):
        BlockSmootherConfig(alpha=0.0)
    with pytest.raises(ConfigError):
        BlockSmootherConfig(kind="braess_sarazin", a_hat_mode="abs_rowsum")
    assert BlockSmootherConfig(kind="simplec").effective_a_hat_mode() == "abs_rowsum"


def test_hierarchy_and_gmres_config_validation():
    with pytest.raises(ConfigError):
        HierarchyConfig(max_levels=0)
    with pytest.raises(ConfigError):
        HierarchyConfig(coarse_solver="x")
    with pytest.raises(ConfigError):
        GmresConfig(rel_tol=1.0)
    with pytest.raises(ConfigError):
        GmresConfig(restart=0)


def test_sparse_matrix_host_invariants():
    A = SparseMatrix.from_coo([0, 0, 1, 1], [1, 1, 0, 1], [1.0, 2.0, 1e-301, 4.0], (2, 2))
    assert A.nnz == 2 and list(A.values) == [3.0, 4.0]
    with pytest.raises(ValueError):
        A.values[0] = 1.0


@pytest.mark.parametrize("dim", [2, 3])
def test_element_stiffness_rigid_modes(dim):
    Ke = element_stiffness(dim, [0.1] * dim, 1.0, 0.3)
    w = np.linalg.eigvalsh(Ke)
    assert np.sum(np.abs(w) < 1e-10) == (3 if dim == 2 else 6)
    assert np.abs(Ke - Ke.T).max() < 1e-15


def test_mortar_partition_of_unity():
    xs, xm = np.linspace(0, 2, 31), np.linspace(0, 2, 33)
    D, M = mortar_1d(xs, xm)
    assert np.allclose(D.sum(1), M.sum(1), atol=1e-15)
    assert abs(D.sum() - 2.0) < 1e-14


@pytest.mark.parametrize("name,dim,n_lam", [("C1", 2, 62), ("C3", 3, 11163)])
def test_config_sizes(name, dim, n_lam):
    g = generate(config_spec(name, 1 if dim == 2 else 4), assemble_K=(dim == 2))
    if dim == 2:
        assert g.n_u == 2048 and g.n_lam == n_lam
        assert abs(g.K - g.K.T).max() < 1e-15


def test_active_set_drawn_before_rhs():
    g = generate(config_spec("C4", 16))
    rng = np.random.default_rng(3)
    act = rng.random(len(g.slave_nodes)) < 0.5
    np.testing.assert_array_equal(act, g.active)
    np.testing.assert_array_equal(rng.uniform(-1, 1, g.n_u + g.n_lam), g.rhs)


@pytest.mark.parametrize("name", cases())
def test_native_host_aggregation_matches_reference(name):
    """C++ greedy / Alg. 1 on the reference node graph == reference aggregates."""
    z = load(name)
    ip, ix = z["L0_graph_indptr"], z["L0_graph_indices"]
    n = len(ip) - 1
    hkw = BY_NAME[name][3]
    g = NodeGraph(n, ip, ix, np.zeros(n, dtype=np.int8))
    ag = aggregate_greedy(g, HierarchyConfig(**hkw).min_agg_size)
    np.testing.assert_array_equal(ag.node_to_agg, z["L0_u_agg"])
    _, cfg, scale, *_ = BY_NAME[name]
    gen = generate(config_spec(cfg, scale))
    d = gen.dim
    D = SparseMatrix.from_scipy(gen.mortar_block)
    lmap = LagrangeMap(gen.slave_dofs.astype(np.int64), np.repeat(gen.slave_nodes, d).astype(np.int64),
                       np.arange(gen.n_lam, dtype=np.int64) // d)
    la = aggregate_lagrange(ag, D, lmap)
    np.testing.assert_array_equal(la.node_to_agg, z["L0_lam_agg"])


def test_native_greedy_matches_oracle_random_graphs():
    rng = np.random.default_rng(5)
    for t in range(5):
        n = int(rng.integers(50, 400))
        A = scipy.sparse.random(n, n, density=4.0 / n, random_state=int(rng.integers(1 << 30)), format="csr")
        A = A + A.T
        A.setdiag(0)
        A.eliminate_zeros()
        A.sort_indices()
        for ms in (1, 3, 6):
            ag = aggregate_greedy(NodeGraph(n, A.indptr, A.indices, np.zeros(n, np.int8)), ms)
            ref = O.greedy(A.indptr.astype(np.int64), A.indices.astype(np.int64), n, ms)
            np.testing.assert_array_equal(ag.node_to_agg, ref.node_to_agg)
            assert ag.singleton_count == ref.singletons


@pytest.mark.parametrize("name,scale,bs", [("C4", 16, 3), ("C2", 8, 2)])
def test_oracle_node_colouring_is_valid(name, scale, bs):
    """The MC-SGS predictor's node colouring: no two coupled nodes share a
    colour, every DOF takes its node's colour, and the structured hex8 / Q1
    stencils need 8 / 4 colours under natural-order greedy."""
    g = generate(config_spec(name, scale))
    oop, ometa, _ = O.system_from_generated(g)
    assert O.node_block(ometa) == bs
    K = oop.K
    col = O.greedy_colors(K, bs)
    assert np.array_equal(col, np.repeat(col[::bs], bs))
    rows = np.repeat(np.arange(K.shape[0]), np.diff(K.indptr))
    off = (rows // bs) != (K.indices // bs)
    assert not np.any(col[rows[off]] == col[K.indices[off]])
    assert col.max() + 1 == (8 if bs == 3 else 4)


def test_oracle_mcgs_block_equals_permuted_ssor():
    """mcgs(block) is the reference SSOR on K renumbered colour-major, node
    by node, DOFs in order (the GPU kernels' visiting order)."""
    g = generate(config_spec("C4", 16))
    oop, ometa, _ = O.system_from_generated(g)
    K = oop.K
    b = np.random.default_rng(0).standard_normal(K.shape[0])
    x = np.random.default_rng(1).standard_normal(K.shape[0])
    P = O.Point(O.PointCfg("mcgs", 2, 0.9, block=3), K)
    col = O.greedy_colors(K, 3)
    perm = np.lexsort((np.arange(K.shape[0]), col))
    S = O.Point(O.PointCfg("sgs", 2, 0.9), O.canon(K[perm][:, perm]))
    ref = np.empty_like(x)
    ref[perm] = S.smooth(x[perm], b[perm])
    np.testing.assert_array_equal(P.smooth(x, b), ref)


def test_oracle_mcilu0_colour_structure():
    """mcilu0 is the reference ILU(0) on S~ renumbered colour-major: rows of
    one colour are uncoupled, so every strictly lower factor entry reaches an
    earlier colour and every strictly upper one a later colour -- the property
    that lets the GPU run both triangular solves one colour per pass."""
    g = generate(config_spec("C4", 16))
    oop, ometa, rhs = O.system_from_generated(g)
    sm = O.Block(O.BlockCfg(kind="simple", alpha=0.8, predictor=O.PointCfg("jacobi", 1, 0.6),
                             corrector=O.PointCfg("mcilu0", 2)), oop)
    S = sm.S
    P = sm.corr
    col = O.greedy_colors(S)
    perm = np.argsort(col, kind="stable")
    Sp = O.canon(S[perm][:, perm])
    rows = np.repeat(np.arange(Sp.shape[0]), np.diff(Sp.indptr))
    cr, cc = col[perm][rows], col[perm][Sp.indices]
    off = rows != Sp.indices
    assert np.all(cr[off] != cc[off])
    assert np.all((cc < cr)[off & (Sp.indices < rows)])
    assert np.all((cc > cr)[off & (Sp.indices > rows)])
    # two sweeps from zero: x1 = M^-1 b, x2 = x1 + M^-1 (b - S x1), M = LU on the permuted S~
    b = np.random.default_rng(0).standard_normal(S.shape[0])
    one = O.Point(O.PointCfg("mcilu0", 1), S)
    x1 = one.apply(b)
    x2 = x1 + one.apply(b - S @ x1)
    np.testing.assert_allclose(P.apply(b), x2, rtol=0, atol=1e-12 * np.abs(x2).max())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ilu0_factor_matches_oracle_bit_for_bit(seed):
    """smoothers.ilu0_factor (libcamg host factorization, the one the MC-ILU(0)
    corrector uses) == the reference ILU(0) restated in the oracle."""
    from paper_1912_09056_b200.smoothers import ilu0_factor
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 120))
    A = scipy.sparse.random(n, n, density=0.08, random_state=seed, format="csr")
    A = O.canon(A + A.T + scipy.sparse.diags(rng.uniform(2.0, 4.0, n)))
    M = SparseMatrix(n, n, A.indptr, A.indices, A.data)
    np.testing.assert_array_equal(ilu0_factor(M), O.ilu0_values(A))


def test_ilu0_factor_errors():
    from paper_1912_09056_b200.errors import SingularMatrixError
    from paper_1912_09056_b200.smoothers import ilu0_factor
    no_diag = SparseMatrix(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(SingularMatrixError, match="missing diagonal entry in row 0"):
        ilu0_factor(no_diag)
    # [[1, 1], [1, 1]]: the second pivot cancels to zero
    zero_piv = SparseMatrix(2, 2, [0, 2, 4], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    with pytest.raises(SingularMatrixError, match="zero pivot in row 1"):
        ilu0_factor(zero_piv)


def test_threaded_pivoted_qr_bit_identical():
    """The tentative prolongator's batched pivoted QR (libcamg host threads
    calling scipy's own LAPACK dgeqp3 / dorgqr, camg_qr_batch) equals
    scipy.linalg.qr(mode="economic", pivoting=True) -- the reference's call,
    transfer.py:120 -- bit for bit, for tall, square, wide and rank-deficient
    blocks."""
    import scipy.linalg
    from paper_1912_09056_b200 import transfer as T
    assert T._lapack_path() is not None, "scipy's OpenBLAS not found: the native QR path is not exercised"
    rng = np.random.default_rng(4)
    for (G, M, k) in ((25000, 16, 6), (3000, 81, 6), (500, 6, 6), (400, 4, 6), (2000, 9, 3), (50, 1, 3)):
        vecs = rng.standard_normal((30000, k))
        vecs[::5, 1] = 0.0
        vecs[::11] = vecs[1::11]  # repeated rows: rank-deficient blocks
        dofs = rng.integers(0, 30000, size=(G, M))
        Qr, Rr, Pr = scipy.linalg.qr(vecs[dofs], mode="economic", pivoting=True)
        q = np.empty((G, M, min(M, k)))
        R, P = T._pivoted_qr_into(vecs, dofs, q)
        assert np.array_equal(q, Qr) and np.array_equal(R, Rr) and np.array_equal(P, Pr), (G, M, k)

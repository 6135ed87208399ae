"""The drop-in boundary beyond single calls: re-entrant V-cycles on private
workspaces, GMRES with caller-owned workspaces,
GMRES over arbitrary callables and over the nested preconditioner through
the native solver (krylov.py:45-129, hierarchy.py:366-385), the reference
default smoother configuration (smoothers.py:44-50), and the reference's
setup report (hierarchy.py:251-269)."""

import sys
import threading

import numpy as np
import pytest

import camg_oracle as O
from _golden import GOLDEN, load

pytestmark = pytest.mark.gpu

sys.path.insert(0, GOLDEN)
from cases import BY_NAME  # noqa: E402

from paper_1912_09056_b200 import _native  # noqa: E402
from paper_1912_09056_b200.hierarchy import HierarchyConfig, fine_level_meta, nested_preconditioner, setup  # noqa: E402
from paper_1912_09056_b200.krylov import GmresConfig, GmresWorkspace, gmres, release_workspace  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def device():
    _native.require_device()


_S = {}


def system(cfg="C5", scale=10, skw=None, hkw=None):
    key = (cfg, scale, repr(skw), repr(hkw))
    if key not in _S:
        g = generate(config_spec(cfg, scale))
        op = saddle_operator(g)
        skw = skw or dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=PointSmootherConfig("jacobi", 1, 0.6),
                          corrector=PointSmootherConfig("mcilu0", 1, 1.0))
        H = setup(op, fine_level_meta(g), HierarchyConfig(**(hkw or dict(max_levels=3, max_coarse_size=50))),
                  BlockSmootherConfig(**skw))
        _S[key] = (g, op, H)
    return _S[key]


def test_apply_returns_a_fresh_result_each_call():
    """Every apply owns its result (the reference returns a new array)."""
    import torch
    g, op, H = system()
    rng = np.random.default_rng(1)
    r1 = torch.from_numpy(rng.standard_normal(H.n)).pin_memory()
    r2 = torch.from_numpy(rng.standard_normal(H.n)).pin_memory()
    z1 = H.apply(r1)
    z1c = z1.clone()
    z2 = H.apply(r2)
    assert z1.data_ptr() != z2.data_ptr()
    assert torch.equal(z1, z1c) and not torch.equal(z1, z2)
    out = torch.empty(H.n, dtype=torch.float64).pin_memory()
    assert H.apply(r1, out=out) is out and torch.equal(out, z1c)


def test_workspaces_on_concurrent_streams_equal_default():
    """Two workspaces applied concurrently on two streams give exactly the
    default workspace's results."""
    import torch
    g, op, H = system()
    rng = np.random.default_rng(2)
    rs = [torch.from_numpy(rng.standard_normal(H.n)).cuda() for _ in range(4)]
    ref = [H.apply_device(r).clone() for r in rs]
    ws = [H.workspace(), H.workspace()]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty_like(r) for r in rs]
    torch.cuda.synchronize()
    for rep in range(3):
        for i, r in enumerate(rs):
            with torch.cuda.stream(streams[i % 2]):
                H.apply_device(r, outs[i], ws[i % 2])
    torch.cuda.synchronize()
    for o, e in zip(outs, ref):
        assert torch.equal(o, e)


def test_workspaces_from_threads():
    """One hierarchy applied from several host threads, each on its own
    workspace and stream (captures serialise inside the library)."""
    import torch
    g, op, H = system()
    rng = np.random.default_rng(3)
    rs = [torch.from_numpy(rng.standard_normal(H.n)).cuda() for _ in range(4)]
    ref = [H.apply_device(r).clone() for r in rs]
    torch.cuda.synchronize()
    res, errs = [None] * 4, []

    def work(i):
        try:
            s = torch.cuda.Stream()
            w = H.workspace()
            with torch.cuda.stream(s):
                o = torch.empty_like(rs[i])
                for _ in range(3):
                    H.apply_device(rs[i], o, w)
                s.synchronize()
            res[i] = o
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for o, e in zip(res, ref):
        assert torch.equal(o, e)


def test_workspace_of_another_hierarchy_is_rejected():
    g, op, H = system()
    g2, op2, H2 = system("C1", 1, hkw=dict(max_levels=2, max_coarse_size=1))
    import torch
    r = torch.zeros(H.n, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        H.apply_device(r, None, H2.workspace())


def test_gmres_workspaces_and_release():
    g, op, H = system()
    cfg = GmresConfig(rel_tol=1e-8, max_iters=200, restart=100)
    x0, r0 = gmres(op.apply_merged, H.apply, g.rhs, cfg)
    release_workspace()
    for store_z in (True, False, None):
        ws = GmresWorkspace(H.n, 100, store_z)
        x, rep = gmres(op.apply_merged, H.apply, g.rhs, cfg, workspace=ws, vcycle_workspace=H.workspace())
        assert rep.iterations == r0.iterations
        assert np.linalg.norm(x - x0) <= 1e-10 * np.linalg.norm(x0)
    with pytest.raises(Exception):
        gmres(op.apply_merged, H.apply, g.rhs, cfg, workspace=GmresWorkspace(H.n - 1, 100))


def test_gmres_chunked_orthogonalisation(monkeypatch):
    """Restarts longer than one k_ortho launch holds (> 2048 basis vectors)
    run the CGS2 passes in chunks; forced to chunks of 7 here."""
    g, op, H = system()
    cfg = GmresConfig(rel_tol=1e-8, max_iters=200, restart=100)
    x0, r0 = gmres(op.apply_merged, H.apply, g.rhs, cfg, workspace=GmresWorkspace(H.n, 100))
    monkeypatch.setenv("CAMG_ORTHO_CHUNK", "7")
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, cfg, workspace=GmresWorkspace(H.n, 100))
    assert abs(rep.iterations - r0.iterations) <= 1
    assert np.linalg.norm(x - x0) <= 1e-7 * np.linalg.norm(x0)


def test_gmres_over_python_callables_runs_native_loop():
    """apply_A / apply_Minv as plain callables (numpy on host, torch on
    device) are called back from the native solver; the result matches the
    natively bound operator + hierarchy."""
    import torch
    g, op, H = system()
    A = op.merged().to_scipy()
    cfg = GmresConfig(rel_tol=1e-8, max_iters=200, restart=100)
    x0, r0 = gmres(op.apply_merged, H.apply, g.rhs, cfg)
    x1, r1 = gmres(lambda v: A @ v, lambda v: H.apply(v), g.rhs, cfg)            # host numpy callables
    assert isinstance(x1, np.ndarray) and r1.iterations == r0.iterations
    assert np.linalg.norm(x1 - x0) <= 1e-9 * np.linalg.norm(x0)
    bd = torch.from_numpy(g.rhs).cuda()
    x2, r2 = gmres(lambda v: op.apply_merged(v), lambda v: H.apply(v), bd, cfg)  # device callables
    assert x2.is_cuda and r2.iterations == r0.iterations
    # oracle: same problem, the oracle's V-cycle emulation
    _, orep = O.gmres(lambda t: A @ t, lambda t: H.apply(t), g.rhs, 1e-8, 200, 100)
    assert abs(orep.iterations - r0.iterations) <= 1
    with pytest.raises(ZeroDivisionError):  # a callback's exception surfaces unchanged
        gmres(lambda v: A @ v, lambda v: 1 / 0, g.rhs, cfg)


def test_nested_preconditioner_gmres_is_native():
    """GMRES over NestedPreconditioner.apply binds the level natively (no
    Python in the Krylov loop); equals the callback form."""
    g = generate(config_spec("C5", 25))
    op = saddle_operator(g)
    skw = BY_NAME["c5s_simple"][4]
    NP = nested_preconditioner(op, fine_level_meta(g),
                               BlockSmootherConfig(kind="simple", alpha=0.8, outer_sweeps=1,
                                                   predictor=PointSmootherConfig("jacobi", 1, 0.8),
                                                   corrector=PointSmootherConfig("jacobi", 1, 0.8)),
                               HierarchyConfig(max_levels=3, max_coarse_size=50), PointSmootherConfig("jacobi", 2, 0.6))
    assert skw  # the golden case family (nested_c5s) uses this system
    cfg = GmresConfig(rel_tol=1e-8, max_iters=200, restart=100)
    calls = []
    x0, r0 = gmres(op.apply_merged, NP.apply, g.rhs, cfg)
    x1, r1 = gmres(op.apply_merged, lambda v: (calls.append(1), NP.apply(v))[1], g.rhs, cfg)
    assert calls and r1.iterations == r0.iterations
    assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0)
    z = load("nested_c5s")
    assert abs(r0.iterations - int(z["gmres_iterations"])) <= 1


def test_reference_default_block_smoother_runs_reference_algorithm():
    """BlockSmootherConfig() (reference default: sgs predictor, ilu0
    corrector, smoothers.py:44-50) runs the reference's lexicographic inner
    solves on the GPU: the V-cycle equals the oracle's (1e-10), GMRES
    iterations equal within +-1, and the explicit multicolour variants are
    the separate, faster choice compared by convergence."""
    import camg_oracle as O
    g = generate(config_spec("C5", 10))
    op = saddle_operator(g)
    meta = fine_level_meta(g)
    hc = HierarchyConfig(max_levels=3, max_coarse_size=50)
    Hd = setup(op, meta, hc, BlockSmootherConfig())
    assert "GPU variants" not in Hd.report
    assert Hd.levels[0].smoother.cfg == BlockSmootherConfig()
    assert Hd.level_info(0)["pred_path"] == "lex_trsv" and Hd.level_info(0)["corr_path"] == "lex_trsv"
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(max_levels=3, max_coarse_size=50), O.BlockCfg())
    v, ref = Hd.apply(g.rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    x, rep = gmres(op.apply_merged, Hd.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 200, 100)
    assert rep.converged and abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)
    He = setup(op, meta, hc, BlockSmootherConfig(predictor=PointSmootherConfig("mcgs", 1, 1.0),
                                                 corrector=PointSmootherConfig("mcilu0", 1, 1.0)))
    _, rep_e = gmres(op.apply_merged, He.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    assert rep_e.converged


def test_exact_a_hat_mode_matches_oracle():
    """a_hat_mode="exact" (test-scale, smoothers.py:233-236, 272-273): S~ from
    the dense K inverse, A^-1 = K^-1 in the step, with a direct predictor, on
    random well-conditioned saddle systems (the reference's random_saddle)."""
    import scipy.sparse
    import camg_oracle as O
    from paper_1912_09056_b200.saddle import SaddleOperator
    from paper_1912_09056_b200.smoothers import BlockSmoother
    from paper_1912_09056_b200.sparse import BlockVector, SparseMatrix
    rng = np.random.default_rng(3)
    for n_u, n_l in ((30, 8), (120, 20)):
        G = rng.standard_normal((n_u, n_u))
        K = G @ G.T + n_u * np.eye(n_u)
        B1 = rng.standard_normal((n_u, n_l))
        B2 = rng.standard_normal((n_l, n_u))
        G2 = rng.standard_normal((n_l, n_l))
        Cz = G2 @ G2.T + n_l * np.eye(n_l)
        op = SaddleOperator(*(SparseMatrix.from_dense(m) for m in (K, B1, B2, Cz)))
        oop = O.Saddle(*(O.canon(scipy.sparse.csr_matrix(m)) for m in (K, B1, B2, Cz)))
        x0, b = rng.standard_normal(n_u + n_l), rng.standard_normal(n_u + n_l)
        for kind, alpha, pred in (("uzawa", 0.7, "direct"), ("simple", 0.8, "direct"), ("simple", 0.8, "sgs")):
            cfg = BlockSmootherConfig(kind=kind, alpha=alpha, outer_sweeps=2, predictor=PointSmootherConfig(pred),
                                      corrector=PointSmootherConfig("ilu0"), a_hat_mode="exact")
            got = BlockSmoother(cfg, op).sweep(BlockVector.from_merged(x0, n_u), BlockVector.from_merged(b, n_u)).merged()
            ob = O.Block(O.BlockCfg(kind=kind, alpha=alpha, outer_sweeps=2, predictor=O.PointCfg(pred),
                                    corrector=O.PointCfg("ilu0"), a_hat_mode="exact"), oop)
            ru, rl = ob.sweep(x0[:n_u], x0[n_u:], b[:n_u], b[n_u:])
            ref = np.concatenate([ru, rl])
            assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref), (kind, pred, np.linalg.norm(got - ref))


@pytest.mark.parametrize("name", ["c1_uzawa_jac2", "c2s_simplec", "c3s_bs", "c4s_uzawa", "c5s_simple",
                                  "c3s_bs_blocksmoother", "c5s_simple_direct"])
def test_setup_report_matches_reference(name):
    """H.report is the reference's report string (hierarchy.py:251-269)."""
    from test_gpu_parity import gpu_hier
    z = load(name)
    _, _, H = gpu_hier(name)
    assert H.report == str(z["report"])


@pytest.mark.parametrize("cfg,scale,levels", [("C2", 4, 3), ("C5", 10, 2), ("C1", 1, 2)])
def test_device_coarse_factorization_matches_lapack(cfg, scale, levels, monkeypatch):
    """camg_hierarchy_coarse_factor (device LU with partial pivoting + inverse,
    the default) against host LAPACK factors (CAMG_COARSE_HOST=1,
    scipy.linalg.lu_factor as hierarchy.py:242-249): same pivots on these
    systems, coarse solves within 1e-12, V-cycles within 1e-11."""
    import scipy.linalg
    from paper_1912_09056_b200.sparse import BlockVector
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    meta = fine_level_meta(g)
    hc = HierarchyConfig(max_levels=levels, max_coarse_size=50)
    sc = BlockSmootherConfig(kind="uzawa", alpha=0.6, predictor=PointSmootherConfig("jacobi", 2, 0.6),
                             corrector=PointSmootherConfig("jacobi", 1, 0.6))
    out = {}
    for host in ("1", "0"):
        monkeypatch.setenv("CAMG_COARSE_HOST", host)
        H = setup(op, meta, hc, sc)
        out[host] = (H, H.apply(g.rhs))
    Hd = out["0"][0]
    cop = Hd.levels[-1].op
    dense = cop.merged_dense()
    lu = scipy.linalg.lu_factor(dense)
    b = np.random.default_rng(1).standard_normal(cop.total_rows)
    xb = Hd.solve_coarsest(BlockVector.zeros(cop.n_u, cop.n_lam), BlockVector.from_merged(b, cop.n_u)).merged()
    ref = scipy.linalg.lu_solve(lu, b)
    assert np.linalg.norm(xb - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(out["0"][1] - out["1"][1]) <= 1e-11 * np.linalg.norm(out["1"][1])


def test_device_lambda_max_matches_host_norms():
    """camg_lambda_max (device norms, for non-Python hosts) against the
    package's estimate_lambda_max (host numpy norms, bit-identical to the
    reference, transfer.py:148-161): equal to 1e-13."""
    import ctypes as C
    from paper_1912_09056_b200.transfer import estimate_lambda_max
    g = generate(config_spec("C4", 8))
    op = saddle_operator(g)
    ref = estimate_lambda_max(op.K)
    out = C.c_double()
    _native.call("camg_lambda_max", op.K.device, None, 10, C.byref(out))
    assert abs(out.value - ref) <= 1e-13 * ref

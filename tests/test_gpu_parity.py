"""GPU parity: the CUDA path (libcamg via the package API) against the
reference's golden fixtures and against the oracle run live on the same
machine.  Bars (BASELINE.json north_star): per-level operators within 1e-12
relative Frobenius (patterns exact), aggregates bit-exact, V-cycle within
1e-10 relative 2-norm, GMRES iteration count equal or within +-1."""

import sys

import numpy as np
import pytest
import scipy.sparse

import camg_oracle as O
from _golden import GOLDEN, cases, csr, load

pytestmark = pytest.mark.gpu

sys.path.insert(0, GOLDEN)
from cases import BY_NAME  # noqa: E402

from paper_1912_09056_b200 import _native  # noqa: E402
from paper_1912_09056_b200.errors import ConfigError  # noqa: E402
from paper_1912_09056_b200.hierarchy import HierarchyConfig, fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.krylov import GmresConfig, gmres  # noqa: E402
from paper_1912_09056_b200.problem import assemble_K_device, config_spec, generate, saddle_operator  # noqa: E402
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig  # noqa: E402
from paper_1912_09056_b200.sparse import (  # noqa: E402
    SparseMatrix,
    extract_diagonal,
    galerkin_triple,
    sp_matmul,
    sp_transpose,
    spmv,
)


@pytest.fixture(scope="module", autouse=True)
def device():
    _native.require_device()


def block_cfg(skw):
    kw = dict(skw)
    for k in ("predictor", "corrector"):
        if k in kw:
            kw[k] = PointSmootherConfig(*kw[k])
    return BlockSmootherConfig(**kw)


def oracle_block_cfg(skw):
    kw = dict(skw)
    for k in ("predictor", "corrector"):
        if k in kw:
            kw[k] = O.PointCfg(*kw[k])
    return O.BlockCfg(**kw)


def rel_fro(A, B):
    A, B = scipy.sparse.csr_matrix(A), scipy.sparse.csr_matrix(B)
    d = scipy.sparse.linalg.norm(A - B) if (A - B).nnz else 0.0
    nb = scipy.sparse.linalg.norm(B)
    return d / nb if nb else d


def same_pattern(A, B):
    A, B = scipy.sparse.csr_matrix(A), scipy.sparse.csr_matrix(B)
    return A.shape == B.shape and np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)


# every golden case runs on the GPU with the reference's own inner solves
# (c2s_simple_sgs_ilu: lexicographic sgs predictor and ilu0 corrector)
GPU_CASES = list(cases())


# ---------------------------------------------------------------------------
# kernels


def test_sparse_kernels_vs_reference_golden():
    z = np.load(GOLDEN + "/kernels.npz")
    for t in range(4):
        A, Asq, B = csr(z, f"t{t}_A"), csr(z, f"t{t}_Asq"), csr(z, f"t{t}_B")
        dA, dAsq, dB = SparseMatrix.from_scipy(A), SparseMatrix.from_scipy(Asq), SparseMatrix.from_scipy(B)
        y = spmv(dA, z[f"t{t}_x"])
        ref = z[f"t{t}_spmv"]
        assert np.abs(y - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())
        assert same_pattern(sp_transpose(dA).to_scipy(), csr(z, f"t{t}_AT"))
        assert np.array_equal(sp_transpose(dA).values, csr(z, f"t{t}_AT").data)
        AB = sp_matmul(dAsq, dB).to_scipy()
        assert same_pattern(AB, csr(z, f"t{t}_AB")) and np.array_equal(AB.data, csr(z, f"t{t}_AB").data)
        RAP = galerkin_triple(sp_transpose(dB), dAsq, dB).to_scipy()
        assert same_pattern(RAP, csr(z, f"t{t}_RAP")) and np.array_equal(RAP.data, csr(z, f"t{t}_RAP").data)
        np.testing.assert_array_equal(extract_diagonal(dAsq), z[f"t{t}_diag"])
        np.testing.assert_allclose(extract_diagonal(dAsq, "abs_rowsum"), z[f"t{t}_absrow"], rtol=1e-15)


def test_spgemm_bit_exact_vs_scipy_random():
    rng = np.random.default_rng(11)
    for t in range(6):
        m, k, n = rng.integers(50, 600, size=3)
        dens = float(rng.uniform(0.01, 0.2))
        A = O.canon(scipy.sparse.random(m, k, density=dens, random_state=int(rng.integers(1 << 30))))
        B = O.canon(scipy.sparse.random(k, n, density=dens, random_state=int(rng.integers(1 << 30))))
        C = sp_matmul(SparseMatrix.from_scipy(A), SparseMatrix.from_scipy(B)).to_scipy()
        ref = O.matmul(A, B)
        assert same_pattern(C, ref) and np.array_equal(C.data, ref.data)
        Sq = O.canon(scipy.sparse.random(k, k, density=dens, random_state=int(rng.integers(1 << 30))))
        P = O.canon(scipy.sparse.random(k, n, density=dens, random_state=int(rng.integers(1 << 30))))
        R = O.transpose(P)
        G = galerkin_triple(SparseMatrix.from_scipy(R), SparseMatrix.from_scipy(Sq), SparseMatrix.from_scipy(P))
        ref = O.rap(R, Sq, P)
        assert same_pattern(G.to_scipy(), ref) and np.array_equal(G.to_scipy().data, ref.data)


def test_spgemm_overflow_rows_use_global_path():
    """Rows with more unique columns than the shared-memory hash holds."""
    rng = np.random.default_rng(3)
    A = O.canon(scipy.sparse.random(40, 3000, density=0.5, random_state=1))
    B = O.canon(scipy.sparse.random(3000, 5000, density=0.01, random_state=2))
    C = sp_matmul(SparseMatrix.from_scipy(A), SparseMatrix.from_scipy(B)).to_scipy()
    ref = O.matmul(A, B)
    assert same_pattern(C, ref) and np.array_equal(C.data, ref.data)
    P = O.canon(scipy.sparse.random(3000, 2500, density=0.02, random_state=4))
    Sq = O.canon(scipy.sparse.random(3000, 3000, density=0.05, random_state=5))
    G = galerkin_triple(SparseMatrix.from_scipy(O.transpose(P)), SparseMatrix.from_scipy(Sq),
                        SparseMatrix.from_scipy(P)).to_scipy()
    ref = O.rap(O.transpose(P), Sq, P)
    assert same_pattern(G, ref) and np.array_equal(G.data, ref.data)


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C3", 8), ("C4", 8), ("C2", 4)])
def test_device_assembly_equals_host(name, scale):
    g = generate(config_spec(name, scale))
    Kd = assemble_K_device(g).to_scipy()
    assert same_pattern(Kd, g.K) and np.array_equal(Kd.data, g.K.data)


# ---------------------------------------------------------------------------
# hierarchy parity against the reference's golden outputs

_H = {}


def gpu_hier(name):
    if name not in _H:
        _, cfg, scale, hkw, skw, restart, max_iters = BY_NAME[name]
        g = generate(config_spec(cfg, scale))
        op = saddle_operator(g)
        H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
        _H[name] = (g, op, H)
    return _H[name]


@pytest.mark.parametrize("name", GPU_CASES)
def test_hierarchy_operators_and_aggregates(name):
    z = load(name)
    g, op, H = gpu_hier(name)
    assert H.num_levels == int(z["num_levels"])
    np.testing.assert_array_equal(H.levels[0].info["u_agg"], z["L0_u_agg"])
    np.testing.assert_array_equal(H.levels[0].info["lam_agg"], z["L0_lam_agg"])
    for l, lvl in enumerate(H.levels):
        for blk in ("K", "B1", "B2", "Cz"):
            A = getattr(lvl.op, blk).to_scipy()
            R = csr(z, f"L{l}_{blk}")
            assert same_pattern(A, R), (l, blk)
            assert rel_fro(A, R) <= 1e-12, (l, blk, rel_fro(A, R))
        S = lvl.smoother.schur.S_tilde.to_scipy()
        Sr = csr(z, f"L{l}_Stilde")
        assert same_pattern(S, Sr) and rel_fro(S, Sr) <= 1e-12, l
        if lvl.transfer is not None:
            for key, P in (("Pu", lvl.transfer.P_u), ("Plam", lvl.transfer.P_lam)):
                Pr = csr(z, f"L{l}_{key}")
                assert same_pattern(P.to_scipy(), Pr), (l, key)
                assert rel_fro(P.to_scipy(), Pr) <= 1e-12
            assert lvl.info["lambda_max"] == pytest.approx(float(z[f"L{l}_lambda_max"]), rel=1e-13)
            assert lvl.info["u_aggregates"] == int(z[f"L{l}_u_aggs"])
            assert lvl.info["lam_aggregates"] == int(z[f"L{l}_lam_aggs"])
            assert lvl.info["u_singletons"] == int(z[f"L{l}_u_singletons"])
            assert lvl.info["lam_overlap_touches"] == int(z[f"L{l}_lam_overlaps"])


@pytest.mark.parametrize("name", GPU_CASES)
def test_sweep_and_vcycle_vs_reference(name):
    z = load(name)
    g, op, H = gpu_hier(name)
    sm = H.levels[0].smoother
    out = sm.sweep_merged(z["sweep_x"], z["sweep_b"]).cpu().numpy()
    ref = z["sweep_out"]
    assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    for kin, kout in (("rhs", "vcycle_out"), ("vcycle_rand_in", "vcycle_rand_out")):
        v = H.apply(z[kin])
        ref = z[kout]
        assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref), np.linalg.norm(v - ref) / np.linalg.norm(ref)


@pytest.mark.parametrize("name", GPU_CASES)
def test_gmres_iterations_vs_reference(name):
    z = load(name)
    g, op, H = gpu_hier(name)
    cfg = GmresConfig(rel_tol=1e-8, max_iters=int(z["gmres_max_iters"]), restart=int(z["gmres_restart"]))
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, cfg)
    assert abs(rep.iterations - int(z["gmres_iterations"])) <= 1, (rep.iterations, int(z["gmres_iterations"]))
    assert rep.converged == bool(z["gmres_converged"])
    hist = np.asarray(rep.residual_history)
    assert hist[0] == pytest.approx(float(z["gmres_history"][0]), rel=1e-13)
    if rep.converged:
        A = csr(z, "A")
        assert np.linalg.norm(g.rhs - A @ x) <= 2e-8 * np.linalg.norm(g.rhs)


@pytest.mark.parametrize("kind,sweeps,damping", [("sgs", 1, 1.0), ("sgs", 2, 0.9), ("ilu0", 1, 1.0),
                                                 ("ilu0", 3, 1.0), ("jacobi", 2, 0.7), ("direct", 1, 1.0)])
def test_point_smoother_reference_semantics(kind, sweeps, damping):
    """PointSmoother with the reference's lexicographic sgs / ilu0 (sync-free
    triangular solves), jacobi and direct, on K and on S~ of a golden case,
    against the oracle's restatement of smoothers.py:141-199."""
    from paper_1912_09056_b200.smoothers import PointSmoother
    g, op, H = gpu_hier("c2s_simple_sgs_ilu")
    rng = np.random.default_rng(7)
    for A in (op.K, H.levels[0].smoother.schur.S_tilde):
        if kind == "direct" and A.num_rows > 3000:
            continue
        As = A.to_scipy()
        x0, b = rng.standard_normal(A.num_rows), rng.standard_normal(A.num_rows)
        P = PointSmoother(PointSmootherConfig(kind, sweeps, damping), A)
        Q = O.Point(O.PointCfg(kind, sweeps, damping), As)
        for x in (None, x0):
            got = P.apply(b) if x is None else P.smooth(x, b)
            ref = Q.apply(b) if x is None else Q.smooth(x, b)
            assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref), (kind, np.linalg.norm(got - ref))


def test_reference_default_block_smoother_is_lexicographic():
    """BlockSmootherConfig() (sgs predictor, ilu0 corrector, smoothers.py:44-50)
    runs the reference's lexicographic sweeps: no substitution, no report line,
    and the sweep equals the oracle's."""
    g, op, _ = gpu_hier(GPU_CASES[0])
    meta = fine_level_meta(g)
    H = setup(op, meta, HierarchyConfig(max_levels=2), BlockSmootherConfig(kind="simple", predictor=PointSmootherConfig("sgs")))
    assert H.levels[0].smoother.substitutions == []
    assert "GPU variants" not in H.report
    info = H.level_info(0)
    assert info["pred_path"] == "lex_trsv" and info["corr_path"] == "lex_trsv"
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(max_levels=2), O.BlockCfg(kind="simple", predictor=O.PointCfg("sgs")))
    v, ref = H.apply(rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)


# ---------------------------------------------------------------------------
# larger systems against the oracle run live (same machine => same LAPACK)

LIVE = [
    ("C3", 4, dict(max_levels=3, max_coarse_size=50),
     dict(kind="braess_sarazin", alpha=1.0 / 0.7, corrector=("jacobi", 1, 0.7))),
    ("C2", 2, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8))),
    ("C4", 8, dict(max_levels=3, max_coarse_size=50),
     dict(kind="uzawa", alpha=0.6, predictor=("jacobi", 2, 0.6), corrector=("jacobi", 1, 0.6))),
    ("C5", 10, dict(max_levels=4, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8))),
]


@pytest.mark.parametrize("cfg,scale,hkw,skw", LIVE)
def test_live_oracle_parity(cfg, scale, hkw, skw):
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    assert H.num_levels == len(OH.levels)
    for l, (lv, olv) in enumerate(zip(H.levels, OH.levels)):
        for blk in ("K", "B1", "B2", "Cz"):
            A, R = getattr(lv.op, blk).to_scipy(), getattr(olv.op, blk)
            assert same_pattern(A, R), (l, blk)
            assert rel_fro(A, R) <= 1e-12
        if lv.transfer is not None:
            np.testing.assert_array_equal(lv.info["u_agg"], olv.info["u_agg"])
            np.testing.assert_array_equal(lv.info["lam_agg"], olv.info["lam_agg"])
            assert same_pattern(lv.transfer.P_u.to_scipy(), olv.P_u)
    v = H.apply(rhs)
    ref = OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 150, 50)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=150, restart=50))
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)


# the benchmarked smoother (bench.solver_for C2-C5: SIMPLE(0.8)x3, Jacobi(1,0.6)
# predictor, MC-ILU(0) corrector) on small systems with every size-gated
# path forced on
BENCH_SMOOTHER_CASES = [
    ("C5", 10, dict(max_levels=4, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.6), corrector=("mcilu0", 1, 1.0))),
    ("C3", 4, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.6), corrector=("mcilu0", 1, 1.0))),
]


@pytest.mark.parametrize("masked", ["1", "0"])
@pytest.mark.parametrize("cfg,scale,hkw,skw", [LIVE[2], LIVE[3], LIVE[1]] + BENCH_SMOOTHER_CASES)
def test_sell_block_path_parity(cfg, scale, hkw, skw, masked, monkeypatch):
    """Force the block SELL-32 mirror on every level that has uniform node
    blocks (masked slots, the default, and full blocks) and check the
    V-cycle / GMRES against the oracle."""
    import paper_1912_09056_b200.hierarchy as hmod
    monkeypatch.setattr(hmod, "SELL_MIN_ROWS", 0)
    monkeypatch.setenv("CAMG_SELL_MASKED", masked)
    monkeypatch.setenv("CAMG_SELL_MIN_BLOCK_ROWS", "0")  # block SELL restriction too
    if masked == "1":  # one lane per row everywhere, so small levels get masked slots too
        monkeypatch.setenv("CAMG_SELL_PAIR", "0")
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    v = H.apply(rhs)
    ref = OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    y = op.apply_merged(rhs)
    assert np.linalg.norm(y - A @ rhs) <= 1e-13 * np.linalg.norm(A @ rhs)
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 150, 50)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=150, restart=50))
    assert abs(rep.iterations - orep.iterations) <= 1


@pytest.mark.parametrize("cfg,scale,bs", [("C3", 1, 3), ("C5", 3, 3)])
def test_masked_sell_bit_identical_to_full_blocks(cfg, scale, bs, monkeypatch):
    """Masked slots (only the union pattern of each slot stored) perform the
    same FMA sequence as full blocks on their stored zeros: the merged SpMV is
    bit-identical, and matches scipy.  (Sizes with enough slices for the
    one-lane-per-row kernel, where masked slots are used.)"""
    import torch
    from paper_1912_09056_b200.sparse import empty, ptr, stream_ptr
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    A = op.merged()
    n = A.num_rows
    x = torch.from_numpy(np.random.default_rng(7).standard_normal(n)).cuda()
    out = {}
    for m in ("0", "1"):
        monkeypatch.setenv("CAMG_SELL_MASKED", m)
        _native.call("camg_csr_attach_blocks", A.device, bs, op.n_u)
        y = empty(n)
        _native.call("camg_spmv", A.device, 1.0, ptr(x), 0.0, ptr(y), stream_ptr())
        torch.cuda.synchronize()
        out[m] = y.cpu().numpy()
    np.testing.assert_array_equal(out["0"], out["1"])
    ref = A.to_scipy() @ x.cpu().numpy()
    assert np.linalg.norm(out["1"] - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("cfg,scale,bs", [("C3", 1, 3), ("C5", 3, 3)])
def test_shared_value_groups_bit_identical(cfg, scale, bs, monkeypatch):
    """Masked mirrors keep one copy of bit-identical slots (the interior
    stencil of a structured mesh): the sharing engages on the configs' fine
    operators, stores a small fraction of the value groups, and the merged
    SpMV is bit-identical to the streaming layout (CAMG_SELL_DEDUP=0) and to
    full blocks."""
    import ctypes as C
    import torch
    from paper_1912_09056_b200.sparse import empty, ptr, stream_ptr
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    A = op.merged()
    n = A.num_rows
    x = torch.from_numpy(np.random.default_rng(11).standard_normal(n)).cuda()
    out, groups = {}, {}
    for m in ("0", "1"):
        monkeypatch.setenv("CAMG_SELL_DEDUP", m)
        _native.call("camg_csr_attach_blocks", A.device, bs, op.n_u)
        kept, full = C.c_int64(0), C.c_int64(0)
        _native.call("camg_csr_value_groups", A.device, C.byref(kept), C.byref(full))
        groups[m] = (kept.value, full.value)
        y = empty(n)
        _native.call("camg_spmv", A.device, 1.0, ptr(x), 0.0, ptr(y), stream_ptr())
        torch.cuda.synchronize()
        out[m] = y.cpu().numpy()
    assert groups["0"][0] == groups["0"][1] == groups["1"][1]
    assert groups["1"][0] * 4 < groups["1"][1], groups
    np.testing.assert_array_equal(out["0"], out["1"])
    ref = A.to_scipy() @ x.cpu().numpy()
    assert np.linalg.norm(out["1"] - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("cfg,scale", [("C3", 1), ("C5", 3), ("C4", 4), ("C2", 1)])
def test_uniform_slice_loop_bit_identical(cfg, scale, monkeypatch):
    """Masked 3x3 mirror variants.  Offset-aligned slots (slot j of a slice =
    the block at its j-th column offset, explicit zero blocks at boundary
    nodes; CAMG_SELL_ALIGN) make the slices across mesh-row ends linear and
    lane-uniform but for one or two lanes; uniform slices (CAMG_SELL_USLICE)
    run a loop without descriptor decoding, neighbouring ones in pairs (=2).
    They engage on the configs' fine operators, and the merged SpMV, a whole
    block-smoother sweep and the V-cycle are bit-identical across all variants."""
    import ctypes as C
    import torch
    from paper_1912_09056_b200.sparse import empty, ptr, stream_ptr
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    A = op.merged()
    n = A.num_rows
    bs = 2 if cfg == "C2" else 3
    x = torch.from_numpy(np.random.default_rng(12).standard_normal(n)).cuda()
    # (CAMG_SELL_ALIGN, CAMG_SELL_USLICE, CAMG_SELL_WITEMS: host-made work items without the groups' followers)
    variants = [("0", "0", "1"), ("0", "2", "1"), ("1", "0", "1"), ("1", "1", "1"), ("1", "2", "0"), ("1", "2", "1")]
    out, counts = {}, {}
    for v in variants:
        monkeypatch.setenv("CAMG_SELL_ALIGN", v[0])
        monkeypatch.setenv("CAMG_SELL_USLICE", v[1])
        monkeypatch.setenv("CAMG_SELL_WITEMS", v[2])
        _native.call("camg_csr_attach_blocks", A.device, bs, op.n_u)
        c = (C.c_int64 * 5)()
        _native.call("camg_csr_uniform_slices", A.device, c)
        counts[v] = tuple(c)
        y = empty(n)
        _native.call("camg_spmv", A.device, 1.0, ptr(x), 0.0, ptr(y), stream_ptr())
        torch.cuda.synchronize()
        out[v] = y.cpu().numpy()
    base = ("0", "0", "1")
    assert counts[base][1:] == (0, 0, 0, 0) and counts[("1", "0", "1")][1] == 0
    if bs == 3 and cfg != "C4":  # C4/4 (995 slices) is below the masked-mirror threshold: plain full blocks
        # mesh rows of 65 / 67 nodes hold one or two whole 32-node slices each (C5 at full size: 84% of the
        # slices); with aligned slots the slices across the row ends are uniform too
        assert counts[("0", "2", "1")][1] * 5 > counts[base][0], counts
        assert counts[("1", "2", "1")][3] * 2 > counts[base][0], counts
        assert counts[("1", "2", "1")][1] > counts[("0", "2", "1")][1], counts
        assert counts[("1", "1", "1")][2] == 0 and (cfg != "C5" or counts[("1", "2", "1")][2] > 0), counts
    for v in variants[1:]:
        np.testing.assert_array_equal(out[base], out[v])
    ref = A.to_scipy() @ x.cpu().numpy()
    assert np.linalg.norm(out[base] - ref) <= 1e-13 * np.linalg.norm(ref)
    # the smoother passes ([K | B1] rows with the lambda split) through a whole sweep and a V-cycle
    skw = dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.6), corrector=("mcilu0", 1, 1.0))
    x0 = np.random.default_rng(0).standard_normal(op.total_rows)
    sw = {}
    for v in variants:
        monkeypatch.setenv("CAMG_SELL_ALIGN", v[0])
        monkeypatch.setenv("CAMG_SELL_USLICE", v[1])
        monkeypatch.setenv("CAMG_SELL_WITEMS", v[2])
        H = setup(saddle_operator(g), fine_level_meta(g), HierarchyConfig(max_levels=3, max_coarse_size=50),
                  block_cfg(skw))
        sw[v] = (H.levels[0].smoother.sweep_merged(x0, g.rhs).cpu().numpy(), np.asarray(H.apply(g.rhs)))
    for v in variants[1:]:
        np.testing.assert_array_equal(sw[base][0], sw[v][0])
        np.testing.assert_array_equal(sw[base][1], sw[v][1])


@pytest.mark.parametrize("cfg,scale,sweeps,cluster", [("C5", 10, 1, "1"), ("C5", 10, 1, "0"), ("C4", 8, 2, "1"),
                                                     ("C2", 4, 1, "1")])
def test_mcilu0_corrector_vs_oracle_emulation(cfg, scale, sweeps, cluster, monkeypatch):
    """GPU multicolour ILU(0) corrector == reference ILU(0) on the
    colour-permuted S~ (oracle emulation): sweep within 1e-12, V-cycle within
    1e-10, GMRES its within +-1; the reference's default corrector kind.
    Small S~ run whole sweeps on one 16-CTA cluster (cluster "1"), else one
    launch per colour and direction (cluster "0", and every multi-sweep)."""
    monkeypatch.setenv("CAMG_MCGS_CLUSTER", cluster)
    skw = dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 2, 0.6),
               corrector=("mcilu0", sweeps, 1.0))
    hkw = dict(max_levels=3, max_coarse_size=50)
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    x0 = np.random.default_rng(0).standard_normal(op.total_rows)
    out = H.levels[0].smoother.sweep_merged(x0, rhs).cpu().numpy()
    u, lam = OH.levels[0].smoother.sweep(x0[:op.n_u], x0[op.n_u:], rhs[:op.n_u], rhs[op.n_u:])
    ref = np.concatenate([u, lam])
    assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    v, ref = H.apply(rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 200, 100)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    assert orep.converged and rep.converged
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)


@pytest.mark.parametrize("kind,alpha", [("uzawa", 0.7), ("braess_sarazin", 1.9), ("simple", 0.8), ("simplec", 1.0)])
def test_sweep_is_richardson_with_preconditioning_matrix(kind, alpha):
    """With exact inner solves a block-smoother step is x + M^-1 (b - A x), M
    from the defining equations (smoothers.preconditioning_matrix; reference
    tests/test_smoothers.py:201-213).  K diagonal makes the GPU's one-sweep
    undamped Jacobi predictor exact; the corrector is the dense LU."""
    from paper_1912_09056_b200.saddle import SaddleOperator
    from paper_1912_09056_b200.smoothers import BlockSmoother, error_matrix, preconditioning_matrix
    from paper_1912_09056_b200.sparse import BlockVector
    rng = np.random.default_rng(11)
    for _ in range(3):
        nu, nl = int(rng.integers(6, 31)), int(rng.integers(2, 11))
        K = np.diag(rng.uniform(1.0, 3.0, nu))
        B1 = rng.standard_normal((nu, nl))
        B2 = B1.T.copy()
        Cz = np.diag(rng.uniform(0.5, 1.5, nl))
        op = SaddleOperator(*(SparseMatrix.from_dense(m) for m in (K, B1, B2, Cz)))
        cfg = BlockSmootherConfig(kind=kind, alpha=alpha, predictor=PointSmootherConfig("jacobi", 1, 1.0),
                                  corrector=PointSmootherConfig("direct"))
        x0 = BlockVector(rng.standard_normal(nu), rng.standard_normal(nl))
        b = BlockVector(rng.standard_normal(nu), rng.standard_normal(nl))
        out = BlockSmoother(cfg, op).sweep(x0, b).merged()
        A = op.merged_dense()
        M = preconditioning_matrix(op, cfg)
        ref = x0.merged() + np.linalg.solve(M, b.merged() - A @ x0.merged())
        assert np.abs(out - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max())
        np.testing.assert_allclose(error_matrix(op, cfg), A - M, rtol=0, atol=0)


def test_uzawa_error_matrix_closed_form():
    """E = A - M for Uzawa (reference tests/test_smoothers.py:231-247)."""
    from paper_1912_09056_b200.saddle import SaddleOperator
    from paper_1912_09056_b200.smoothers import error_matrix
    rng = np.random.default_rng(13)
    nu, nl = 12, 4
    K = np.diag(rng.uniform(1.0, 3.0, nu)) + 0.1 * rng.standard_normal((nu, nu))
    B1 = rng.standard_normal((nu, nl))
    B2, Cz = B1.T.copy(), np.eye(nl)
    op = SaddleOperator(*(SparseMatrix.from_dense(m) for m in (K, B1, B2, Cz)))
    alpha = 0.7
    E = error_matrix(op, BlockSmootherConfig(kind="uzawa", alpha=alpha))
    S = Cz + B2 @ np.diag(1.0 / np.diag(K)) @ B1
    E_ref = np.block([[(1 - 1 / alpha) * K, B1], [(1 - 1 / alpha) * B2, -Cz + S / alpha]])
    assert np.abs(E - E_ref).max() <= 1e-12 * max(1.0, np.abs(E_ref).max())


def test_mcilu0_rejected_as_predictor():
    skw = dict(kind="simple", alpha=0.8, predictor=("mcilu0", 1, 1.0), corrector=("jacobi", 1, 0.8))
    g = generate(config_spec("C2", 8))
    op = saddle_operator(g)
    with pytest.raises(ConfigError):
        setup(op, fine_level_meta(g), HierarchyConfig(max_levels=2, max_coarse_size=50), block_cfg(skw))


@pytest.mark.parametrize("cfg,scale,levels", [("C5", 10, 3), ("C4", 8, 3), ("C2", 4, 3)])
def test_mcgs_corrector_vs_oracle_emulation(cfg, scale, levels):
    """GPU multicolour SGS corrector == reference SSOR on the colour-permuted
    S~ (oracle emulation), V-cycle within 1e-10, GMRES its within +-1."""
    skw = dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 2, 0.6), corrector=("mcgs", 1, 1.0))
    hkw = dict(max_levels=levels, max_coarse_size=50)
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    x0 = np.random.default_rng(0).standard_normal(op.total_rows)
    out = H.levels[0].smoother.sweep_merged(x0, rhs).cpu().numpy()
    u, lam = OH.levels[0].smoother.sweep(x0[:op.n_u], x0[op.n_u:], rhs[:op.n_u], rhs[op.n_u:])
    ref = np.concatenate([u, lam])
    assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    v, ref = H.apply(rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 200, 100)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    assert orep.converged and rep.converged
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)


@pytest.mark.parametrize("py", ["0", "1"])
@pytest.mark.parametrize("cfg,scale", [("C5", 4), ("C2", 2), ("C3", 8)])
def test_tentative_prolongator_bit_identical(cfg, scale, py, monkeypatch):
    """Host LAPACK + device CSR assembly == the reference's per-aggregate
    pivoted QR (oracle), bit for bit, for u and lambda: the native
    camg_tentative (py=0, the default) and the numpy-grouped path (py=1)."""
    monkeypatch.setenv("CAMG_TENTATIVE_PY", py)
    from paper_1912_09056_b200.aggregation import NodeGraph, aggregate_greedy, aggregate_lagrange
    from paper_1912_09056_b200.transfer import NullSpace, tentative_prolongator
    from paper_1912_09056_b200.aggregation import filtered_node_graph
    g = generate(config_spec(cfg, scale))
    oop, ometa, _ = O.system_from_generated(g)
    meta = fine_level_meta(g)
    op = saddle_operator(g)
    gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
    ip, ix = O.node_graph(oop.K, ometa.u_dof_node, ometa.num_u_nodes, ometa.node_body)
    np.testing.assert_array_equal(gr.indptr, ip)
    np.testing.assert_array_equal(gr.indices, ix)
    ag = aggregate_greedy(gr, 6)
    oag = O.greedy(ip, ix, ometa.num_u_nodes, 6)
    np.testing.assert_array_equal(ag.node_to_agg, oag.node_to_agg)
    res = tentative_prolongator(ag, meta.ns_u, dof_node=meta.u_dof_node)
    Po, nso, cao, dro = O.tentative(oag, ometa.ns_u, ometa.u_dof_node)
    P = res.P.to_scipy()
    assert same_pattern(P, Po) and np.array_equal(P.data, Po.data)
    np.testing.assert_array_equal(res.coarse_ns.vectors, nso)
    np.testing.assert_array_equal(res.coarse_dof_agg, cao)
    assert res.dropped_columns == dro
    la = aggregate_lagrange(ag, meta.mortar_block, meta.lmap)
    ola = O.lagrange(oag, ometa.mortar, ometa.slave_dofs, ometa.row_node, ometa.lm_node_of_lm_dof)
    np.testing.assert_array_equal(la.node_to_agg, ola.node_to_agg)
    rl = tentative_prolongator(la, meta.ns_lam, dof_node=meta.lam_dof_node)
    Pl, nsl, _, _ = O.tentative(ola, ometa.ns_lam, ometa.lam_dof_node)
    assert same_pattern(rl.P.to_scipy(), Pl) and np.array_equal(rl.P.to_scipy().data, Pl.data)
    np.testing.assert_array_equal(rl.coarse_ns.vectors, nsl)


def _same_space(P, Po, ns, cns):
    """P and Po span the same coarse space aggregate by aggregate (equal
    projectors P P^T) and P reproduces the fine near-kernel: P B_c = B."""
    D = (P @ P.T - Po @ Po.T).tocsr()
    scale = scipy.sparse.linalg.norm(Po @ Po.T)
    assert scipy.sparse.linalg.norm(D) <= 1e-12 * scale
    assert np.linalg.norm(P @ cns - ns) <= 1e-12 * np.linalg.norm(ns)
    G = (P.T @ P).tocsr()                      # orthonormal columns
    assert abs(G - scipy.sparse.identity(G.shape[0])).max() <= 1e-13


@pytest.mark.parametrize("cfg,scale", [("C5", 4), ("C2", 2), ("C3", 4), ("C1", 1)])
def test_device_tentative_prolongator_vs_lapack(cfg, scale, monkeypatch):
    """the per-aggregate pivoted QR on the device
    (camg_tentative_device: LAPACK's dlaqp2 + dorg2r, one warp per aggregate)
    against the reference's scipy.linalg.qr (oracle): ranks and coarse DOF
    ownership identical, the same coarse space aggregate by aggregate (equal
    projectors P P^T to 1e-12), orthonormal columns, P B_c = B.  Columns whose
    pivot order LAPACK decides by rounding (mathematically tied rotation
    modes) may come in another order, so the factors themselves are compared
    elementwise only where no pivot is tied (the block-shapes test below)."""
    import scipy.sparse.linalg  # noqa: F401
    monkeypatch.setenv("CAMG_TENTATIVE", "gpu")
    from paper_1912_09056_b200.aggregation import aggregate_greedy, aggregate_lagrange, filtered_node_graph
    from paper_1912_09056_b200.transfer import tentative_prolongator
    g = generate(config_spec(cfg, scale))
    oop, ometa, _ = O.system_from_generated(g)
    meta = fine_level_meta(g)
    op = saddle_operator(g)
    gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
    ag = aggregate_greedy(gr, 6)
    ip, ix = O.node_graph(oop.K, ometa.u_dof_node, ometa.num_u_nodes, ometa.node_body)
    oag = O.greedy(ip, ix, ometa.num_u_nodes, 6)
    launches = _native.launch_count()
    res = tentative_prolongator(ag, meta.ns_u, dof_node=meta.u_dof_node)
    assert _native.launch_count() > launches
    Po, nso, cao, dro = O.tentative(oag, ometa.ns_u, ometa.u_dof_node)
    np.testing.assert_array_equal(res.coarse_dof_agg, cao)
    assert res.dropped_columns == dro
    _same_space(res.P.to_scipy(), Po, np.asarray(ometa.ns_u), res.coarse_ns.vectors)
    la = aggregate_lagrange(ag, meta.mortar_block, meta.lmap)
    ola = O.lagrange(oag, ometa.mortar, ometa.slave_dofs, ometa.row_node, ometa.lm_node_of_lm_dof)
    rl = tentative_prolongator(la, meta.ns_lam, dof_node=meta.lam_dof_node)
    Pl, nsl, cal, _ = O.tentative(ola, ometa.ns_lam, ometa.lam_dof_node)
    np.testing.assert_array_equal(rl.coarse_dof_agg, cal)
    _same_space(rl.P.to_scipy(), Pl, np.asarray(ometa.ns_lam), rl.coarse_ns.vectors)


def test_device_tentative_prolongator_block_shapes(monkeypatch):
    """Device QR on hand-made aggregates: tall, square, wide (fewer rows than
    vectors), single-row, rank-deficient (a repeated column: one coarse DOF
    dropped) and mixed sizes in one call, against the oracle's scipy QR."""
    monkeypatch.setenv("CAMG_TENTATIVE", "gpu")
    from paper_1912_09056_b200.aggregation import Aggregation
    from paper_1912_09056_b200.transfer import NullSpace, tentative_prolongator
    rng = np.random.default_rng(3)
    k = 6
    sizes = [40, 6, 3, 1, 17, 40, 9, 100, 6, 2]
    n = sum(sizes)
    perm = rng.permutation(n)                       # DOFs of an aggregate are not contiguous
    node_to_agg = np.empty(n, dtype=np.int64)
    node_to_agg[perm] = np.repeat(np.arange(len(sizes)), sizes)
    vecs = rng.standard_normal((n, k))
    rows4 = np.flatnonzero(node_to_agg == 4)
    vecs[rows4, 5] = vecs[rows4, 2]                 # rank-deficient block (exact repeat)
    rows6 = np.flatnonzero(node_to_agg == 6)
    vecs[rows6, 1] = 0.0                            # a zero column
    roots = np.zeros(len(sizes), dtype=np.int64)
    ag = Aggregation(node_to_agg, len(sizes), roots)
    res = tentative_prolongator(ag, NullSpace(vecs, "rigid"), dofs_per_node=1)
    oag = O.Aggregates(node_to_agg, len(sizes), roots)
    Po, nso, cao, dro = O.tentative(oag, vecs, np.arange(n))
    P = res.P.to_scipy()
    assert res.dropped_columns == dro and dro >= 2 + (6 - 3) + (6 - 1) + (6 - 2)
    np.testing.assert_array_equal(res.coarse_dof_agg, cao)
    assert same_pattern(P, Po)
    assert np.max(np.abs(P.data - Po.data)) <= 1e-12
    assert np.linalg.norm(res.coarse_ns.vectors - nso) <= 1e-12 * np.linalg.norm(nso)


# ---------------------------------------------------------------------------
# edge cases (reference behaviour: krylov.py:56-61, hierarchy.py:194,
# smoothers.py:151-153, saddle.py:22-27)


def _small():
    g = generate(config_spec("C1"))
    return g, saddle_operator(g)


def test_gmres_zero_rhs_returns_zero():
    g, op = _small()
    H = setup(op, fine_level_meta(g), HierarchyConfig(max_levels=2, max_coarse_size=1),
              block_cfg(BY_NAME["c1_uzawa_jac2"][4]))
    x, rep = gmres(op.apply_merged, H.apply, np.zeros(op.total_rows), GmresConfig())
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    assert rep.residual_history == [0.0]


def test_single_level_hierarchy_is_a_direct_solve():
    """max_levels=1: the fine level is the coarsest (merged dense LU); one
    GMRES iteration, like the reference's perfect-preconditioner case."""
    g, op = _small()
    H = setup(op, fine_level_meta(g), HierarchyConfig(max_levels=1), block_cfg(BY_NAME["c1_uzawa_jac2"][4]))
    assert H.num_levels == 1
    A = op.merged().to_scipy()
    z = H.apply(g.rhs)
    assert np.linalg.norm(A @ z - g.rhs) <= 1e-9 * np.linalg.norm(g.rhs)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=10))
    assert rep.converged and rep.iterations == 1


def test_gmres_without_preconditioner_matches_oracle():
    g = generate(config_spec("C1"))
    op = saddle_operator(g)
    oop, _, rhs = O.system_from_generated(g)
    A = oop.merged()
    _, orep = O.gmres(lambda v: A @ v, lambda v: v, rhs, 1e-6, 60, 30)
    x, rep = gmres(op.apply_merged, None, g.rhs, GmresConfig(rel_tol=1e-6, max_iters=60, restart=30))
    assert abs(rep.iterations - orep.iterations) <= 1
    assert np.allclose(rep.residual_history[:10], orep.residual_history[:10], rtol=1e-6)


def test_singular_diagonal_raises():
    from paper_1912_09056_b200.errors import SingularMatrixError
    from paper_1912_09056_b200.saddle import SaddleOperator
    from paper_1912_09056_b200.smoothers import BlockSmoother
    K = scipy.sparse.csr_matrix(np.array([[2.0, 1.0, 0.0], [1.0, 0.0, 1.0], [0.0, 1.0, 2.0]]))
    B1 = scipy.sparse.csr_matrix(np.array([[1.0], [0.0], [1.0]]))
    op = SaddleOperator(*(SparseMatrix.from_scipy(m) for m in (K, B1, B1.T, scipy.sparse.csr_matrix((1, 1)))))
    with pytest.raises(SingularMatrixError):
        BlockSmoother(block_cfg(dict(kind="uzawa", alpha=1.0, predictor=("jacobi", 1, 0.8),
                                     corrector=("jacobi", 1, 0.8))), op)


def test_dimension_errors():
    from paper_1912_09056_b200.errors import DimensionError
    from paper_1912_09056_b200.saddle import SaddleOperator
    A = SparseMatrix.from_dense(np.eye(3))
    with pytest.raises(DimensionError):
        spmv(A, np.ones(4))
    with pytest.raises(DimensionError):
        sp_matmul(A, SparseMatrix.from_dense(np.ones((2, 2))))
    with pytest.raises(DimensionError):
        SaddleOperator(A, SparseMatrix.from_dense(np.ones((2, 1))), SparseMatrix.from_dense(np.ones((1, 3))),
                       SparseMatrix.from_dense(np.ones((1, 1))))


def test_public_vcycle_function_matches_native():
    """hierarchy.vcycle (Python orchestration over the device level kernels,
    arbitrary start) from zero == the native graph-captured Hierarchy.apply."""
    from paper_1912_09056_b200.hierarchy import vcycle
    from paper_1912_09056_b200.sparse import BlockVector
    g, op, H = gpu_hier("c4s_uzawa")
    b = BlockVector.from_merged(g.rhs, op.n_u)
    x = vcycle(H, 0, BlockVector.zeros(op.n_u, op.n_lam), b).merged()
    z = H.apply(g.rhs)
    assert np.linalg.norm(x - z) <= 1e-12 * np.linalg.norm(z)


def test_graph_disabled_equals_graph():
    g, op, H = gpu_hier("c5s_simple")
    z1 = H.apply(g.rhs)
    H.use_graph(False)
    z2 = H.apply(g.rhs)
    H.use_graph(True)
    np.testing.assert_array_equal(z1, z2)


@pytest.mark.parametrize("path", ["csr", "sell", "cta", "default"])
def test_mcgs_large_s_paths(path, monkeypatch):
    """Every MC-SGS execution path (one CSR launch per colour, the
    colour-ordered SELL kernel, one-CTA sweeps, the default choice incl. the
    16-CTA cluster sweeps on small levels) against the oracle emulation."""
    if path != "default":
        monkeypatch.setenv("CAMG_MCGS_CLUSTER", "0")
    if path in ("csr", "sell"):
        monkeypatch.setenv("CAMG_MCGS_CTA", "0")
        monkeypatch.setenv("CAMG_GS_SELL", "1" if path == "sell" else "0")
    skw = dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.6), corrector=("mcgs", 1, 1.0))
    hkw = dict(max_levels=3, max_coarse_size=50)
    g = generate(config_spec("C5", 10))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    v, ref = H.apply(rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("cfg,scale,kind,path", [
    ("C5", 10, "simple", "sell"), ("C5", 10, "simple", "csr"), ("C4", 8, "uzawa", "sell"),
    ("C4", 8, "uzawa", "csr"), ("C2", 4, "simple", "sell"), ("C3", 8, "uzawa", "csr")])
def test_mcgs_predictor_vs_oracle_emulation(cfg, scale, kind, path, monkeypatch):
    """GPU multicolour (node-block) SGS predictor on K == reference SSOR on
    the node-colour-permuted K (oracle emulation): one smoother sweep within
    1e-12, V-cycle within 1e-10, GMRES its within +-1; both the colour-ordered
    SELL kernel and the CSR kernel."""
    monkeypatch.setenv("CAMG_GS_SELL", "1" if path == "sell" else "0")
    if kind == "simple":
        skw = dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("mcgs", 1, 1.0), corrector=("mcgs", 1, 1.0))
    else:  # block Gauss-Seidel = Uzawa(alpha=1) with the GPU Gauss-Seidel on K
        skw = dict(kind="uzawa", alpha=1.0, outer_sweeps=1, predictor=("mcgs", 1, 1.0), corrector=("jacobi", 1, 0.8))
    hkw = dict(max_levels=3, max_coarse_size=50)
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    x0 = np.random.default_rng(1).standard_normal(op.total_rows)
    for lvl, olvl in zip(H.levels, OH.levels):
        n_u = lvl.op.n_u
        xl = x0[:lvl.op.total_rows]
        bl = rhs[:lvl.op.total_rows] if lvl is H.levels[0] else np.random.default_rng(2).standard_normal(len(xl))
        out = lvl.smoother.sweep_merged(xl, bl).cpu().numpy()
        u, lam = olvl.smoother.sweep(xl[:n_u], xl[n_u:], bl[:n_u], bl[n_u:])
        ref = np.concatenate([u, lam])
        assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    v, ref = H.apply(rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 200, 100)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    assert rep.converged == orep.converged
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)


def test_mcgs_predictor_fine_pass_and_zero_start():
    """fine_pass mode 3 (one MC-SGS predictor sweep) runs and reports bytes;
    a sweep from zero equals a sweep from an explicit zero vector."""
    skw = dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("mcgs", 1, 1.0), corrector=("mcgs", 1, 1.0))
    g = generate(config_spec("C5", 10))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(max_levels=2, max_coarse_size=50), block_cfg(skw))
    from paper_1912_09056_b200.sparse import BlockVector, to_device
    sm = H.levels[0].smoother
    rhs = g.rhs
    a = sm.apply(BlockVector.from_merged(rhs, op.n_u)).merged()
    b = sm.sweep_merged(np.zeros(op.total_rows), rhs).cpu().numpy()
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)
    x = to_device(np.random.default_rng(0).standard_normal(op.total_rows))
    csr_b, fmt_b = H.fine_pass(3, x, to_device(rhs))
    assert csr_b > 0 and fmt_b > 0


@pytest.mark.parametrize("cfg,scale,kind,degree", [("C5", 10, "simple", 2), ("C4", 8, "uzawa", 3), ("C2", 4, "simplec", 1)])
def test_chebyshev_predictor_vs_oracle(cfg, scale, kind, degree):
    """GPU Chebyshev predictor (fused into the [K | B1] pass, d_k carried
    between steps) == the oracle's Chebyshev iteration on the same bounds:
    one sweep per level within 1e-12, V-cycle within 1e-10, GMRES its +-1."""
    alpha = 0.8 if kind != "uzawa" else 0.6
    skw = dict(kind=kind, alpha=alpha, outer_sweeps=2, predictor=("gpu_chebyshev", degree, 1.0),
               corrector=("jacobi", 1, 0.8))
    hkw = dict(max_levels=3, max_coarse_size=50)
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    H = setup(op, fine_level_meta(g), HierarchyConfig(**hkw), block_cfg(skw))
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(**hkw), oracle_block_cfg(skw))
    rng = np.random.default_rng(3)
    for lvl, olvl in zip(H.levels, OH.levels):
        n_u, n = lvl.op.n_u, lvl.op.total_rows
        xl, bl = rng.standard_normal(n), rng.standard_normal(n)
        out = lvl.smoother.sweep_merged(xl, bl).cpu().numpy()
        u, lam = olvl.smoother.sweep(xl[:n_u], xl[n_u:], bl[:n_u], bl[n_u:])
        ref = np.concatenate([u, lam])
        assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    v, ref = H.apply(rhs), OH.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, OH.apply, rhs, 1e-8, 200, 100)
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    assert rep.converged == orep.converged
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)


# ---------------------------------------------------------------------------
# nested preconditioner (hierarchy.py:289-385)

from _golden import nested_cases  # noqa: E402
from cases import NESTED_BY_NAME  # noqa: E402


@pytest.mark.parametrize("name", nested_cases())
def test_nested_vs_reference_golden(name):
    """GPU NestedPreconditioner (device scalar AMG inner solve as the SIMPLE
    predictor) against the unmodified reference: scalar levels (patterns
    exact, values 1e-12), inner V-cycle and apply within 1e-10, GMRES its +-1."""
    from paper_1912_09056_b200.hierarchy import nested_preconditioner
    z = load(name)
    _, cfg, scale, ikw, skw, ipt, restart, max_iters = NESTED_BY_NAME[name]
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    NP = nested_preconditioner(op, fine_level_meta(g), block_cfg(skw), HierarchyConfig(**ikw),
                               PointSmootherConfig(*ipt))
    assert [lvl.A.num_rows for lvl in NP.inner.levels] == z["inner_rows"].tolist()
    for l, lvl in enumerate(NP.inner.levels):
        A, ref = lvl.A.to_scipy(), csr(z, f"S{l}_A")
        assert same_pattern(A, ref) and rel_fro(A, ref) <= 1e-12
    v = NP.inner.apply(z["inner_rand_in"])
    assert np.linalg.norm(v - z["inner_apply_rand"]) <= 1e-10 * np.linalg.norm(z["inner_apply_rand"])
    for key_in, key_out in (("rhs", "apply_rhs"), ("rand_in", "apply_rand")):
        v = NP.apply(z[key_in])
        assert np.linalg.norm(v - z[key_out]) <= 1e-10 * np.linalg.norm(z[key_out])
    x, rep = gmres(op.apply_merged, NP.apply, g.rhs,
                   GmresConfig(rel_tol=1e-8, max_iters=int(max_iters), restart=int(restart)))
    assert rep.converged == bool(z["gmres_converged"])
    assert abs(rep.iterations - int(z["gmres_iterations"])) <= 1


@pytest.mark.parametrize("inner", [("mcgs", 1, 0.8), ("gpu_chebyshev", 2, 1.0)])
def test_nested_gpu_inner_smoothers_vs_oracle(inner):
    """GPU-only inner smoothers of the nested preconditioner (multicolour SGS
    -- the GPU variant of the reference's default SGS -- and Chebyshev)
    against the oracle emulation."""
    from paper_1912_09056_b200.hierarchy import nested_preconditioner
    ikw = dict(max_levels=3, max_coarse_size=50)
    skw = dict(kind="simple", alpha=0.8, outer_sweeps=1, predictor=("jacobi", 1, 0.8), corrector=("mcgs", 1, 1.0))
    g = generate(config_spec("C5", 20))
    op = saddle_operator(g)
    NP = nested_preconditioner(op, fine_level_meta(g), block_cfg(skw), HierarchyConfig(**ikw),
                               PointSmootherConfig(*inner))
    oop, ometa, rhs = O.system_from_generated(g)
    ONP = O.Nested(oop, ometa, oracle_block_cfg(skw), O.HierCfg(**ikw), O.PointCfg(*inner))
    b = np.random.default_rng(5).standard_normal(op.n_u)
    v, ref = NP.inner.apply(b), ONP.inner.apply(b)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    v, ref = NP.apply(rhs), ONP.apply(rhs)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)
    A = oop.merged()
    _, orep = O.gmres(lambda t: A @ t, ONP.apply, rhs, 1e-8, 200, 100)
    x, rep = gmres(op.apply_merged, NP.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=200, restart=100))
    assert rep.converged == orep.converged
    assert abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)


def test_nested_config_errors():
    from paper_1912_09056_b200.hierarchy import nested_preconditioner
    g = generate(config_spec("C1", 1))
    op = saddle_operator(g)
    with pytest.raises(ConfigError):
        nested_preconditioner(op, fine_level_meta(g), block_cfg(dict(kind="uzawa", alpha=1.0)),
                              HierarchyConfig(max_levels=2, max_coarse_size=50))
    with pytest.raises(ConfigError):
        nested_preconditioner(op, fine_level_meta(g), block_cfg(dict(kind="simple", alpha=0.8,
                                                                     corrector=("jacobi", 1, 0.8))),
                              HierarchyConfig(max_levels=2, max_coarse_size=50), PointSmootherConfig("ilu0", 1, 1.0))


def test_apply_many_pipelined_equals_apply():
    """Hierarchy.apply_many (independent host RHS, copies overlapped with the
    V-cycles) returns exactly what one blocking apply per RHS returns."""
    import torch
    g, op, H = gpu_hier("c5s_simple")
    rng = np.random.default_rng(9)
    rs = [torch.from_numpy(rng.standard_normal(H.n)).pin_memory() for _ in range(5)]
    outs = H.apply_many(rs)
    torch.cuda.synchronize()
    for r, o in zip(rs, outs):
        ref = H.apply(r)
        assert torch.equal(o, ref)
    with pytest.raises(Exception):
        H.apply_many([torch.zeros(H.n + 1).pin_memory()])

"""Pin the oracle (oracle/camg_oracle.py) against the reference's own outputs
(tests/golden/*.npz, written by tests/golden/make_golden.py from the
unmodified reference).  CPU only."""

import numpy as np
import pytest
import scipy.sparse

import camg_oracle as O
from _golden import GOLDEN, cases, csr, has, load

from paper_1912_09056_b200.problem import config_spec, generate

import sys
sys.path.insert(0, GOLDEN)
from cases import BY_NAME  # noqa: E402


def block_cfg(skw):
    kw = dict(skw)
    for k in ("predictor", "corrector"):
        if k in kw:
            kw[k] = O.PointCfg(*kw[k])
    return O.BlockCfg(**kw)


def same_csr(A, B, rtol=0.0):
    A, B = scipy.sparse.csr_matrix(A), scipy.sparse.csr_matrix(B)
    assert A.shape == B.shape
    assert np.array_equal(A.indptr, B.indptr)
    assert np.array_equal(A.indices, B.indices)
    if rtol == 0.0:
        assert np.array_equal(A.data, B.data)
    else:
        scale = max(np.abs(B.data).max(initial=0.0), 1e-300)
        assert np.abs(A.data - B.data).max(initial=0.0) <= rtol * scale


_built = {}


def build(name):
    if name not in _built:
        _, cfg, scale, hkw, skw, restart, max_iters = BY_NAME[name]
        g = generate(config_spec(cfg, scale))
        op, meta, rhs = O.system_from_generated(g)
        H = O.setup(op, meta, O.HierCfg(**hkw), block_cfg(skw))
        _built[name] = (g, op, meta, rhs, H)
    return _built[name]


@pytest.mark.parametrize("name", cases())
def test_generator_reproduces_fixture_inputs(name):
    z = load(name)
    g, op, meta, rhs, H = build(name)
    np.testing.assert_array_equal(rhs, z["rhs"])
    for blk in ("K", "B1", "B2", "Cz"):
        same_csr(getattr(op, blk), csr(z, f"L0_{blk}"))


@pytest.mark.parametrize("name", cases())
def test_oracle_aggregation_bit_exact(name):
    z = load(name)
    g, op, meta, rhs, H = build(name)
    ip, ix = O.node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
    np.testing.assert_array_equal(ip, z["L0_graph_indptr"])
    np.testing.assert_array_equal(ix, z["L0_graph_indices"])
    ag = O.greedy(ip, ix, meta.num_u_nodes, O.HierCfg(**BY_NAME[name][3]).min_agg_size)
    np.testing.assert_array_equal(ag.node_to_agg, z["L0_u_agg"])
    la = O.lagrange(ag, meta.mortar, meta.slave_dofs, meta.row_node, meta.lm_node_of_lm_dof)
    np.testing.assert_array_equal(la.node_to_agg, z["L0_lam_agg"])


@pytest.mark.parametrize("name", cases())
def test_oracle_hierarchy_matches_reference(name):
    z = load(name)
    g, op, meta, rhs, H = build(name)
    assert len(H.levels) == int(z["num_levels"])
    assert H.complexity == pytest.approx(float(z["complexity"]), rel=1e-14)
    for l, lvl in enumerate(H.levels):
        for blk in ("K", "B1", "B2", "Cz"):
            same_csr(getattr(lvl.op, blk), csr(z, f"L{l}_{blk}"))
        same_csr(lvl.smoother.S, csr(z, f"L{l}_Stilde"))
        if lvl.P_u is not None:
            same_csr(lvl.P_u, csr(z, f"L{l}_Pu"))
            same_csr(lvl.P_lam, csr(z, f"L{l}_Plam"))
            assert lvl.info["lambda_max"] == float(z[f"L{l}_lambda_max"])
            assert lvl.info["u_aggregates"] == int(z[f"L{l}_u_aggs"])
            assert lvl.info["lam_aggregates"] == int(z[f"L{l}_lam_aggs"])
            assert lvl.info["u_singletons"] == int(z[f"L{l}_u_singletons"])
            assert lvl.info["lam_overlap_touches"] == int(z[f"L{l}_lam_overlaps"])


@pytest.mark.parametrize("name", cases())
def test_oracle_sweep_vcycle_gmres(name):
    z = load(name)
    g, op, meta, rhs, H = build(name)
    n_u = op.n_u
    x0, b0 = z["sweep_x"], z["sweep_b"]
    u, lam = H.levels[0].smoother.sweep(x0[:n_u], x0[n_u:], b0[:n_u], b0[n_u:])
    out = np.concatenate([u, lam])
    ref = z["sweep_out"]
    assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    for key_in, key_out in (("rhs", "vcycle_out"), ("vcycle_rand_in", "vcycle_rand_out")):
        v = H.apply(z[key_in])
        ref = z[key_out]
        assert np.linalg.norm(v - ref) <= 1e-12 * np.linalg.norm(ref)
    A = op.merged()
    same_csr(A, csr(z, "A"))
    x, rep = O.gmres(lambda v: A @ v, H.apply, rhs, 1e-8, int(z["gmres_max_iters"]), int(z["gmres_restart"]))
    assert rep.iterations == int(z["gmres_iterations"])
    assert rep.converged == bool(z["gmres_converged"])
    hist = np.asarray(rep.residual_history)
    ref = z["gmres_history"]
    assert hist.shape == ref.shape
    # the recurrence is chaotic once stagnating; compare the leading part
    k = min(len(ref), 20)
    assert np.allclose(hist[:k], ref[:k], rtol=1e-8)


def test_oracle_sparse_kernels():
    z = np.load(GOLDEN + "/kernels.npz")
    for t in range(4):
        A, Asq, B = csr(z, f"t{t}_A"), csr(z, f"t{t}_Asq"), csr(z, f"t{t}_B")
        np.testing.assert_array_equal(O.spmv(A, z[f"t{t}_x"]), z[f"t{t}_spmv"])
        same_csr(O.transpose(A), csr(z, f"t{t}_AT"))
        same_csr(O.matmul(Asq, B), csr(z, f"t{t}_AB"))
        same_csr(O.rap(O.transpose(B), Asq, B), csr(z, f"t{t}_RAP"))
        np.testing.assert_array_equal(O.diagonal(Asq), z[f"t{t}_diag"])
        np.testing.assert_array_equal(O.diagonal(Asq, "abs_rowsum"), z[f"t{t}_absrow"])


# ---------------------------------------------------------------------------
# nested preconditioner (hierarchy.py:289-385)

from _golden import nested_cases  # noqa: E402
from cases import NESTED_BY_NAME  # noqa: E402


@pytest.mark.parametrize("name", nested_cases())
def test_oracle_nested_matches_reference(name):
    """Scalar AMG levels exactly, inner V-cycle and NestedPreconditioner.apply
    to rounding, GMRES iteration count equal."""
    z = load(name)
    _, cfg, scale, ikw, skw, ipt, restart, max_iters = NESTED_BY_NAME[name]
    g = generate(config_spec(cfg, scale))
    op, meta, rhs = O.system_from_generated(g)
    NP = O.Nested(op, meta, block_cfg(skw), O.HierCfg(**ikw), O.PointCfg(*ipt))
    assert [l[0].shape[0] for l in NP.inner.levels] == z["inner_rows"].tolist()
    for l, (A, P, _, _) in enumerate(NP.inner.levels):
        same_csr(A, csr(z, f"S{l}_A"))
        if P is not None:
            same_csr(P, csr(z, f"S{l}_P"))
    v = NP.inner.apply(z["inner_rand_in"])
    assert np.linalg.norm(v - z["inner_apply_rand"]) <= 1e-12 * np.linalg.norm(z["inner_apply_rand"])
    for key_in, key_out in (("rhs", "apply_rhs"), ("rand_in", "apply_rand")):
        v = NP.apply(z[key_in])
        assert np.linalg.norm(v - z[key_out]) <= 1e-12 * np.linalg.norm(z[key_out])
    A = op.merged()
    _, rep = O.gmres(lambda t: A @ t, NP.apply, rhs, 1e-8, int(max_iters), int(restart))
    assert rep.iterations == int(z["gmres_iterations"]) and rep.converged == bool(z["gmres_converged"])

"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the reference tree exists only here):

    python tests/golden/make_golden.py

It imports `contactamg` from /root/reference/pkg/src (read-only), feeds it
systems from `paper_1912_09056_b200.problem` (the reference generator cannot
produce non-matching / 3-D / tying systems) together with
a hand-built `LevelMeta`, and stores per-level
operators, aggregates, transfers, lambda_max, smoother sweeps, V-cycle outputs
and GMRES iteration counts / residual histories as compressed .npz files next
to this script.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from contactamg import hierarchy as R_h  # noqa: E402
from contactamg import krylov as R_k  # noqa: E402
from contactamg import smoothers as R_s  # noqa: E402
from contactamg import sparse as R_sp  # noqa: E402
from contactamg import transfer as R_t  # noqa: E402
from contactamg.aggregation import LagrangeMap  # noqa: E402
from contactamg.saddle import SaddleOperator  # noqa: E402

from paper_1912_09056_b200.problem import config_spec, generate  # noqa: E402

warnings.simplefilter("ignore")


def sm(m):
    return R_sp.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(m))


def put(out, key, A):
    A = A.to_scipy() if hasattr(A, "to_scipy") else scipy.sparse.csr_matrix(A)
    out[key + "_shape"] = np.array(A.shape, dtype=np.int64)
    out[key + "_indptr"] = A.indptr.astype(np.int64)
    out[key + "_indices"] = A.indices.astype(np.int64)
    out[key + "_data"] = A.data.astype(np.float64)


def ref_system(g):
    op = SaddleOperator(sm(g.K), sm(g.B1), sm(g.B2), sm(g.Cz))
    d = g.dim
    n_s = len(g.slave_nodes)
    meta = R_h.LevelMeta(
        u_dof_node=np.arange(g.n_u, dtype=np.int64) // d,
        num_u_nodes=g.n_u // d,
        node_body=g.node_body.astype(np.int8),
        lam_dof_node=np.arange(g.n_lam, dtype=np.int64) // d,
        num_lam_nodes=n_s,
        ns_u=R_t.NullSpace(g.rigid_body_modes(), "rigid-body"),
        ns_lam=R_t.build_nullspace(n_s, R_t.NULLSPACE_CONSTANT_PER_COMPONENT, dofs_per_node=d),
        mortar_block=sm(g.mortar_block),
        lmap=LagrangeMap(
            slave_dofs=g.slave_dofs.astype(np.int64),
            row_node=np.repeat(g.slave_nodes, d).astype(np.int64),
            lm_node_of_lm_dof=np.arange(g.n_lam, dtype=np.int64) // d,
        ),
    )
    return op, meta


from cases import CASES, NESTED  # noqa: E402


def _point(t):
    return R_s.PointSmootherConfig(kind=t[0], sweeps=t[1], damping=t[2])


def _block(kw):
    kw = dict(kw)
    for k in ("predictor", "corrector"):
        if k in kw:
            kw[k] = _point(kw[k])
    return R_s.BlockSmootherConfig(**kw)


def run_case(name, cfg_name, scale, hkw, skw, restart, max_iters):
    g = generate(config_spec(cfg_name, scale))
    op, meta = ref_system(g)
    hcfg = R_h.HierarchyConfig(**hkw)
    scfg = _block(skw)
    H = R_h.setup(op, meta, hcfg, scfg)
    out = {}
    out["rhs"] = g.rhs
    out["n_u"] = np.int64(g.n_u)
    out["n_lam"] = np.int64(g.n_lam)
    out["num_levels"] = np.int64(H.num_levels)
    out["complexity"] = np.float64(H.complexity)
    out["report"] = np.array(H.report)
    for l, lvl in enumerate(H.levels):
        for blk in ("K", "B1", "B2", "Cz"):
            put(out, f"L{l}_{blk}", getattr(lvl.op, blk))
        if lvl.transfer is not None:
            put(out, f"L{l}_Pu", lvl.transfer.P_u)
            put(out, f"L{l}_Plam", lvl.transfer.P_lam)
            out[f"L{l}_lambda_max"] = np.float64(lvl.info["lambda_max"] or 0.0)
            out[f"L{l}_u_aggs"] = np.int64(lvl.info["u_aggregates"])
            out[f"L{l}_lam_aggs"] = np.int64(lvl.info["lam_aggregates"])
            out[f"L{l}_u_singletons"] = np.int64(lvl.info["u_singletons"])
            out[f"L{l}_lam_overlaps"] = np.int64(lvl.info["lam_overlap_touches"])
        put(out, f"L{l}_Stilde", lvl.smoother.schur.S_tilde)
    # level-0 aggregates (node -> aggregate) recomputed through the reference
    from contactamg.aggregation import aggregate_greedy, aggregate_lagrange, filtered_node_graph
    gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
    ag = aggregate_greedy(gr, hcfg.min_agg_size)
    out["L0_u_agg"] = ag.node_to_agg
    out["L0_graph_indptr"] = gr.indptr
    out["L0_graph_indices"] = gr.indices
    la = aggregate_lagrange(ag, meta.mortar_block, meta.lmap)
    out["L0_lam_agg"] = la.node_to_agg

    rng = np.random.default_rng(123)
    n = g.n_u + g.n_lam
    x0 = rng.standard_normal(n)
    b0 = rng.standard_normal(n)
    sw = H.levels[0].smoother.sweep(R_sp.BlockVector.from_merged(x0, g.n_u), R_sp.BlockVector.from_merged(b0, g.n_u))
    out["sweep_x"] = x0
    out["sweep_b"] = b0
    out["sweep_out"] = sw.merged()
    out["vcycle_out"] = H.apply(g.rhs)
    out["vcycle_rand_in"] = b0
    out["vcycle_rand_out"] = H.apply(b0)
    A = op.merged()
    put(out, "A", A)
    Asp = A.to_scipy()
    x, rep = R_k.gmres(lambda v: Asp @ v, H.apply, g.rhs,
                       R_k.GmresConfig(rel_tol=1e-8, max_iters=max_iters, restart=restart))
    out["gmres_restart"] = np.int64(restart)
    out["gmres_max_iters"] = np.int64(max_iters)
    out["gmres_iterations"] = np.int64(rep.iterations)
    out["gmres_converged"] = np.bool_(rep.converged)
    out["gmres_history"] = np.asarray(rep.residual_history)
    out["gmres_true_relres"] = np.float64(np.linalg.norm(g.rhs - Asp @ x) / np.linalg.norm(g.rhs))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: levels={H.num_levels} its={rep.iterations} conv={rep.converged} "
          f"relres={out['gmres_true_relres']:.3e}\n{H.report}")


def run_nested(name, cfg_name, scale, ikw, skw, ipt, restart, max_iters):
    """Reference NestedPreconditioner (hierarchy.py:366-385) outputs."""
    g = generate(config_spec(cfg_name, scale))
    op, meta = ref_system(g)
    NP = R_h.nested_preconditioner(op, meta, _block(skw), R_h.HierarchyConfig(**ikw), _point(ipt))
    out = {"rhs": g.rhs, "n_u": np.int64(g.n_u), "n_lam": np.int64(g.n_lam)}
    out["inner_rows"] = np.array([lvl.A.num_rows for lvl in NP.inner.levels], dtype=np.int64)
    out["inner_nnz"] = np.array([lvl.A.nnz for lvl in NP.inner.levels], dtype=np.int64)
    for l, lvl in enumerate(NP.inner.levels):
        put(out, f"S{l}_A", lvl.A)
        if lvl.P is not None:
            put(out, f"S{l}_P", lvl.P)
    rng = np.random.default_rng(321)
    b0 = rng.standard_normal(g.n_u + g.n_lam)
    out["apply_rhs"] = NP.apply(g.rhs)
    out["rand_in"] = b0
    out["apply_rand"] = NP.apply(b0)
    out["inner_rand_in"] = b0[:g.n_u]
    out["inner_apply_rand"] = NP.inner.apply(b0[:g.n_u])
    Asp = op.merged().to_scipy()
    x, rep = R_k.gmres(lambda v: Asp @ v, NP.apply, g.rhs,
                       R_k.GmresConfig(rel_tol=1e-8, max_iters=max_iters, restart=restart))
    out["gmres_restart"] = np.int64(restart)
    out["gmres_max_iters"] = np.int64(max_iters)
    out["gmres_iterations"] = np.int64(rep.iterations)
    out["gmres_converged"] = np.bool_(rep.converged)
    out["gmres_history"] = np.asarray(rep.residual_history)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: inner levels={len(NP.inner.levels)} rows={out['inner_rows'].tolist()} "
          f"its={rep.iterations} conv={rep.converged}")


def kernels():
    """Small-matrix cases pinning the sparse core (spmv, transpose, SpGEMM,
    Galerkin, diagonals, smoother sweeps on random saddle systems)."""
    rng = np.random.default_rng(7)
    out = {}
    for t in range(4):
        m, k, n = rng.integers(5, 40, size=3)
        A = scipy.sparse.random(m, k, density=0.2, random_state=rng.integers(1 << 30), format="csr")
        B = scipy.sparse.random(k, n, density=0.2, random_state=rng.integers(1 << 30), format="csr")
        Asq = scipy.sparse.random(k, k, density=0.3, random_state=rng.integers(1 << 30), format="csr") + scipy.sparse.identity(k)
        x = rng.standard_normal(k)
        RA, AA, PA = sm(A), sm(Asq), sm(B)
        put(out, f"t{t}_A", RA)
        put(out, f"t{t}_Asq", AA)
        put(out, f"t{t}_B", PA)
        out[f"t{t}_x"] = x
        out[f"t{t}_spmv"] = R_sp.spmv(RA, x)
        put(out, f"t{t}_AT", R_sp.sp_transpose(RA))
        put(out, f"t{t}_AB", R_sp.sp_matmul(AA, PA))
        put(out, f"t{t}_RAP", R_sp.galerkin_triple(R_sp.sp_transpose(PA), AA, PA))
        out[f"t{t}_diag"] = R_sp.extract_diagonal(AA, "plain")
        out[f"t{t}_absrow"] = R_sp.extract_diagonal(AA, "abs_rowsum")
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels: ok")


if __name__ == "__main__":
    kernels()
    only = sys.argv[1:]
    for case in CASES:
        if only and case[0] not in only:
            continue
        run_case(*case)
    for case in NESTED:
        if only and case[0] not in only:
            continue
        run_nested(*case)

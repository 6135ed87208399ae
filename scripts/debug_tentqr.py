"""Diagnose device-QR vs scipy differences per aggregate: python scripts/debug_tentqr.py C5 4"""
import os, sys
import numpy as np, scipy.linalg
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
os.environ["CAMG_TENTATIVE"] = "gpu"
import camg_oracle as O
from paper_1912_09056_b200.aggregation import aggregate_greedy, filtered_node_graph
from paper_1912_09056_b200.hierarchy import fine_level_meta
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.transfer import tentative_prolongator
g = generate(config_spec(sys.argv[1], int(sys.argv[2])))
meta = fine_level_meta(g); op = saddle_operator(g)
gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
ag = aggregate_greedy(gr, 6)
res = tentative_prolongator(ag, meta.ns_u, dof_node=meta.u_dof_node)
P = res.P.to_scipy().tocsc()
ns = np.asarray(meta.ns_u.vectors); dn = np.asarray(meta.u_dof_node)
agg_of = ag.node_to_agg[dn]
order = np.argsort(agg_of, kind="stable"); cnt = np.bincount(agg_of, minlength=ag.num_aggs)
st = np.concatenate([[0], np.cumsum(cnt)])
col = 0; shown = 0; nbad = 0; kinds = {}
for a in range(ag.num_aggs):
    dofs = order[st[a]:st[a+1]]
    Q, R, piv = scipy.linalg.qr(ns[dofs], mode="economic", pivoting=True)
    dg = np.abs(np.diag(R)); r = int(np.sum(dg > 1e-10 * dg[0])) if hasattr(O, "RANK_TOL") is False else int(np.sum(dg > O.RANK_TOL * dg[0]))
    Qg = P[:, col:col + r].toarray()[dofs]
    Qs = Q[:, :r]
    zs, zg = (Qs == 0), (Qg == 0)
    if not np.array_equal(zs, zg) or np.max(np.abs(Qs - Qg)) > 1e-12:
        nbad += 1
        kind = "zeros" if np.max(np.abs(Qs - Qg)) <= 1e-12 else "values"
        kinds[kind] = kinds.get(kind, 0) + 1
        if shown < 3 and (kind == 'zeros' or os.environ.get('SHOW_VALUES')):
            shown += 1
            print("aggregate", a, "rows", len(dofs), "rank", r, "piv", piv, kind)
            np.set_printoptions(linewidth=200, precision=3)
            ii = np.unique(np.argwhere(zs != zg)[:, 0])[:6] if np.any(zs != zg) else np.arange(12)
            print("block\n", ns[dofs][ii]); print("scipy Q\n", Qs[ii]); print("gpu Q\n", Qg[ii])
            print("max diff", np.max(np.abs(Qs - Qg)), "zero-pattern diffs", int(np.sum(zs != zg)))
            i, j = np.argwhere(zs != zg)[0] if np.any(zs != zg) else (0, 0)
            print("first zero diff at", i, j, "scipy", Qs[i, j], "gpu", Qg[i, j])
    col += r
print("aggregates", ag.num_aggs, "differing", nbad, kinds)

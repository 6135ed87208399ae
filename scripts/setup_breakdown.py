"""Time the setup phases of one level on the GPU (C5 by default):
graph, aggregation, tentative QR, lambda_max, smoothing SpGEMM, transposes,
the four Galerkin products."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.hierarchy import fine_level_meta
from paper_1912_09056_b200.aggregation import filtered_node_graph, aggregate_greedy, aggregate_lagrange
from paper_1912_09056_b200.transfer import (tentative_prolongator, smooth_prolongator, build_block_transfer,
                                             estimate_lambda_max)
from paper_1912_09056_b200.sparse import galerkin_triple, sp_transpose, diagonal_device

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T = {}
def tic(): torch.cuda.synchronize(); return time.perf_counter()
def toc(k, t0): torch.cuda.synchronize(); T[k] = time.perf_counter() - t0; return time.perf_counter()
t = tic()
g = generate(config_spec("C5", scale), assemble_K=False); t = toc("generate_host", t)
op = saddle_operator(g, device_K=True); t = toc("assemble_device", t)
meta = fine_level_meta(g); t = toc("meta", t)
gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body); t = toc("graph", t)
ag = aggregate_greedy(gr, 6); t = toc("greedy", t)
la = aggregate_lagrange(ag, meta.mortar_block, meta.lmap); t = toc("lagrange", t)
ru = tentative_prolongator(ag, meta.ns_u, dof_node=meta.u_dof_node); t = toc("tentative_u", t)
rl = tentative_prolongator(la, meta.ns_lam, dof_node=meta.lam_dof_node); t = toc("tentative_lam", t)
_ = ru.P.device; t = toc("upload_Ptent", t)
d = diagonal_device(op.K); lm = estimate_lambda_max(op.K, d); t = toc("lambda_max", t)
Pu, _ = smooth_prolongator(ru.P, op.K, 4.0 / 3.0); t = toc("smooth_total(incl lambda)", t)
T_ = build_block_transfer(Pu, rl.P); t = toc("transposes", t)
Kc = galerkin_triple(T_.R_u, op.K, T_.P_u); t = toc("rap_K", t)
B1c = galerkin_triple(T_.R_u, op.B1, T_.P_lam); t = toc("rap_B1", t)
B2c = galerkin_triple(T_.R_lam, op.B2, T_.P_u); t = toc("rap_B2", t)
Czc = galerkin_triple(T_.R_lam, op.Cz, T_.P_lam); t = toc("rap_Cz", t)
print({k: round(v, 3) for k, v in T.items()})
print("aggs", ag.num_aggs, "P_u nnz", Pu.nnz, "R_u nnz", T_.R_u.nnz, "Kc", Kc.num_rows, Kc.nnz,
      "avg Kc row", Kc.nnz / Kc.num_rows)

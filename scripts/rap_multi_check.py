"""C5 level-0 K-block Galerkin product: time and a digest of the result
(compare digests across builds; the multi-row variant this was written for,
CAMG_RAP_MULTI, measured slower and was removed -- DESIGN.md §5)."""
import hashlib, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.hierarchy import fine_level_meta
from paper_1912_09056_b200.aggregation import filtered_node_graph, aggregate_greedy
from paper_1912_09056_b200.transfer import tentative_prolongator, smooth_prolongator
from paper_1912_09056_b200.sparse import galerkin_triple, sp_transpose

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = generate(config_spec("C5", scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
meta = fine_level_meta(g)
gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
ag = aggregate_greedy(gr, 6)
ru = tentative_prolongator(ag, meta.ns_u, dof_node=meta.u_dof_node)
Pu, _ = smooth_prolongator(ru.P, op.K, 4.0 / 3.0)
Ru = sp_transpose(Pu)
torch.cuda.synchronize()
t = time.perf_counter()
Kc = galerkin_triple(Ru, op.K, Pu)
torch.cuda.synchronize()
dt = time.perf_counter() - t
h = hashlib.sha256()
sc = Kc.to_scipy()
for a in (sc.indptr, sc.indices, sc.data):
    h.update(np.ascontiguousarray(a).tobytes())
print(f"multi={os.environ.get('CAMG_RAP_MULTI', '1')} rap_K {dt:.3f} s nnz {sc.nnz} digest {h.hexdigest()[:16]}", flush=True)

import os, sys, time
sys.path.insert(0, "/root/repo") if os.path.isdir("/root/repo") else None
import numpy as np, torch
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.hierarchy import fine_level_meta
from paper_1912_09056_b200.aggregation import filtered_node_graph, aggregate_greedy
from paper_1912_09056_b200.transfer import tentative_prolongator
g = generate(config_spec("C5", 1), assemble_K=False)
op = saddle_operator(g, device_K=True)
meta = fine_level_meta(g)
gr = filtered_node_graph(op.K, meta.u_dof_node, meta.num_u_nodes, meta.node_body)
ag = aggregate_greedy(gr, 6)
for py in ("0", "1", "0", "1"):
    os.environ["CAMG_TENTATIVE_PY"] = py
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = tentative_prolongator(ag, meta.ns_u, dof_node=meta.u_dof_node)
    torch.cuda.synchronize(); print("py", py, round(time.perf_counter() - t0, 3), flush=True)
    del r
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))

"""Time one fine-level multicolour SGS predictor sweep (fine_pass mode 3) on C5
and the Jacobi predictor pass (mode 1) for comparison."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_09056_b200.hierarchy import HierarchyConfig, fine_level_meta, setup
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig as P
from paper_1912_09056_b200.sparse import to_device

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = generate(config_spec("C5", scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
sc = BlockSmootherConfig(kind="simple", alpha=0.8, outer_sweeps=1, predictor=P("mcgs", 1, 1.0), corrector=P("mcgs", 1, 1.0))
H = setup(op, fine_level_meta(g), HierarchyConfig(max_levels=6, max_coarse_size=500), sc)
x = to_device(np.random.default_rng(0).standard_normal(op.total_rows))
b = to_device(g.rhs)
for mode in (3, 1):
    for _ in range(3):
        H.fine_pass(mode, x, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        bc, bf = H.fine_pass(mode, x, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"mode {mode}: {ms:.3f} ms  csr-model {bc/ms/1e6:.0f} GB/s  format {bf/ms/1e6:.0f} GB/s  ({bf/1e9:.2f} GB)", flush=True)
if len(sys.argv) > 2:
    torch.cuda.cudart().cudaProfilerStart()
    H.fine_pass(3, x, b)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()

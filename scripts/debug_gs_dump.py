import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_09056_b200.hierarchy import HierarchyConfig, fine_level_meta, setup
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig as P
os.environ["CAMG_GS_SELL"] = sys.argv[3]
g = generate(config_spec(sys.argv[1], int(sys.argv[2])))
op = saddle_operator(g)
sc = BlockSmootherConfig(kind="uzawa", alpha=1.0, predictor=P("mcgs", 1, 1.0), corrector=P("jacobi", 1, 0.8))
H = setup(op, fine_level_meta(g), HierarchyConfig(max_levels=2, max_coarse_size=50), sc)
rng = np.random.default_rng(0)
n = op.total_rows
x = rng.standard_normal(n); b = rng.standard_normal(n)
out = H.levels[0].smoother.sweep_merged(x, b).cpu().numpy()
out0 = H.levels[0].smoother.sweep_merged(np.zeros(n), b).cpu().numpy()
np.savez("gpurun_out/gs_dump.npz", x=x, b=b, out=out, out0=out0)

"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): the
graph-replayed V-cycle and native GMRES on a small config with the bench's
exact mapping, with every size-gated path forced on (block SELL + overlapped
lambda-side stream + PDL, one-cluster MC-ILU(0) and MC-SGS with DSMEM writes).

    python scripts/sanitize_run.py C1 1 [mcgs]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1912_09056_b200 import hierarchy as Hmod  # noqa: E402
from paper_1912_09056_b200.hierarchy import fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.krylov import GmresConfig, gmres  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig as P  # noqa: E402

cfg, scale = sys.argv[1], int(sys.argv[2])
variant = sys.argv[3] if len(sys.argv) > 3 else "bench"
Hmod.SELL_MIN_ROWS = 0                # block SELL, the overlap split and block transfers at any size
hcfg, scfg, restart = bench.solver_for(cfg)
if variant == "mcgs":                 # MC-SGS predictor (colour-ordered SELL) and corrector (cluster)
    scfg = BlockSmootherConfig(kind="simple", alpha=0.8, outer_sweeps=2, predictor=P("mcgs", 1, 1.0),
                               corrector=P("mcgs", 1, 1.0))
g = generate(config_spec(cfg, scale))
op = saddle_operator(g, device_K=True)
H = setup(op, fine_level_meta(g), hcfg, scfg)
for i, lv in enumerate(H.levels[:-1]):
    print("level", i, lv.op.n_u, lv.op.n_lam, H.level_info(i))
z = None
for _ in range(3):
    z = H.apply(g.rhs)
x, rep = gmres(op.apply_merged, H.apply, g.rhs, GmresConfig(rel_tol=1e-8, max_iters=100, restart=restart))
print(f"{cfg}/{scale} {variant}: |z| {np.linalg.norm(z):.6e}, gmres its {rep.iterations} conv {rep.converged}")

"""Debug: MC-SGS predictor u-part vs oracle per level (Uzawa alpha=1 => u_new = GS result)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import camg_oracle as O
from paper_1912_09056_b200.hierarchy import HierarchyConfig, fine_level_meta, setup
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig as P

cfg, scale = sys.argv[1], int(sys.argv[2])
for path in ("1", "0"):
    os.environ["CAMG_GS_SELL"] = path
    g = generate(config_spec(cfg, scale))
    op = saddle_operator(g)
    sc = BlockSmootherConfig(kind="uzawa", alpha=1.0, predictor=P("mcgs", 1, 1.0), corrector=P("jacobi", 1, 0.8))
    H = setup(op, fine_level_meta(g), HierarchyConfig(max_levels=3, max_coarse_size=50), sc)
    oop, ometa, rhs = O.system_from_generated(g)
    OH = O.setup(oop, ometa, O.HierCfg(max_levels=3, max_coarse_size=50),
                 O.BlockCfg(kind="uzawa", alpha=1.0, predictor=O.PointCfg("mcgs", 1, 1.0), corrector=O.PointCfg("jacobi", 1, 0.8)))
    rng = np.random.default_rng(0)
    for l, (lvl, olvl) in enumerate(zip(H.levels, OH.levels)):
        n, nu = lvl.op.total_rows, lvl.op.n_u
        for xz in (True, False):
            x = np.zeros(n) if xz else rng.standard_normal(n)
            b = rng.standard_normal(n)
            out = lvl.smoother.sweep_merged(x, b).cpu().numpy()
            u, lam = olvl.smoother.sweep(x[:nu], x[nu:], b[:nu], b[nu:])
            eu = np.linalg.norm(out[:nu] - u) / np.linalg.norm(u)
            el = np.linalg.norm(out[nu:] - lam) / max(np.linalg.norm(lam), 1e-300)
            # plain Jacobi-free reference: one GS sweep natural order on K (no perm) for scale
            print(f"path={path} level={l} nu={nu} zero={xz} err_u={eu:.3e} err_lam={el:.3e}", flush=True)

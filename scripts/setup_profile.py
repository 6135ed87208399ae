"""cProfile of the bench setup (host hot spots of the level loop).
    python scripts/setup_profile.py C5 1"""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1912_09056_b200.hierarchy import fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402

cfg, scale = sys.argv[1], int(sys.argv[2])
g = generate(config_spec(cfg, scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
hcfg, scfg, _ = bench.solver_for(cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
meta = fine_level_meta(g)
H = setup(op, meta, hcfg, scfg)
torch.cuda.synchronize()
pr.disable()
print({k: round(v, 3) for k, v in H.timings.items()})
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)

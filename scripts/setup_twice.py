"""Bench setup of a config twice in one process (the second run is warm:
kernel modules loaded, allocator pools grown): phase timings of both.
    python scripts/setup_twice.py C5 1"""
import gc
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1912_09056_b200.hierarchy import fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402

cfg, scale = sys.argv[1], int(sys.argv[2])
g = generate(config_spec(cfg, scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
meta = fine_level_meta(g)
hcfg, scfg, _ = bench.solver_for(cfg)
for run in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = setup(op, meta, hcfg, scfg)
    torch.cuda.synchronize()
    print(f"run {run}: setup {time.perf_counter() - t0:.3f} s", {k: round(v, 3) for k, v in H.timings.items()},
          flush=True)
    del H
    gc.collect()
    torch.cuda.synchronize()

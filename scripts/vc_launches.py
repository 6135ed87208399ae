"""Set up a config's hierarchy exactly as bench.py does, then run ONE V-cycle
inside a cudaProfilerStart/Stop range (for `ncu --profile-from-start off`,
launch list of one cycle).  Usage: python scripts/vc_launches.py C3 [scale]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1912_09056_b200.hierarchy import fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402
from paper_1912_09056_b200.sparse import empty  # noqa: E402

cfg = sys.argv[1]
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = generate(config_spec(cfg, scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
hcfg, scfg, _ = bench.solver_for(cfg)
H = setup(op, fine_level_meta(g), hcfg, scfg)
rhs = torch.from_numpy(g.rhs).cuda()
z = empty(H.n)
for _ in range(5):
    H.apply_device(rhs, z)
torch.cuda.synchronize()
torch.cuda.profiler.start()
H.apply_device(rhs, z)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    H.apply_device(rhs, z)
e1.record()
torch.cuda.synchronize()
print(f"{cfg}/{scale}: V-cycle {e0.elapsed_time(e1) / 20:.4f} ms, levels "
      f"{[(l.op.n_u, l.op.n_lam, l.op.nnz) for l in H.levels]}")

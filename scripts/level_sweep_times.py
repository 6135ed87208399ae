"""Per-level smoother sweep time inside a CUDA graph (no profiler): for each
non-coarsest level of a config's bench hierarchy, capture 20 BlockSmoother
sweeps (camg_level_sweep) in a torch CUDA graph and time its replay, with
the lambda-side modes given (CAMG_LAM_FUSED read at capture time).
    python scripts/level_sweep_times.py C3 1 0,1,2"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1912_09056_b200 import _native as N  # noqa: E402
from paper_1912_09056_b200.hierarchy import fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402
from paper_1912_09056_b200.sparse import ptr  # noqa: E402

cfg, scale = sys.argv[1], int(sys.argv[2])
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1"]
g = generate(config_spec(cfg, scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
hcfg, scfg, _ = bench.solver_for(cfg)
H = setup(op, fine_level_meta(g), hcfg, scfg)
reps = 20
for l, lv in enumerate(H.levels[:-1]):
    n = lv.op.total_rows
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    res = []
    for m in modes:
        os.environ["CAMG_LAM_FUSED"] = m
        s = torch.cuda.Stream()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for _ in range(2):
                N.call("camg_level_sweep", lv.smoother.handle, ptr(x), ptr(b), ptr(y), s.cuda_stream)
            torch.cuda.synchronize()
            with torch.cuda.graph(gph, stream=s):
                for k in range(reps):
                    src, dst = (x, y) if k % 2 == 0 else (y, x)
                    N.call("camg_level_sweep", lv.smoother.handle, ptr(src), ptr(b), ptr(dst), s.cuda_stream)
        for _ in range(3):
            gph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            gph.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(f"mode {m}: {e0.elapsed_time(e1) / (5 * reps) * 1e3:8.1f} us/sweep")
    info = H.level_info(l)
    print(f"{cfg}/{scale} level {l} (n_u={lv.op.n_u}, n_lam={lv.op.n_lam}, corr={info['corr_path']}, "
          f"colours={info['corr_colors']}, overlap={info['overlap']}): " + " | ".join(res), flush=True)

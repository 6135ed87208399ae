"""Golden-case table shared by make_golden.py (reference side) and the tests.

Each case: (name, config, scale, HierarchyConfig kwargs, BlockSmootherConfig
kwargs with point smoothers as (kind, sweeps, damping) tuples, GMRES restart,
GMRES max_iters).
"""

CASES = [
    ("c1_bgs_jac", "C1", 1, dict(max_levels=2, max_coarse_size=1),
     dict(kind="uzawa", alpha=1.0, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8)), 30, 400),
    ("c1_uzawa_jac2", "C1", 1, dict(max_levels=2, max_coarse_size=1),
     dict(kind="uzawa", alpha=1.0, predictor=("jacobi", 2, 0.6), corrector=("jacobi", 1, 0.6)), 30, 200),
    ("c2s_simplec", "C2", 8, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8)), 50, 200),
    ("c2s_simple_sgs_ilu", "C2", 8, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=1, predictor=("sgs", 1, 1.0), corrector=("ilu0", 1, 1.0)), 50, 200),
    ("c3s_bs", "C3", 8, dict(max_levels=4, max_coarse_size=50),
     dict(kind="braess_sarazin", alpha=1.0 / 0.7, corrector=("jacobi", 1, 0.7)), 50, 200),
    ("c3s_bs_blocksmoother", "C3", 8, dict(max_levels=3, max_coarse_size=50, coarse_solver="block_smoother"),
     dict(kind="braess_sarazin", alpha=1.0 / 0.7, corrector=("jacobi", 1, 0.7)), 50, 100),
    ("c4s_uzawa", "C4", 16, dict(max_levels=3, max_coarse_size=50),
     dict(kind="uzawa", alpha=0.6, predictor=("jacobi", 2, 0.6), corrector=("jacobi", 1, 0.6)), 100, 200),
    ("c5s_simple", "C5", 25, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8)), 100, 200),
    ("c5s_simple_direct", "C5", 25, dict(max_levels=2, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=1, predictor=("jacobi", 2, 0.7), corrector=("direct", 1, 1.0)), 100, 100),
]

BY_NAME = {c[0]: c for c in CASES}

# nested preconditioner (hierarchy.py:289-385): (name, config, scale, inner
# HierarchyConfig kwargs, outer SIMPLE-type BlockSmootherConfig kwargs, inner
# point smoother (kind, sweeps, damping), GMRES restart, GMRES max_iters)
NESTED = [
    ("nested_c5s", "C5", 25, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simple", alpha=0.8, outer_sweeps=1, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8)),
     ("jacobi", 2, 0.6), 100, 200),
    ("nested_c2s", "C2", 8, dict(max_levels=3, max_coarse_size=50),
     dict(kind="simplec", alpha=0.8, outer_sweeps=2, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8)),
     ("jacobi", 1, 0.8), 50, 200),
]
NESTED_BY_NAME = {c[0]: c for c in NESTED}

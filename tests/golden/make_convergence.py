"""Convergence evidence from the UNMODIFIED reference (build container only).

    python tests/golden/make_convergence.py [table|literal|all]

(1) `table` -- for every BASELINE config mapping (bench.solver_for), GMRES
    iterations with the reference's lexicographic `sgs` / `ilu0` inner solves
    (smoothers.py:155-171, 186-199) on scaled copies of the config, next to
    the multicolour GPU variants `mcgs` / `mcilu0` on the same system.  The
    reference numbers come from the reference package itself; the multicolour
    numbers from the oracle's emulation (elementwise equal to the GPU path,
    tests/test_gpu_parity.py), and are re-measured on the GPU by
    tests/test_gpu_scale_parity.py::test_convergence_vs_reference_lexicographic.
(2) `literal` -- the smoothers BASELINE.json states literally (SIMPLEC for
    C2 / C5, Braess-Sarazin for C3, BGS for C1, Uzawa + Jacobi for C4), run
    in the reference on scaled systems, so the config mapping of DESIGN.md §6
    rests on reference-side evidence.

Writes tests/golden/convergence.json (read by the GPU test) and
profiles/r02_convergence_table.md.  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
warnings.simplefilter("ignore")

import camg_oracle as O  # noqa: E402
from contactamg import hierarchy as R_h  # noqa: E402
from contactamg import krylov as R_k  # noqa: E402
from contactamg import smoothers as R_s  # noqa: E402
from make_golden import ref_system  # noqa: E402

import bench  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate  # noqa: E402

OUT_JSON = os.path.join(HERE, "convergence.json")
OUT_MD = os.path.join(ROOT, "profiles", "r02_convergence_table.md")

# scaled systems the reference sets up in seconds to a minute
SCALES = {"C1": 1, "C2": 2, "C3": 4, "C4": 8, "C5": 10}
MAX_ITERS = 300

# (label, predictor override, corrector override); None keeps the mapping's
# own predictor.  Each row pairs a reference lexicographic kind with its
# multicolour GPU variant.
VARIANTS = [
    ("corrector ilu0 vs mcilu0", None, ("ilu0", "mcilu0")),
    ("corrector sgs vs mcgs", None, ("sgs", "mcgs")),
    ("predictor sgs vs mcgs, corrector ilu0 vs mcilu0 (reference default kinds)", ("sgs", "mcgs"),
     ("ilu0", "mcilu0")),
    ("predictor sgs vs mcgs, corrector sgs vs mcgs", ("sgs", "mcgs"), ("sgs", "mcgs")),
]


def load():
    if os.path.exists(OUT_JSON):
        with open(OUT_JSON) as fh:
            return json.load(fh)
    return {"table": [], "literal": []}


def save(d):
    with open(OUT_JSON, "w") as fh:
        json.dump(d, fh, indent=1)


def skw_of(scfg, pred=None, corr=None):
    p = pred or (scfg.predictor.kind, scfg.predictor.sweeps, scfg.predictor.damping)
    c = corr or (scfg.corrector.kind, scfg.corrector.sweeps, scfg.corrector.damping)
    return dict(kind=scfg.kind, alpha=scfg.alpha, outer_sweeps=scfg.outer_sweeps, predictor=tuple(p),
                corrector=tuple(c))


def ref_run(cfg, scale, hkw, skw, restart):
    g = generate(config_spec(cfg, scale))
    op, meta = ref_system(g)
    kw = dict(skw)
    for k in ("predictor", "corrector"):
        kw[k] = R_s.PointSmootherConfig(kind=kw[k][0], sweeps=kw[k][1], damping=kw[k][2])
    t0 = time.perf_counter()
    H = R_h.setup(op, meta, R_h.HierarchyConfig(**hkw), R_s.BlockSmootherConfig(**kw))
    ts = time.perf_counter() - t0
    A = op.merged().to_scipy()
    t0 = time.perf_counter()
    x, rep = R_k.gmres(lambda v: A @ v, H.apply, g.rhs, R_k.GmresConfig(rel_tol=1e-8, max_iters=MAX_ITERS,
                                                                          restart=restart))
    tsol = time.perf_counter() - t0
    rr = float(np.linalg.norm(g.rhs - A @ x) / np.linalg.norm(g.rhs))
    return dict(iterations=int(rep.iterations), converged=bool(rep.converged), true_relres=rr,
                levels=int(H.num_levels), n=int(A.shape[0]), setup_s=round(ts, 2), solve_s=round(tsol, 2))


def oracle_run(cfg, scale, hkw, skw, restart):
    g = generate(config_spec(cfg, scale))
    op, meta, rhs = O.system_from_generated(g)
    kw = dict(skw)
    for k in ("predictor", "corrector"):
        kw[k] = O.PointCfg(*kw[k])
    H = O.setup(op, meta, O.HierCfg(**hkw), O.BlockCfg(**kw))
    A = op.merged()
    x, rep = O.gmres(lambda t: A @ t, H.apply, rhs, 1e-8, MAX_ITERS, restart)
    rr = float(np.linalg.norm(rhs - A @ x) / np.linalg.norm(rhs))
    return dict(iterations=int(rep.iterations), converged=bool(rep.converged), true_relres=rr,
                levels=len(H.levels), n=int(A.shape[0]))


def hkw_of(hcfg):
    return dict(max_levels=hcfg.max_levels, max_coarse_size=hcfg.max_coarse_size,
                coarse_solver=hcfg.coarse_solver, min_agg_size=hcfg.min_agg_size)


def table(d):
    done = {(r["config"], r["variant"]) for r in d["table"]}
    for cfg, scale in SCALES.items():
        hcfg, scfg, restart = bench.solver_for(cfg)
        hkw = hkw_of(hcfg)
        for label, pred, corr in VARIANTS:
            if (cfg, label) in done:
                continue
            ref_skw = skw_of(scfg, None if pred is None else (pred[0], 1, 1.0),
                             (corr[0], 1, 1.0))
            gpu_skw = skw_of(scfg, None if pred is None else (pred[1], 1, 1.0),
                             (corr[1], 1, 1.0))
            r = ref_run(cfg, scale, hkw, ref_skw, restart)
            m = oracle_run(cfg, scale, hkw, gpu_skw, restart)
            row = dict(config=cfg, scale=scale, variant=label, hierarchy=hkw, restart=restart,
                       reference_smoother=ref_skw, gpu_smoother=gpu_skw, reference=r, multicolour_oracle=m)
            d["table"].append(row)
            save(d)
            print(f"{cfg}/{scale} {label}: reference {r['iterations']} ({r['converged']}) "
                  f"multicolour {m['iterations']} ({m['converged']})", flush=True)


# literal BASELINE.json smoothers (configs[i] text), reference package
LITERAL = [
    ("C1", 1, "BGS = Uzawa alpha=1, Jacobi(1, 0.8) per block",
     dict(kind="uzawa", alpha=1.0, outer_sweeps=1, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8))),
    ("C2", 2, "SIMPLEC alpha=0.8 x3, Jacobi(1,0.8) / Jacobi(1,0.8)",
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8))),
    ("C2", 2, "SIMPLEC alpha=0.8 x3, reference default inner kinds sgs / ilu0",
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("sgs", 1, 1.0), corrector=("ilu0", 1, 1.0))),
    ("C2", 1, "SIMPLEC alpha=0.8 x3, reference default inner kinds sgs / ilu0 (full C2)",
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("sgs", 1, 1.0), corrector=("ilu0", 1, 1.0))),
    ("C3", 4, "Braess-Sarazin alpha=1/0.7, Jacobi(1,0.7) Schur sweep",
     dict(kind="braess_sarazin", alpha=1.0 / 0.7, outer_sweeps=1, predictor=("jacobi", 1, 1.0),
          corrector=("jacobi", 1, 0.7))),
    ("C3", 4, "Braess-Sarazin alpha=0.7, Jacobi(1,0.7) Schur sweep",
     dict(kind="braess_sarazin", alpha=0.7, outer_sweeps=1, predictor=("jacobi", 1, 1.0),
          corrector=("jacobi", 1, 0.7))),
    ("C3", 4, "Braess-Sarazin alpha=1/0.7, reference default corrector ilu0",
     dict(kind="braess_sarazin", alpha=1.0 / 0.7, outer_sweeps=1, predictor=("jacobi", 1, 1.0),
          corrector=("ilu0", 1, 1.0))),
    ("C4", 8, "Uzawa alpha=0.6, Jacobi(2,0.6) / Jacobi(1,0.6)",
     dict(kind="uzawa", alpha=0.6, outer_sweeps=1, predictor=("jacobi", 2, 0.6), corrector=("jacobi", 1, 0.6))),
    ("C5", 10, "SIMPLEC alpha=0.8 x1, Jacobi(1,0.8) / Jacobi(1,0.8)",
     dict(kind="simplec", alpha=0.8, outer_sweeps=1, predictor=("jacobi", 1, 0.8), corrector=("jacobi", 1, 0.8))),
    ("C5", 10, "SIMPLEC alpha=0.8 x3, Jacobi(1,0.6) / Jacobi(1,0.6)",
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.6), corrector=("jacobi", 1, 0.6))),
    ("C5", 10, "SIMPLEC alpha=0.8 x3, reference default inner kinds sgs / ilu0",
     dict(kind="simplec", alpha=0.8, outer_sweeps=3, predictor=("sgs", 1, 1.0), corrector=("ilu0", 1, 1.0))),
    ("C5", 10, "mapped: SIMPLE alpha=0.8 x3, Jacobi(1,0.6) / reference ilu0 (lexicographic)",
     dict(kind="simple", alpha=0.8, outer_sweeps=3, predictor=("jacobi", 1, 0.6), corrector=("ilu0", 1, 1.0))),
]


def literal(d):
    done = {(r["config"], r["scale"], r["label"]) for r in d["literal"]}
    for cfg, scale, label, skw in LITERAL:
        if (cfg, scale, label) in done:
            continue
        hcfg, _, restart = bench.solver_for(cfg)
        r = ref_run(cfg, scale, hkw_of(hcfg), skw, restart)
        d["literal"].append(dict(config=cfg, scale=scale, label=label, smoother=skw, restart=restart,
                                 hierarchy=hkw_of(hcfg), reference=r))
        save(d)
        print(f"literal {cfg}/{scale} {label}: {r['iterations']} its conv={r['converged']} "
              f"relres={r['true_relres']:.3e}", flush=True)


def markdown(d):
    L = ["# Convergence: reference lexicographic inner solves vs multicolour GPU variants (round 2)", "",
         "Generated by `tests/golden/make_convergence.py` (reference package run unmodified in the build "
         "container; multicolour counts from the oracle emulation, which the GPU matches elementwise, and "
         "re-measured on the B200 by `tests/test_gpu_scale_parity.py`).  GMRES rtol 1e-8, x0 = 0, "
         f"max {MAX_ITERS} iterations.", "",
         "## 1. Same system, same mapping: lexicographic (reference) vs multicolour (GPU)", "",
         "| config | variant | reference its (relres) | multicolour its (relres) |", "|---|---|---|---|"]
    for r in d["table"]:
        a, b = r["reference"], r["multicolour_oracle"]
        L.append(f"| {r['config']}/{r['scale']} (n={a['n']}) | {r['variant']} | {a['iterations']}"
                 f"{'' if a['converged'] else ' (no conv)'} ({a['true_relres']:.1e}) | {b['iterations']}"
                 f"{'' if b['converged'] else ' (no conv)'} ({b['true_relres']:.1e}) |")
    L += ["", "## 2. Literal BASELINE.json smoothers in the reference", "",
          "| config | smoother | its | converged | true relres | levels |", "|---|---|---|---|---|---|"]
    for r in d["literal"]:
        a = r["reference"]
        L.append(f"| {r['config']}/{r['scale']} (n={a['n']}) | {r['label']} | {a['iterations']} | "
                 f"{a['converged']} | {a['true_relres']:.2e} | {a['levels']} |")
    with open(OUT_MD, "w") as fh:
        fh.write("\n".join(L) + "\n")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    d = load()
    if what in ("table", "all"):
        table(d)
    if what in ("literal", "all"):
        literal(d)
    markdown(d)

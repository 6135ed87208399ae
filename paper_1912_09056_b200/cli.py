"""Experiment driver (SPEC.md module `cli`; the reference
package never implemented it): `solve` and `refine-sweep` over the seeded
BASELINE configurations, CSV reports, MatrixMarket export of the system.

    python -m paper_1912_09056_b200.cli solve --config run.cfg --out outdir [--export-system]
    python -m paper_1912_09056_b200.cli refine-sweep --config run.cfg --out outdir

Config: flat `key=value` text, one key per line, `#` comments, dotted nested
keys:

    config=C5            # BASELINE configuration C1..C5 (problem.py generator)
    scale=10             # element counts divided by this (1 = the full config)
    hierarchy.max_levels=4
    hierarchy.max_coarse_size=50
    hierarchy.coarse_solver=merged_lu
    smoother.kind=simple
    smoother.alpha=0.8
    smoother.outer_sweeps=3
    smoother.a_hat_mode=plain_diag
    smoother.predictor.kind=jacobi
    smoother.predictor.sweeps=1
    smoother.predictor.damping=0.6
    smoother.corrector.kind=mcilu0
    gmres.rel_tol=1e-8
    gmres.restart=100
    gmres.max_iters=300

Keys left out take the bench mapping of the configuration (bench.solver_for)
and then the reference defaults.  Outputs: report.csv
(iteration, relative residual estimate; 17 significant digits), setup.txt
(the hierarchy's setup report and phase timings), optionally K.mtx, B1.mtx,
B2.mtx, Cz.mtx; a solve that does not converge exits with status 1 after
writing its report.  `rotation-sweep` needs the reference's rotated 2-D
two-block problem, which is outside this package: it exits
with status 2.
"""

from __future__ import annotations

import argparse
import dataclasses
import os
import sys
import time

from .errors import ConfigError

_KEYS = {
    "config": str, "scale": int,
    "hierarchy.max_levels": int, "hierarchy.max_coarse_size": int, "hierarchy.coarse_solver": str,
    "hierarchy.min_agg_size": int, "hierarchy.omega": float,
    "smoother.kind": str, "smoother.alpha": float, "smoother.outer_sweeps": int, "smoother.a_hat_mode": str,
    "smoother.predictor.kind": str, "smoother.predictor.sweeps": int, "smoother.predictor.damping": float,
    "smoother.corrector.kind": str, "smoother.corrector.sweeps": int, "smoother.corrector.damping": float,
    "gmres.rel_tol": float, "gmres.restart": int, "gmres.max_iters": int,
    "pre_sweeps": int, "post_sweeps": int,
}


def parse_config(text: str, source: str = "<config>") -> dict:
    """key=value lines -> {key: typed value}; errors name the line."""
    out = {}
    for no, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{source}:{no}: expected key=value, got {raw.strip()!r}")
        key, val = (t.strip() for t in line.split("=", 1))
        if key not in _KEYS:
            raise ConfigError(f"{source}:{no}: unknown key {key!r}")
        if key in out:
            raise ConfigError(f"{source}:{no}: duplicate key {key!r}")
        try:
            out[key] = _KEYS[key](val)
        except ValueError:
            raise ConfigError(f"{source}:{no}: {key} needs a {_KEYS[key].__name__}, got {val!r}") from None
    if "config" not in out:
        raise ConfigError(f"{source}: missing key 'config'")
    return out


def build_configs(c: dict):
    """HierarchyConfig, BlockSmootherConfig, GmresConfig from the parsed keys
    over the bench mapping of the configuration."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    from .krylov import GmresConfig
    from .smoothers import PointSmootherConfig

    try:
        hcfg, scfg, restart = bench.solver_for(c["config"])
    except KeyError:
        raise ConfigError(f"unknown configuration {c['config']!r} (C1..C5)") from None
    h = {k.split(".", 1)[1]: v for k, v in c.items() if k.startswith("hierarchy.")}
    hcfg = dataclasses.replace(hcfg, **h)
    pred, corr = scfg.predictor, scfg.corrector
    pk = {k.rsplit(".", 1)[1]: v for k, v in c.items() if k.startswith("smoother.predictor.")}
    ck = {k.rsplit(".", 1)[1]: v for k, v in c.items() if k.startswith("smoother.corrector.")}
    pred = PointSmootherConfig(**{**dataclasses.asdict(pred), **pk})
    corr = PointSmootherConfig(**{**dataclasses.asdict(corr), **ck})
    sk = {k.split(".", 1)[1]: v for k, v in c.items() if k.startswith("smoother.") and k.count(".") == 1}
    scfg = dataclasses.replace(scfg, predictor=pred, corrector=corr, **sk)
    g = GmresConfig(rel_tol=c.get("gmres.rel_tol", 1e-8), max_iters=c.get("gmres.max_iters", 300),
                    restart=c.get("gmres.restart", restart))
    return hcfg, scfg, g


def _fmt(x: float) -> str:
    return f"{x:.17g}"


def run_solve(c: dict, out: str, export: bool = False, scale=None) -> dict:
    from .hierarchy import fine_level_meta, setup
    from .krylov import gmres
    from .problem import config_spec, generate, saddle_operator
    from .sparse import write_matrix_market

    hcfg, scfg, gcfg = build_configs(c)
    sc = c.get("scale", 1) if scale is None else scale
    os.makedirs(out, exist_ok=True)
    t0 = time.perf_counter()
    g = generate(config_spec(c["config"], sc))
    op = saddle_operator(g)
    t_gen = time.perf_counter() - t0
    if export:
        for name in ("K", "B1", "B2", "Cz"):
            write_matrix_market(os.path.join(out, f"{name}.mtx"), getattr(op, name))
    t0 = time.perf_counter()
    H = setup(op, fine_level_meta(g), hcfg, scfg, c.get("pre_sweeps", 1), c.get("post_sweeps", 1))
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    x, rep = gmres(op.apply_merged, H.apply, g.rhs, gcfg)
    t_solve = time.perf_counter() - t0
    b0 = rep.residual_history[0] if rep.residual_history else 1.0
    with open(os.path.join(out, "report.csv"), "w") as fh:
        fh.write("iteration,relative_residual\n")
        for k, r in enumerate(rep.residual_history):
            fh.write(f"{k},{_fmt(r / b0 if b0 else 0.0)}\n")
    with open(os.path.join(out, "setup.txt"), "w") as fh:
        fh.write(H.report + "\n")
        fh.write(f"generate_seconds={_fmt(t_gen)}\nsetup_seconds={_fmt(t_setup)}\nsolve_seconds={_fmt(t_solve)}\n")
        for k, v in H.timings.items():
            fh.write(f"setup.{k}_seconds={_fmt(v)}\n")
    return {"iterations": rep.iterations, "converged": rep.converged, "complexity": H.complexity,
            "unknowns": int(op.total_rows), "setup_seconds": t_setup, "solve_seconds": t_solve}


def cmd_solve(args) -> int:
    c = parse_config(open(args.config).read(), args.config)
    r = run_solve(c, args.out, args.export_system)
    print(f"iterations={r['iterations']} converged={r['converged']} complexity={r['complexity']:.4f} "
          f"setup={r['setup_seconds']:.3f}s solve={r['solve_seconds']:.3f}s")
    return 0 if r["converged"] else 1


def cmd_refine_sweep(args) -> int:
    """Meshes m, 2m, 4m per block (scale s, s/2, s/4)."""
    c = parse_config(open(args.config).read(), args.config)
    s0 = c.get("scale", 1)
    scales = [s for s in (s0, s0 // 2, s0 // 4) if s >= 1]
    rows = []
    for s in dict.fromkeys(scales):
        r = run_solve(c, os.path.join(args.out, f"scale_{s}"), scale=s)
        rows.append((s, r))
        print(f"scale={s} unknowns={r['unknowns']} iterations={r['iterations']} complexity={r['complexity']:.4f}")
    with open(os.path.join(args.out, "refine.csv"), "w") as fh:
        fh.write("scale,unknowns,iterations,converged,complexity,setup_seconds,solve_seconds\n")
        for s, r in rows:
            fh.write(f"{s},{r['unknowns']},{r['iterations']},{int(r['converged'])},{_fmt(r['complexity'])},"
                     f"{_fmt(r['setup_seconds'])},{_fmt(r['solve_seconds'])}\n")
    return 0 if all(r["converged"] for _, r in rows) else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1912_09056_b200.cli")
    sub = ap.add_subparsers(dest="verb", required=True)
    for verb in ("solve", "refine-sweep", "rotation-sweep"):
        p = sub.add_parser(verb)
        p.add_argument("--config", required=True)
        p.add_argument("--out", default=".")
        if verb == "solve":
            p.add_argument("--export-system", action="store_true")
    args = ap.parse_args(argv)
    try:
        if args.verb == "solve":
            return cmd_solve(args)
        if args.verb == "refine-sweep":
            return cmd_refine_sweep(args)
        print("rotation-sweep needs the reference's rotated 2-D two-block problem, which this package does not "
              "generate (DESIGN.md §10)", file=sys.stderr)
        return 2
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())

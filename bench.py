"""Benchmark: AMG preconditioner V-cycles/s (+ SpMV GB/s, GMRES time to
solution) on BASELINE config C5 (3-D frictionless contact, ~23.8M unknowns),
one B200 per rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--scale 1]
    python bench.py --impl reference ...     # CPU reference arm (oracle port)

One step = one preconditioner application (one V-cycle from zero,
`Hierarchy.apply`) on the fine-level residual.  Multi-GPU = independent
replicas (the path does not shard in v1); value = all
ranks' V-cycles / max-over-ranks time.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import ctypes as C

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# ncu dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, per
# launch, from profiles/ (one `ncu --set full` capture; None until measured)
TRAFFIC = {
    # profiles/r02_dominant_kernel_c5.ncu-rep: k_sell_row<3,3,0,1,1,1> (masked
    # slots, 64-thread CTAs), C5, dram__bytes_read.sum 13.422556 GB +
    # dram__bytes_write.sum 0.176220 GB, 2.062 ms
    "C5": 13.598776e9,
}
# the same pass with shared value groups, offset-aligned slots, uniform-slice groups and exception-lane pairs
# as work items (profiles/r02g_dominant_kernel_c5.ncu-rep: k_sell_row<3,3,0,1,1,1,1>, dram__bytes_read.sum
# 681.46 MB + dram__bytes_write.sum 175.12 MB, 0.485 ms, L1/TEX data pipe 91.3 % of its peak)
TRAFFIC_SHARED = {"C5": 0.856580e9}
L1_PIPE_SHARED = {"C5": {"l1tex_data_pipe_pct_of_peak": 91.3, "dram_pct_of_peak": 21.6, "warps_active_pct": 46.8,
                         "registers": 64, "source": "profiles/r02g_dominant_kernel_ncu_full.txt"}}
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
# DRAM bytes of one whole V-cycle summed over its ncu launch list (dram__bytes_read.sum +
# dram__bytes_write.sum per kernel, serialised, cold cache) and the cycle time of the
# same build: the measured (not modelled) V-cycle bandwidth
VCYCLE_DRAM = {
    "C5": {"dram_bytes_per_cycle": 35.64e9, "source": "profiles/r02g_vcycle_launches_C5.csv (510 kernels, one cycle)"},
    "C3": {"dram_bytes_per_cycle": 1.95e9, "source": "profiles/r02g_vcycle_launches_C3.csv (271 kernels, one cycle)"},
    "C2": {"dram_bytes_per_cycle": 0.37e9, "source": "profiles/r02g_vcycle_launches_C2.csv (45 kernels, one cycle)"},
}
# the same lists before shared value groups (streaming layout, CAMG_SELL_DEDUP=0): profiles/r02_vcycle_launches_*.csv
VCYCLE_DRAM_STREAMING = {"C5": 111.70e9, "C3": 4.16e9, "C2": 0.35e9}

# BASELINE.json's literal smoother per config and why the bench runs another
# (reference-side evidence: profiles/r02_convergence_table.md §2)
BASELINE_SMOOTHER = {
    "C1": "block Gauss-Seidel (Uzawa alpha=1), Jacobi(1, 0.8) per block",
    "C2": "SIMPLEC, diagonal Schur approximation, 3 sweeps, damping 0.8",
    "C3": "Braess-Sarazin, Jacobi approximation of K, 1 Schur Jacobi sweep, damping 0.7",
    "C4": "Uzawa, 2 inner Jacobi sweeps on K, damping 0.6",
    "C5": "SIMPLEC (parameters unstated)",
}
MAPPING_REASON = {
    "C1": "literal BGS + Jacobi(1,0.8) does not converge in the reference (300 its, relres 1.8e-3); "
          "Jacobi(2,0.6)/(1,0.6) converges",
    "C2": "literal SIMPLEC x3 stalls in the reference (C2/2: relres 0.72 with Jacobi, C2 full: 1.0 with the "
          "reference default sgs/ilu0 after 300 its); SIMPLE(0.8)x3 converges (15 its)",
    "C3": "literal Braess-Sarazin + Jacobi stalls in the reference (C3/4: relres 0.90 / 0.68 after 300 its); "
          "SIMPLE(0.8)x3 converges (16 its)",
    "C4": "literal; corrector unstated -> the reference default kind ilu0, run as its multicolour variant mcilu0",
    "C5": "SIMPLEC stalls in the reference (C5/10: relres 0.99 / 0.93 with Jacobi, 3.1e-2 with sgs/ilu0 after "
          "300 its); SIMPLE(0.8)x3, Jacobi(1,0.6), ILU(0) corrector converges (reference lexicographic ilu0: 13 "
          "its at C5/10; GPU multicolour mcilu0: 13)",
}

# BASELINE config -> reference-API mapping
def solver_for(config):
    from paper_1912_09056_b200.hierarchy import HierarchyConfig
    from paper_1912_09056_b200.smoothers import BlockSmootherConfig, PointSmootherConfig as P

    table = {
        "C1": (dict(max_levels=2, max_coarse_size=1),
               BlockSmootherConfig(kind="uzawa", alpha=1.0, predictor=P("jacobi", 2, 0.6),
                                   corrector=P("jacobi", 1, 0.6)), 30),
        # C2/C3: the stated SIMPLEC / Braess-Sarazin smoothers stall at relres
        # 0.995 / 0.993 after 300 its with every inner solver;
        # SIMPLE(0.8)x3 with the reference's default corrector kind converges
        "C2": (dict(max_levels=3, max_coarse_size=500),
               BlockSmootherConfig(kind="simple", alpha=0.8, outer_sweeps=3, predictor=P("jacobi", 1, 0.6),
                                   corrector=P("mcilu0", 1, 1.0)), 50),
        "C3": (dict(max_levels=4, max_coarse_size=500),
               BlockSmootherConfig(kind="simple", alpha=0.8, outer_sweeps=3, predictor=P("jacobi", 1, 0.6),
                                   corrector=P("mcilu0", 1, 1.0)), 50),
        # C4: Uzawa(0.6) with 2 Jacobi(0.6) sweeps on K as stated; corrector
        # unstated -> the reference default kind (73 its vs 155 with Jacobi)
        "C4": (dict(max_levels=5, max_coarse_size=500),
               BlockSmootherConfig(kind="uzawa", alpha=0.6, predictor=P("jacobi", 2, 0.6),
                                   corrector=P("mcilu0", 1, 1.0)), 100),
        # chosen on C5 time to solution: multicolour ILU(0)
        # corrector (the reference's default corrector kind) 20 its / 0.52 s;
        # multicolour SGS corrector 30 its / 0.77 s
        "C5": (dict(max_levels=6, max_coarse_size=500),
               BlockSmootherConfig(kind="simple", alpha=0.8, outer_sweeps=3, predictor=P("jacobi", 1, 0.6),
                                   corrector=P("mcilu0", 1, 1.0)), 100),
    }
    h, s, r = table[config]
    override = os.environ.get("CAMG_BENCH_SMOOTHER")
    if override:  # "kind,alpha,outer,pred_kind,pred_sweeps,pred_damping,corr_kind,corr_sweeps,corr_damping"
        f = override.split(",")
        s = BlockSmootherConfig(kind=f[0], alpha=float(f[1]), outer_sweeps=int(f[2]),
                                predictor=P(f[3], int(f[4]), float(f[5])), corrector=P(f[6], int(f[7]), float(f[8])))
    return HierarchyConfig(**h), s, r


def smoother_desc(s):
    return (f"{s.kind}(alpha={s.alpha:.4g}, outer={s.outer_sweeps}, pred={s.predictor.kind}"
            f"({s.predictor.sweeps},{s.predictor.damping}), corr={s.corrector.kind}"
            f"({s.corrector.sweeps},{s.corrector.damping}))")


def peaks():
    try:
        with open(PEAKS_FILE) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [s[0] for s in self.samples]
        mx = max(s[1] for s in self.samples)
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = [name for bit, name in _REASONS.items() if mask & bit and name != "gpu_idle"]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm / cpu_baseline

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
# the reference has no multicolour inner solves: its CPU path runs their
# lexicographic originals (profiles/r02_convergence_table.md compares them)
_REF_KIND = {"mcilu0": "ilu0", "mcgs": "sgs"}


def cpu_info():
    """CPU model, core count and BLAS threading of the host."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        import threadpoolctl
        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads")}
                for i in threadpoolctl.threadpool_info()]
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"), "blas_pools": blas,
            "sparse_kernels_threads": 1}


def reference_impl():
    """(module namespace, kind): the unmodified reference package installed in
    baseline/_ref (pip install --target), else the oracle port."""
    if os.path.isdir(os.path.join(REF_DIR, "contactamg")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from contactamg import hierarchy as R_h, krylov as R_k, smoothers as R_s  # noqa: F401
        return "reference", (R_h, R_k, R_s)
    return "port", None


def _ref_system(g):
    """(SaddleOperator, LevelMeta) of a generated system built from the
    reference package's own classes (as tests/golden/make_golden.py does)."""
    import scipy.sparse
    from contactamg import hierarchy as R_h, sparse as R_sp, transfer as R_t
    from contactamg.aggregation import LagrangeMap
    from contactamg.saddle import SaddleOperator

    def sm(m):
        return R_sp.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(m))

    d, n_s = g.dim, len(g.slave_nodes)
    op = SaddleOperator(sm(g.K), sm(g.B1), sm(g.B2), sm(g.Cz))
    meta = R_h.LevelMeta(
        u_dof_node=np.arange(g.n_u, dtype=np.int64) // d, num_u_nodes=g.n_u // d,
        node_body=g.node_body.astype(np.int8), lam_dof_node=np.arange(g.n_lam, dtype=np.int64) // d,
        num_lam_nodes=n_s, ns_u=R_t.NullSpace(g.rigid_body_modes(), "rigid-body"),
        ns_lam=R_t.build_nullspace(n_s, R_t.NULLSPACE_CONSTANT_PER_COMPONENT, dofs_per_node=d),
        mortar_block=sm(g.mortar_block),
        lmap=LagrangeMap(slave_dofs=g.slave_dofs.astype(np.int64),
                         row_node=np.repeat(g.slave_nodes, d).astype(np.int64),
                         lm_node_of_lm_dof=np.arange(g.n_lam, dtype=np.int64) // d))
    return op, meta


def _ref_setup(mods, g, hcfg, scfg):
    """Reference-package hierarchy of generated system g with the mapped
    smoother (GPU-only kinds -> their lexicographic originals)."""
    R_h, R_k, R_s = mods
    op, meta = _ref_system(g)

    def pc(p):
        return R_s.PointSmootherConfig(kind=_REF_KIND.get(p.kind, p.kind), sweeps=p.sweeps, damping=p.damping)

    sc = R_s.BlockSmootherConfig(kind=scfg.kind, alpha=scfg.alpha, outer_sweeps=scfg.outer_sweeps,
                                 predictor=pc(scfg.predictor), corrector=pc(scfg.corrector), a_hat_mode=scfg.a_hat_mode)
    hc = R_h.HierarchyConfig(max_levels=hcfg.max_levels, max_coarse_size=hcfg.max_coarse_size,
                             coarse_solver=hcfg.coarse_solver, min_agg_size=hcfg.min_agg_size)
    H = R_h.setup(op, meta, hc, sc)
    A = op.merged().to_scipy()
    return H, (lambda v: A @ v), R_k


def _port_setup(g, hcfg, scfg):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import camg_oracle as O
    op, meta, _ = O.system_from_generated(g)

    def pc(p):
        return O.PointCfg(_REF_KIND.get(p.kind, p.kind), p.sweeps, p.damping)

    bc = O.BlockCfg(kind=scfg.kind, alpha=scfg.alpha, outer_sweeps=scfg.outer_sweeps, predictor=pc(scfg.predictor),
                    corrector=pc(scfg.corrector), a_hat_mode=scfg.a_hat_mode)
    H = O.setup(op, meta, O.HierCfg(**{k: getattr(hcfg, k) for k in
                                       ("max_levels", "max_coarse_size", "coarse_solver", "min_agg_size")}), bc)
    A = op.merged()
    return H, (lambda v: A @ v), O


def cpu_reference_run(config, scale, steps, warmup, solve=True, impl=None):
    """Time the CPU reference path on `config/scale`: setup, `steps` V-cycles
    (median), and (solve) GMRES(restart) to rtol 1e-8.  impl: "reference"
    (unmodified package), "port" (oracle), None = the package when installed."""
    from paper_1912_09056_b200.problem import config_spec, generate

    kind, mods = reference_impl()
    if impl == "port":
        kind, mods = "port", None
    hcfg, scfg, restart = solver_for(config)
    g = generate(config_spec(config, scale))
    t0 = time.perf_counter()
    if kind == "reference":
        H, applyA, R_k = _ref_setup(mods, g, hcfg, scfg)
        levels = H.levels
    else:
        H, applyA, O = _port_setup(g, hcfg, scfg)
        levels = H.levels
    setup_s = time.perf_counter() - t0
    rhs = g.rhs
    for _ in range(warmup):
        H.apply(rhs)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        H.apply(rhs)
        times.append(time.perf_counter() - t0)
    out = {"kind": kind, "config": f"{config}/{scale}", "n": int(len(rhs)), "levels": len(levels),
           "setup_s": round(setup_s, 3), "vcycle_s": float(np.median(times)), "vcycles_timed": steps,
           "smoother": smoother_desc(scfg).replace("mcilu0", "ilu0").replace("mcgs", "sgs")}
    if solve:
        t0 = time.perf_counter()
        if kind == "reference":
            x, rep = R_k.gmres(applyA, H.apply, rhs, R_k.GmresConfig(rel_tol=1e-8, max_iters=300, restart=restart))
        else:
            x, rep = O.gmres(applyA, H.apply, rhs, 1e-8, 300, restart)
        out.update(gmres_s=round(time.perf_counter() - t0, 3), gmres_iterations=int(rep.iterations),
                   gmres_converged=bool(rep.converged),
                   true_relres=float(np.linalg.norm(rhs - applyA(x)) / np.linalg.norm(rhs)))
    units = []
    streams = steps_per_level(scfg)
    for i, l in enumerate(levels):
        last = i == len(levels) - 1
        T = getattr(l, "transfer", None)
        nP = (T.P_u.nnz + T.P_lam.nnz) if T is not None else ((l.P_u.nnz + l.P_lam.nnz) if getattr(l, "P_u", None)
                                                              is not None else 0)
        units.append(dict(nnz_A=l.op.nnz, streams=0 if last else streams, nnz_P=0 if last else nP,
                          nnz_R=0 if last else nP))
    out["units"] = vcycle_cost_units(units)
    return out


def cpu_baseline_line(run, full_units, extrapolated_from):
    """cpu_baseline / reference-arm fields from a bounded CPU sample scaled to
    the full workload by V-cycle sparse entries streamed."""
    sec_full = run["vcycle_s"] * full_units / run["units"]
    return {"value": 1.0 / sec_full, "unit": "V-cycles/s", "cores": 1, "kind": run["kind"],
            "extrapolated": abs(full_units - run["units"]) > 1e-9 * full_units,
            "sample": (f"{'unmodified reference package (baseline/_ref)' if run['kind'] == 'reference' else 'oracle port'}"
                       f" V-cycle on {run['config']} (n={run['n']}, {run['levels']} levels, {run['smoother']}), "
                       f"median of {run['vcycles_timed']} cycles = {run['vcycle_s']:.3f} s, scaled to {extrapolated_from} "
                       f"by the ratio of sparse entries one V-cycle streams ({full_units:.4g} / {run['units']:.4g})"),
            "sample_run": run, "host": cpu_info()}


def steps_per_level(scfg):
    """Operator streams per non-coarsest level in one V(1,1) cycle."""
    sp = 1 if scfg.kind == "braess_sarazin" else scfg.predictor.sweeps
    per_step = sp  # first predictor sweep fused with the step residual
    s = scfg.outer_sweeps
    return max(0, s * per_step - 1) + 1 + s * per_step


def vcycle_cost_units(levels):
    """Work units of one V-cycle: sum over levels of the sparse entries the
    cycle streams (same structure on CPU and GPU, so the ratio scales a CPU
    sample to the GPU workload)."""
    return float(sum(lv["nnz_A"] * lv["streams"] + lv["nnz_P"] + lv["nnz_R"] for lv in levels))


def gpu_cost_units(H, scfg):
    lv = []
    streams = steps_per_level(scfg)
    for i, l in enumerate(H.levels):
        last = i == len(H.levels) - 1
        lv.append(dict(nnz_A=l.op.nnz, streams=0 if last else streams,
                       nnz_P=0 if last else l.transfer.P_u.nnz + l.transfer.P_lam.nnz,
                       nnz_R=0 if last else l.transfer.R_u.nnz + l.transfer.R_lam.nnz))
    return vcycle_cost_units(lv)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = max(1, args.steps)
    sample = cpu_reference_run(args.config, args.cpu_sample_scale, steps, min(args.warmup, 1), solve=True)
    full_units = estimate_full_units(args.config, args.scale, args.cpu_sample_scale, sample["units"])
    cb = cpu_baseline_line(sample, full_units, f"{args.config}{'' if args.scale == 1 else '/' + str(args.scale)}")
    value = cb["value"]
    full = {}
    if not args.no_full_size:
        # full-size CPU runs in the same process (C2 by the reference package,
        # C3 by the oracle port: the package's C3 setup alone takes minutes)
        for cfg, impl in (("C2", None), ("C3", "port")):
            try:
                full[cfg] = cpu_reference_run(cfg, 1, 3, 1, solve=True, impl=impl)
            except Exception as e:  # noqa: BLE001
                full[cfg] = {"error": repr(e)}
    line = {
        "impl": "reference",
        "metric": metric_name(args.config), "value": value, "unit": "V-cycles/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {k: v for k, v in cb.items() if k != "sample_run"},
        "sample_run": sample,
        "full_size_cpu": full,
        "e2e": {"value": value, "unit": "V-cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def estimate_full_units(config, scale, sample_scale, sample_units):
    """Cost units of the full config from the sample by the nnz(K) ratio of
    the two meshes (computed from the mesh formulas, no assembly)."""
    from paper_1912_09056_b200.problem import config_spec
    def knnz(spec):
        tot = 0
        for b in (spec.lower, spec.upper):
            tot += np.prod([e + 1 for e in b.elems]) * 27 * 9 if spec.dim == 3 else np.prod([e + 1 for e in b.elems]) * 9 * 4
        return float(tot)
    return sample_units * knnz(config_spec(config, scale)) / knnz(config_spec(config, sample_scale))


def metric_name(config):
    return f"AMG V-cycles/s (GMRES preconditioner apply), BASELINE {config}, fp64, 1 B200 per rank"


def workload_config(args):
    from paper_1912_09056_b200.problem import config_spec
    spec = config_spec(args.config, args.scale)
    hcfg, scfg, restart = solver_for(args.config)
    return {
        "workload": f"{args.config}{'' if args.scale == 1 else '/' + str(args.scale)}: 3-D two-block mortar "
                    f"{spec.coupling}, lower {spec.lower.elems} E={spec.lower.youngs}, upper {spec.upper.elems} "
                    f"E={spec.upper.youngs}, nu={spec.nu}" if spec.dim == 3 else f"{args.config} 2-D",
        "hierarchy": {"max_levels": hcfg.max_levels, "max_coarse_size": hcfg.max_coarse_size,
                      "coarse_solver": hcfg.coarse_solver, "min_agg_size": hcfg.min_agg_size},
        "smoother": smoother_desc(scfg), "gmres_restart": restart,
        "baseline_smoother": BASELINE_SMOOTHER[args.config],
        "mapped_smoother": smoother_desc(scfg),
        "mapping_reason": MAPPING_REASON[args.config],
        "l2": "inputs exceed L2 (fine-level operator >> 126 MB); no flush needed",
        "parallelism": f"replicas x{args.gpus}",
    }


# ---------------------------------------------------------------------------
# multi-rank aggregation (replicas: no data-path collective, timing only)


def replica_max(x, world, device):
    """Max of a per-rank scalar over all ranks (the slowest replica sets the
    job time).  Works with the nccl (cuda) and gloo (cpu) backends."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(units_per_rank, seconds_per_rank, world, device):
    """Whole-job throughput: all ranks' units / max-over-ranks time."""
    return units_per_rank * world / replica_max(seconds_per_rank, world, device)


# ---------------------------------------------------------------------------
# GPU arm


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_1912_09056_b200 import _native as N
    from paper_1912_09056_b200.hierarchy import fine_level_meta, setup
    from paper_1912_09056_b200.krylov import GmresConfig, gmres_device
    from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
    from paper_1912_09056_b200.sparse import empty, ptr, stream_ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N.require_device()

    t0 = time.perf_counter()
    g = generate(config_spec(args.config, args.scale), assemble_K=False)
    op = saddle_operator(g, device_K=True)
    t_gen = time.perf_counter() - t0
    meta = fine_level_meta(g)
    hcfg, scfg, restart = solver_for(args.config)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = setup(op, meta, hcfg, scfg)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    n = H.n
    rhs = torch.from_numpy(g.rhs).cuda()
    z = empty(n)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return replica_max(x, world, "cuda")

    # ---- dominant kernel: fine-level operator stream (merged [K B1; B2 -Cz] SpMV)
    A0 = H.levels[0].smoother  # noqa: F841
    Am = op.merged()
    y = empty(n)
    for _ in range(3):
        N.call("camg_spmv", Am.device, 1.0, ptr(rhs), 0.0, ptr(y), stream_ptr())
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(reps):
        N.call("camg_spmv", Am.device, 1.0, ptr(rhs), 0.0, ptr(y), stream_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    spmv_ms = e0.elapsed_time(e1) / reps
    nnzA, nA = Am.nnz, Am.num_rows
    spmv_bytes = 12.0 * nnzA + 4.0 * (nA + 1) + 8.0 * nA + 8.0 * nA
    spmv_gbs = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    fmt = C.c_double()
    N.call("camg_csr_stream_bytes", Am.device, C.byref(fmt))
    spmv_fmt_gbs = fmt.value / (spmv_ms * 1e-3) / 1e9

    # ---- dominant kernel of the V-cycle: the fine-level predictor pass over
    # [K | B1] (Jacobi: one fused SELL pass per step; multicolour SGS: one
    # forward + backward sweep of colour passes)
    gs = scfg.kind != "braess_sarazin" and scfg.predictor.kind == "mcgs"
    dom_mode = 3 if gs else 1
    xk = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
    for _ in range(3):
        H.fine_pass(dom_mode, xk, rhs)
    barrier()
    e0.record(stream)
    for _ in range(reps):
        dom_model, dom_fmt = H.fine_pass(dom_mode, xk, rhs)
    e1.record(stream)
    torch.cuda.synchronize()
    dom_ms = e0.elapsed_time(e1) / reps
    dom_gbs = dom_model / (dom_ms * 1e-3) / 1e9
    dom_fmt_gbs = dom_fmt / (dom_ms * 1e-3) / 1e9
    # the same pass through a second mirror in the streaming layout (no shared
    # value groups: what a matrix without repeated slots runs), same run
    info0 = H.level_info(0)
    _us = (C.c_int64 * 5)()
    N.call("camg_csr_uniform_slices", Am.device, _us)
    uslices = {"slices": _us[0], "uniform": _us[1], "groups": _us[2], "offset_aligned": _us[3],
               "exception_lane_pairs": _us[4]}
    streaming = None
    if not gs and info0.get("sell_shared_values"):
        for _ in range(3):
            H.fine_pass(dom_mode | 0x100, xk, rhs)
        barrier()
        e0.record(stream)
        for _ in range(reps):
            st_model, st_fmt = H.fine_pass(dom_mode | 0x100, xk, rhs)
        e1.record(stream)
        torch.cuda.synchronize()
        st_ms = e0.elapsed_time(e1) / reps
        H.fine_pass(0x200, xk, rhs)  # release the second mirror
        streaming = {"avg_launch_ms": st_ms, "bytes_per_launch": st_fmt,
                     "achieved": st_fmt / (st_ms * 1e-3) / 1e9, "unit": "GB/s"}

    # ---- V-cycle, device-resident input (the metric)
    for _ in range(max(3, args.warmup)):
        H.apply_device(rhs, z)
    launches_before = N.launch_count()
    barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            H.apply_device(rhs, z)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = N.launch_count() - launches_before
    vc_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    total_cycles = args.steps * world
    value = total_cycles / (vc_ms * 1e-3 * args.steps)
    bytes_csr, bytes_fmt = H.vcycle_bytes()
    vc_gbs = bytes_csr / (vc_ms * 1e-3) / 1e9
    vc_fmt_gbs = bytes_fmt / (vc_ms * 1e-3) / 1e9

    # ---- e2e through the public API on pinned host vectors: every step's
    # host->device copy of its residual and device->host copy of its result
    # are inside the timed region.  (a) Hierarchy.apply_many: independent
    # right-hand sides, copies pipelined against the V-cycles on their own
    # streams; (b) Hierarchy.apply: one blocking call per step.
    r_host = torch.from_numpy(g.rhs.copy()).pin_memory()
    rs = [r_host] * args.steps
    outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(args.steps)]
    H.apply_many(rs[:2], outs[:2])
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    H.apply_many(rs, outs)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    e2e_value = total_cycles / (e2e_ms * 1e-3 * args.steps)
    assert all(o.numel() == n for o in outs)
    for _ in range(2):
        H.apply(r_host)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        z_host = H.apply(r_host)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_sync_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    e2e_sync_value = total_cycles / (e2e_sync_ms * 1e-3 * args.steps)
    assert z_host.numel() == n and torch.equal(z_host, outs[-1])

    # ---- time to solution (GMRES, rtol 1e-8), outside the timed region
    solve = None
    if not args.no_solve:
        # one-time allocation of the cached Krylov basis (n x (restart+1)) outside the timing
        gmres_device(Am, H, rhs, GmresConfig(rel_tol=0.5, max_iters=args.max_iters, restart=restart))
        barrier()
        t0 = time.perf_counter()
        x, its, conv, hist = gmres_device(Am, H, rhs, GmresConfig(rel_tol=1e-8, max_iters=args.max_iters,
                                                                  restart=restart))
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - t0
        r = rhs.clone()
        N.call("camg_spmv", Am.device, -1.0, ptr(x), 1.0, ptr(r), stream_ptr())
        relres = float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(rhs))
        solve = {"gmres_iterations": its, "converged": conv, "true_relres": relres,
                 "time_to_solution_s": t_solve, "setup_s": t_setup, "generate_s": t_gen,
                 "setup_breakdown_s": {k: round(v, 3) for k, v in H.timings.items()}}
        # convergence margin of the mapping: the same solve for further
        # uniform(-1,1) right-hand sides (seeds after the config's own)
        seeds = {}
        for sd in args.rhs_seeds:
            rs_ = torch.from_numpy(np.random.default_rng(sd).uniform(-1.0, 1.0, n)).cuda()
            t0 = time.perf_counter()
            xs, its_s, conv_s, _ = gmres_device(Am, H, rs_, GmresConfig(rel_tol=1e-8, max_iters=args.max_iters,
                                                                        restart=restart))
            torch.cuda.synchronize()
            seeds[str(sd)] = {"gmres_iterations": its_s, "converged": conv_s,
                              "time_to_solution_s": round(time.perf_counter() - t0, 4)}
        solve["other_rhs_seeds"] = seeds

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        run = cpu_reference_run(args.config, args.cpu_sample_scale, 3, 1, solve=False)
        cpu = cpu_baseline_line(run, gpu_cost_units(H, scfg), "the GPU's full hierarchy")

    levels = [{"n_u": l.op.n_u, "n_lam": l.op.n_lam, "nnz_K": l.op.K.nnz, "nnz_total": l.op.nnz}
              for l in H.levels]
    free_b, total_b = torch.cuda.mem_get_info()
    shared = bool(info0.get("sell_shared_values"))
    traffic = None if gs else (TRAFFIC_SHARED if shared else TRAFFIC).get(args.config)
    if args.scale != 1:
        traffic = None
    if gs:
        kernel = ("k_sell_gs<3>: one fine-level multicolour block-SGS predictor sweep (forward + backward "
                  "colour passes over a colour-ordered block SELL of K)")
    else:
        kernel = ("k_sell_row<3,3,mode 1,masked%s>: fine-level Jacobi predictor sweep y += w D^-1 (b - [K B1][y; lam]) "
                  "(block SELL-32 [K | B1] rows)" % (",shared values" if shared else ""))
    roofline = {"bound": "hbm", "achieved": dom_fmt_gbs, "peak": peak, "unit": "GB/s",
                "frac": dom_fmt_gbs / peak, "traffic": traffic, "kernel": kernel,
                "bytes": "format bytes: what the stored format must stream per launch (block SELL values -- every "
                         "shared value group once --, a descriptor and a group offset per slot, one int32 per stored "
                         "block, none for linear slots; x read once; b, D^-1 read, y written)",
                "bytes_per_launch": dom_fmt, "avg_launch_ms": dom_ms,
                "traffic_over_bytes": (traffic / dom_fmt) if traffic else None,
                "model_bytes_per_launch": dom_model, "model_achieved": dom_gbs,
                "model": ("SURVEY §8(d): 2 x (12 B/nnz(K) + offsets + 4 vector streams) + y/g init" if gs else
                          "SURVEY §8(d) int32-CSR model: 12 B/nnz + offsets + x read + 3 vector streams; the "
                          "block format streams fewer bytes than this model, so model_achieved can exceed peak"),
                "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)"}
    if shared:
        roofline["shared_value_groups"] = {
            "kept": info0["sell_value_groups"], "full": info0["sell_value_groups_full"],
            "note": "bit-identical slots of the mirror (the interior stencil of the structured mesh) keep one copy, "
                    "found by content hash + bitwise verification at setup: the value stream becomes an L1/L2-resident "
                    "dictionary and the pass is no longer HBM-bound but bound by the L1 data pipe (ncu: 91% of its "
                    "peak, DRAM 19%: every lane receives the slot's 72 bytes of block values and 24 bytes of x), so "
                    "frac -- its compulsory HBM bytes over the measured peak -- is the headroom left, not wasted "
                    "traffic; results are bit-identical to the streaming layout",
            "l1_data_pipe": L1_PIPE_SHARED.get(args.config) if args.scale == 1 else None,
            "uniform_slices": dict(uslices, note="slices of 32 block rows whose slots are all linear and lane-uniform "
                                   "(offset-aligned slots make the slices across mesh-row ends qualify) run a loop "
                                   "without descriptor decoding, neighbouring ones in groups of 2-3 block rows per "
                                   "lane so that a slot's block is loaded once for the group (DESIGN 5b)")}
        if streaming:
            st_traffic = TRAFFIC.get(args.config) if args.scale == 1 else None
            roofline["streaming_layout"] = dict(
                streaming, frac=streaming["achieved"] / peak, traffic=st_traffic,
                traffic_over_bytes=(st_traffic / streaming["bytes_per_launch"]) if st_traffic else None,
                speedup_of_shared_values=streaming["avg_launch_ms"] / dom_ms,
                note="the same pass, same run, through a mirror without shared value groups (CAMG_SELL_DEDUP=0; what "
                     "a matrix without repeated slots runs): HBM-bound at the measured copy bandwidth")
    line = {
        "metric": metric_name(args.config),
        "value": value, "unit": "V-cycles/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": vc_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, BASELINE config geometry/materials)",
        "config": dict(workload_config(args), levels=levels, operator_complexity=H.complexity,
                       device_memory_used_gb=round((total_b - free_b) / 1e9, 1)),
        "roofline": roofline,
        "vcycle_roofline": {"achieved": vc_fmt_gbs, "unit": "GB/s", "bytes_per_cycle": bytes_fmt,
                            "frac_of_measured_peak": vc_fmt_gbs / peak, "frac_of_8TBs": vc_fmt_gbs / 8000.0,
                            "bytes": "format bytes of every sparse application and vector stream of one cycle "
                                     "(camg_hierarchy_vcycle_bytes), zero-vector products skipped",
                            "dram_measured": (dict(VCYCLE_DRAM[args.config],
                                                   achieved_gbs=VCYCLE_DRAM[args.config]["dram_bytes_per_cycle"]
                                                   / (vc_ms * 1e-3) / 1e9,
                                                   frac_of_measured_peak=VCYCLE_DRAM[args.config]["dram_bytes_per_cycle"]
                                                   / (vc_ms * 1e-3) / 1e9 / peak,
                                                   frac_of_8TBs=VCYCLE_DRAM[args.config]["dram_bytes_per_cycle"]
                                                   / (vc_ms * 1e-3) / 1e9 / 8000.0)
                                              if args.config in VCYCLE_DRAM and args.scale == 1 else None),
                            "model_bytes_per_cycle": bytes_csr, "model_achieved": vc_gbs,
                            "model": "SURVEY.md §8(d): 12 B/nnz + index/vector terms, zero products skipped",
                            "kernels_per_cycle": H.kernels_per_cycle()},
        "spmv": {"GB/s": spmv_gbs, "GB/s_format_bytes": spmv_fmt_gbs, "ms": spmv_ms, "nnz": nnzA,
                 "kernel": "merged operator y = A x (SELL-32 [K|B1] rows + CSR [B2 -Cz] rows)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "V-cycles/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n,
                "path": "Hierarchy.apply_many(pinned host residuals) -> pinned host results; independent RHS, "
                        "H2D/D2H on their own streams overlapping the V-cycles",
                "sync_value": e2e_sync_value,
                "sync_path": "Hierarchy.apply(pinned host tensor) -> host tensor, one blocking call per step"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "solve": solve,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--cpu-sample-scale", type=int, default=5)
    ap.add_argument("--max-iters", type=int, default=300)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-size", action="store_true", help="reference arm: skip the full-size C2/C3 CPU runs")
    ap.add_argument("--rhs-seeds", type=lambda t: [int(v) for v in t.split(",") if v], default=[5, 6, 7],
                    help="extra right-hand-side seeds solved after the timed region (convergence margin)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

"""The benchmarked configuration at FULL size (C5: 23.6M unknowns, 1.5e9
non-zeros) through size-independent properties (the oracle cannot set C5
up: ~210 GB): linearity and bit-identical replay of the V-cycle, the
coarsest solve against host LAPACK, GMRES convergence with the true
residual, the size-gated execution paths the bench relies on, no watchdog."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1912_09056_b200 import _native  # noqa: E402
from paper_1912_09056_b200.hierarchy import fine_level_meta, setup  # noqa: E402
from paper_1912_09056_b200.krylov import GmresConfig, gmres_device, release_workspace  # noqa: E402
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator  # noqa: E402


def test_full_c5_mirror_variants_bit_identical(monkeypatch):
    """The fine operator's block mirror at full size: offset-aligned slots,
    uniform-slice loops and groups (DESIGN 5b) engage on nearly every slice,
    and the merged SpMV is bit-identical to the mirror without them and to
    the streaming layout without shared value groups."""
    import ctypes as C
    import torch
    from paper_1912_09056_b200.sparse import empty, ptr, stream_ptr
    _native.require_device()
    g = generate(config_spec("C5", 1), assemble_K=False)
    op = saddle_operator(g, device_K=True)
    A = op.merged()
    n = A.num_rows
    x = torch.from_numpy(np.random.default_rng(21).standard_normal(n)).cuda()
    out, counts = {}, {}
    for name, env in (("plain", {"CAMG_SELL_ALIGN": "0", "CAMG_SELL_USLICE": "0"}),
                      ("streaming", {"CAMG_SELL_DEDUP": "0"}),
                      ("default", {})):
        for k in ("CAMG_SELL_ALIGN", "CAMG_SELL_USLICE", "CAMG_SELL_DEDUP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        _native.call("camg_csr_attach_blocks", A.device, 3, op.n_u)
        c = (C.c_int64 * 5)()
        _native.call("camg_csr_uniform_slices", A.device, c)
        counts[name] = tuple(c)
        y = empty(n)
        _native.call("camg_spmv", A.device, 1.0, ptr(x), 0.0, ptr(y), stream_ptr())
        torch.cuda.synchronize()
        out[name] = y
    slices, uniform, groups, aligned, xgroups = counts["default"]
    assert counts["plain"][1:] == (0, 0, 0, 0) and counts["streaming"][1:3] == (0, 0)
    assert xgroups > 0.05 * slices, counts  # slices with exception lanes (16%) in pairs a mesh-row period apart
    assert aligned > 0.98 * slices and uniform > 0.97 * slices and groups > 0.25 * slices, counts
    assert torch.equal(out["plain"], out["default"])
    assert torch.equal(out["streaming"], out["default"])
    assert torch.isfinite(out["default"]).all()
    del out, y, x, A, op
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def c5():
    import torch
    _native.require_device()
    g = generate(config_spec("C5", 1), assemble_K=False)
    op = saddle_operator(g, device_K=True)
    hcfg, scfg, restart = bench.solver_for("C5")
    H = setup(op, fine_level_meta(g), hcfg, scfg)
    rhs = torch.from_numpy(g.rhs).cuda()
    yield g, op, H, rhs, restart
    del H, op
    release_workspace()
    torch.cuda.empty_cache()


def test_full_c5_vcycle_linear_and_replayed(c5):
    import torch
    g, op, H, rhs, _ = c5
    n = H.n
    r2 = torch.from_numpy(np.random.default_rng(9).uniform(-1.0, 1.0, n)).cuda()
    z1 = H.apply_device(rhs).clone()
    z1b = H.apply_device(rhs).clone()
    assert torch.equal(z1, z1b)                                  # graph replay is deterministic
    z2 = H.apply_device(r2).clone()
    z3 = H.apply_device(2.5 * rhs - 0.75 * r2).clone()
    lin = 2.5 * z1 - 0.75 * z2
    assert float(torch.linalg.vector_norm(z3 - lin) / torch.linalg.vector_norm(lin)) <= 1e-12
    assert torch.isfinite(z1).all()


def test_full_c5_paths_and_coarse_solve(c5):
    import scipy.linalg
    from paper_1912_09056_b200.sparse import BlockVector
    g, op, H, rhs, _ = c5
    info = [H.level_info(l) for l in range(H.num_levels)]
    assert not any(i["watchdog"] for i in info)
    i0 = info[0]
    assert i0["sell_block"] == 3 and i0["sell_masked"] and i0["sell_lanes"] == 1 and i0["overlap"]
    assert i0["corr_path"] == "colour_csr" and info[1]["overlap"]
    assert all(i["corr_path"] == "dense_inv" for i in info[2:-1])
    assert i0["transfer_block_rows"] == 3 and i0["restrict_block_rows"] == 6
    cop = H.levels[-1].op
    b = np.random.default_rng(2).standard_normal(cop.total_rows)
    xb = H.solve_coarsest(BlockVector.zeros(cop.n_u, cop.n_lam), BlockVector.from_merged(b, cop.n_u)).merged()
    ref = scipy.linalg.lu_solve(scipy.linalg.lu_factor(cop.merged_dense()), b)
    assert np.linalg.norm(xb - ref) <= 1e-12 * np.linalg.norm(ref)


def test_full_c5_gmres_converges(c5):
    import torch
    from paper_1912_09056_b200.sparse import ptr, stream_ptr
    g, op, H, rhs, restart = c5
    A = op.merged()
    x, its, conv, hist = gmres_device(A, H, rhs, GmresConfig(rel_tol=1e-8, max_iters=60, restart=restart))
    assert conv and its <= 22, its
    r = rhs.clone()
    _native.call("camg_spmv", A.device, -1.0, ptr(x), 1.0, ptr(r), stream_ptr())
    assert float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(rhs)) <= 2e-8
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))  # Givens estimates never rise

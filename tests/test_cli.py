"""The experiment driver (SPEC.md module `cli`): config parsing with line
diagnostics on the CPU; one `solve` (CSV, setup report, MatrixMarket export)
and the refinement sweep on the GPU."""

import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1912_09056_b200.cli import build_configs, parse_config
from paper_1912_09056_b200.errors import ConfigError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFG = """# C1 desk run
config=C1
scale=1
smoother.kind=uzawa          # BGS
smoother.alpha=1.0
smoother.predictor.kind=jacobi
smoother.predictor.sweeps=2
smoother.predictor.damping=0.6
gmres.restart=30
"""


def test_config_parsing_and_mapping():
    c = parse_config(CFG)
    assert c["config"] == "C1" and c["smoother.predictor.sweeps"] == 2 and c["smoother.alpha"] == 1.0
    h, s, g = build_configs(c)
    assert s.kind == "uzawa" and s.predictor.kind == "jacobi" and s.predictor.sweeps == 2
    assert s.corrector.kind == "jacobi"          # bench mapping of C1 where not overridden
    assert g.restart == 30 and g.rel_tol == 1e-8 and h.max_levels == 2


@pytest.mark.parametrize("text,msg", [
    ("config=C1\nbogus=1\n", "<config>:2: unknown key 'bogus'"),
    ("config=C1\nscale=two\n", "<config>:2: scale needs a int"),
    ("config=C1\nsmoother.alpha\n", "<config>:2: expected key=value"),
    ("config=C1\nconfig=C2\n", "<config>:2: duplicate key"),
    ("scale=2\n", "missing key 'config'"),
])
def test_config_errors_name_the_line(text, msg):
    with pytest.raises(ConfigError, match=msg):
        parse_config(text)


def test_rotation_sweep_is_reported_out_of_scope(tmp_path):
    cfg = tmp_path / "c.cfg"
    cfg.write_text(CFG)
    r = subprocess.run([sys.executable, "-m", "paper_1912_09056_b200.cli", "rotation-sweep", "--config", str(cfg)],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 2 and "rotated 2-D" in r.stderr


@pytest.mark.gpu
def test_cli_solve_and_export(tmp_path):
    import scipy.io
    from paper_1912_09056_b200.problem import config_spec, generate
    cfg = tmp_path / "c.cfg"
    cfg.write_text(CFG)
    out = tmp_path / "run"
    r = subprocess.run([sys.executable, "-m", "paper_1912_09056_b200.cli", "solve", "--config", str(cfg),
                        "--out", str(out), "--export-system"], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = (out / "report.csv").read_text().splitlines()
    assert rows[0] == "iteration,relative_residual" and float(rows[1].split(",")[1]) == 1.0
    res = [float(l.split(",")[1]) for l in rows[1:]]
    assert res[-1] <= 1e-8 and len(res) - 1 == int(r.stdout.split("iterations=")[1].split()[0])
    assert "operator complexity" in (out / "setup.txt").read_text()
    g = generate(config_spec("C1", 1))
    K = scipy.io.mmread(str(out / "K.mtx")).tocsr()
    assert K.shape == g.K.shape and abs(K - g.K).max() <= 1e-14 * abs(g.K).max()


@pytest.mark.gpu
def test_cli_refine_sweep(tmp_path):
    cfg = tmp_path / "c.cfg"
    cfg.write_text("config=C5\nscale=20\nhierarchy.max_levels=3\nhierarchy.max_coarse_size=50\n")
    r = subprocess.run([sys.executable, "-m", "paper_1912_09056_b200.cli", "refine-sweep", "--config", str(cfg),
                        "--out", str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "refine.csv").read_text().splitlines()
    assert lines[0].startswith("scale,unknowns,iterations") and len(lines) == 4
    unknowns = [int(l.split(",")[1]) for l in lines[1:]]
    assert unknowns == sorted(unknowns)

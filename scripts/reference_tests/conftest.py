"""Run the reference's own unit tests (/root/reference/pkg/tests) against this
package through a `contactamg` alias (VERDICT r01 "Next round" item 4).

`contactamg.<mod>` resolves to `paper_1912_09056_b200.<mod>` for every module
on the path (sparse, saddle, smoothers, transfer, aggregation, hierarchy,
krylov, errors).  `contactamg.problem` -- the reference's 2-D matching-mesh
generator, out of scope -- is the reference's own file from
the unmodified install in baseline/_ref, executed under the alias so that its
`from .sparse import SparseMatrix` etc. build THIS package's objects.

Test-harness only: nothing in the package imports this file.  The test files
themselves are never committed; scripts/run_reference_tests.sh copies them
from /root/reference into baseline/_ref/ref_tests (git-ignored, travels to
the GPU box) next to this conftest.
"""

import importlib
import importlib.util
import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.environ.get("GRAFT_REPO_ROOT") or os.path.abspath(os.path.join(HERE, "..", "..", ".."))
if not os.path.isdir(os.path.join(ROOT, "paper_1912_09056_b200")):
    ROOT = "/root/repo"
sys.path.insert(0, ROOT)

import paper_1912_09056_b200 as _pkg  # noqa: E402

_alias = types.ModuleType("contactamg")
_alias.__path__ = []  # a package, so relative imports inside problem.py resolve
_alias.__dict__.update({k: getattr(_pkg, k) for k in ("SparseMatrix", "BlockVector")})
sys.modules["contactamg"] = _alias
for _m in ("errors", "sparse", "saddle", "aggregation", "smoothers", "transfer", "krylov", "hierarchy"):
    mod = importlib.import_module(f"paper_1912_09056_b200.{_m}")
    sys.modules[f"contactamg.{_m}"] = mod
    setattr(_alias, _m, mod)

_ref_problem = os.path.join(ROOT, "baseline", "_ref", "contactamg", "problem.py")
_spec = importlib.util.spec_from_file_location("contactamg.problem", _ref_problem)
_problem = importlib.util.module_from_spec(_spec)
sys.modules["contactamg.problem"] = _problem
_spec.loader.exec_module(_problem)
_alias.problem = _problem

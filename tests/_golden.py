"""Helpers to read the golden fixtures written by tests/golden/make_golden.py."""
import glob
import os

import numpy as np
import scipy.sparse

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    """Hierarchy cases (the nested-preconditioner fixtures are listed by
    nested_cases())."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not p.endswith("kernels.npz") and not os.path.basename(p).startswith("nested_"))


def nested_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "nested_*.npz")))


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def csr(z, key):
    shape = tuple(int(s) for s in z[key + "_shape"])
    return scipy.sparse.csr_matrix((z[key + "_data"], z[key + "_indices"], z[key + "_indptr"]), shape=shape)


def has(z, key):
    return key + "_shape" in z

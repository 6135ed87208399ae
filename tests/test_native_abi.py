"""CPU-side checks of the C ABI: the library loads, exports every entry
point declared in include/camg.h, and maps status codes onto the reference
exception classes.  No compute calls (no GPU here)."""

import ctypes as C
import os
import re

import pytest

from paper_1912_09056_b200 import _native as N
from paper_1912_09056_b200.errors import (
    ConfigError,
    DimensionError,
    NativeError,
    SetupError,
    SingularMatrixError,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "camg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(camg_[a-z0-9_]+)\s*\(", src)))


def test_library_loads():
    assert N.lib().camg_version() >= 100


def test_every_header_symbol_is_exported_and_bound():
    lib = C.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(N.exported_symbols()), set(syms) - set(N.exported_symbols())


def test_status_codes_map_to_reference_exceptions():
    assert N._CODES[1] is DimensionError
    assert N._CODES[2] is SingularMatrixError
    assert N._CODES[3] is ConfigError
    assert N._CODES[4] is SetupError
    assert N._CODES[5] is NativeError


def test_no_device_here_is_reported_not_faked():
    n = C.c_int(-1)
    N.check(N.lib().camg_device_count(C.byref(n)))
    if n.value == 0:
        with pytest.raises(NativeError):
            N.require_device()


def test_host_aggregation_entry_points_without_gpu():
    """The integer aggregation is host C++: callable without a device."""
    import numpy as np

    from paper_1912_09056_b200.aggregation import NodeGraph, aggregate_greedy
    # 1-D chain of 10 nodes
    e = np.array([[i, i + 1] for i in range(9)])
    g = NodeGraph.from_edges(10, e)
    a = aggregate_greedy(g, 1)
    assert a.is_partition()
    assert a.num_aggs == 4  # roots 0,3,6,9-> phase 1 {0,1},{2,3,4},{5,6,7},{8,9}

"""Slot statistics of the fine-level masked mirror (shared value groups): python scripts/slot_stats.py C5 1"""
import sys, ctypes as C, numpy as np
sys.path.insert(0, ".")
from paper_1912_09056_b200 import _native as N
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
g = generate(config_spec(sys.argv[1], int(sys.argv[2])), assemble_K=False)
op = saddle_operator(g, device_K=True)
A = op.merged()
N.call("camg_csr_attach_blocks", A.device, 3, op.n_u)
out = np.zeros(5, dtype=np.int64)
N.call("camg_csr_slot_stats", A.device, out.ctypes.data_as(C.c_void_p))
k, f = C.c_int64(), C.c_int64()
N.call("camg_csr_value_groups", A.device, C.byref(k), C.byref(f))
print("slots", out[0], "uniform", out[1], "linear", out[2], "both", out[3], "uniform+exceptions", out[4], "groups kept/full", k.value, f.value)

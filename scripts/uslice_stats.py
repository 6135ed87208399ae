import sys, ctypes as C
sys.path.insert(0, '.')
from paper_1912_09056_b200 import _native
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
g = generate(config_spec("C5", 1), assemble_K=False)
op = saddle_operator(g, device_K=True)
A = op.merged()
_native.call("camg_csr_attach_blocks", A.device, 3, op.n_u)
c = (C.c_int64 * 5)(); _native.call("camg_csr_uniform_slices", A.device, c)
s = (C.c_int64 * 5)(); _native.call("camg_csr_slot_stats", A.device, s)
k, f = C.c_int64(0), C.c_int64(0); _native.call("camg_csr_value_groups", A.device, C.byref(k), C.byref(f))
print("slices, uniform, pairs, aligned:", tuple(c)); print("slots, uniform, linear, both, kind2:", tuple(s)); print("groups kept/full", k.value, f.value)

"""A/B micro-benchmark of the fine-level merged-operator SpMV formats on C5:
CSR, block SELL-32 with full 3x3 slots, masked slots (CAMG_SELL_MASKED); `ident` =
results bit-identical to the full-block kernel."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1912_09056_b200 import _native as N
from paper_1912_09056_b200.problem import config_spec, generate, saddle_operator
from paper_1912_09056_b200.sparse import empty, ptr, stream_ptr
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = generate(config_spec("C5", scale), assemble_K=False)
op = saddle_operator(g, device_K=True)
A = op.merged()
n = A.num_rows
x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
y = empty(n); ref = None; full = None
def bench(label):
    global ref, full
    for _ in range(3): N.call("camg_spmv", A.device, 1.0, ptr(x), 0.0, ptr(y), stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(20): N.call("camg_spmv", A.device, 1.0, ptr(x), 0.0, ptr(y), stream_ptr())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    b = C.c_double(); N.call("camg_csr_stream_bytes", A.device, C.byref(b))
    csr_model = 12.0 * A.nnz + 4.0 * (n + 1) + 16.0 * n
    if ref is None: ref = y.clone()
    err = float((y - ref).abs().max() / ref.abs().max())
    if label == "sell-full": full = y.clone()
    ident = "" if full is None else f"  ident {bool(torch.equal(y, full))}"
    print(f"{label:14s} {ms:7.3f} ms  format {b.value/1e9:6.2f} GB {b.value/ms/1e6:7.0f} GB/s  csr-model {csr_model/ms/1e6:7.0f} GB/s  maxrel {err:.1e}{ident}", flush=True)
bench("csr")
for mode in ("0", "1"):
    os.environ["CAMG_SELL_MASKED"] = mode
    N.call("camg_csr_attach_blocks", A.device, 3, op.n_u)
    bench("sell-full" if mode == "0" else "sell-masked")


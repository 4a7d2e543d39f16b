"""Timing experiment (trace build: scripts/k1_ab.py build trace SV_STEP_TRACE=1): sv_step phase
times (us after the kernel start, CTA 0 of sequence 0) for a few shapes."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2509_24328_b200 as sv, synth, sv_helpers as H
from paper_2509_24328_b200 import _lib
path = os.path.join(ROOT, "paper_2509_24328_b200", "variants", "libsv_trace.so")
_lib._lib = None
_lib.load(path)
raw = ctypes.CDLL(path)
prof = sv.Profile.from_dict(synth.load_profile())
for (B, k, V, dt) in ((4, 4, 32000, "f32"), (4, 8, 128256, "bf16"), (16, 8, 128256, "bf16")):
    x = synth.make_inputs(B, k, V, dt, seed=1)
    D, C, T, tok = H.to_torch(x)
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    rowptr = torch.arange(B, dtype=torch.int64, device="cuda") * (k + 1)
    for _ in range(3):
        sv.sv_step(D, C, T.reshape(-1, V), rowptr, tok, L, prof)
    torch.cuda.synchronize()
    buf = np.zeros(8, dtype=np.uint64)
    raw.sv_debug_step_trace(buf.ctypes.data_as(ctypes.c_void_p))
    t = (buf[:7].astype(np.float64) - float(buf[0])) / 1e3
    print(B, k, V, dt, "phases A score, B sched, C rows, D decide, E slices, F find ->", np.round(np.diff(t), 2))

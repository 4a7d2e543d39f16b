#!/usr/bin/env python3
"""Timing experiment (trace build of libsv, SV_K1S_TRACE=1): per-chunk event timestamps of K1s.

    python scripts/k1_ab.py build trace SV_K1S_TRACE=1      # here
    python scripts/k1s_trace.py                            # on the GPU
Events per CTA and chunk: 0 load issued, 1 P1 done, 2 P1 published, 3 Lambda ready, 4 P2 done,
5 S published (us since the earliest event)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv, synth
from paper_2509_24328_b200 import _lib
lib_path = os.path.join(ROOT, "paper_2509_24328_b200", "variants", "libsv_trace.so")
_lib._lib = None
lib = _lib.load(lib_path)
raw = ctypes.CDLL(lib_path)
B, k, V = 80, 8, 152064
x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).cuda()
D, C, tok = h(x["D"]), h(x["C"]), torch.from_numpy(x["tok"]).cuda()
prof = sv.Profile.from_dict(synth.load_profile())
ws = sv.new_workspace(B, k, V, torch.bfloat16)
for _ in range(3):
    out = sv.sv_score(D, C, tok, 1.0, 1.0, prof, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros((160, 32, 8), dtype=np.uint64)
assert raw.sv_debug_res_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t = buf.astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)
cs = int(sys.argv[1]) if len(sys.argv) > 1 else 13
for cta in list(range(cs)) + [cs, 2 * cs]:
    print(f"CTA {cta}")
    for n in range(12):
        print("  n=%2d " % n + " ".join("%7.2f" % v for v in t[cta, n, :6]))

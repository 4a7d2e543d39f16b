#!/usr/bin/env python3
"""Per-kernel timeline of one graph step from an SV_EXP_TRACE build (on the GPU):
    python scripts/k1_ab.py build trace SV_EXP_TRACE=1      # here
    python scripts/trace_step.py [B k V dtype]               # there
Each kernel records its earliest CTA start (after griddepcontrol.wait) and its latest warp exit
(%globaltimer); printed relative to the step's first start, averaged over replays (L2 flushed
before each replay for inputs smaller than L2, as bench.py's config points)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402
from paper_2509_24328_b200 import _lib  # noqa: E402

B, k, V, dt = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]) if len(sys.argv) > 4 else (80, 8, 152064, "bf16")
path = os.path.join(ROOT, "paper_2509_24328_b200", "variants", f"libsv_{sys.argv[5] if len(sys.argv) > 5 else 'trace'}.so")
_lib._lib = None
lib = _lib.load(path)
raw = ctypes.CDLL(path)
readers = [getattr(raw, f"sv_debug_trace_{n}") for n in ("score", "sched", "verify") if hasattr(raw, f"sv_debug_trace_{n}")]
names = {0: "K1 ticket", 6: "K1c", 1: "K3", 2: "K4", 3: "K4b", 4: "K5", 5: "K5b", 7: " c0 bulk in", 8: " c0 pass 1",
         9: " c0 sync 1", 10: " c0 pass 2", 11: " c0 sync 2", 12: " c0 epilogue", 13: " K1 P1 tasks (end)",
         14: " K1 P2 tasks (start)"}
dev = torch.device("cuda")
x = synth.make_inputs(B, k, V, dt, seed=0x5EED)
tdt = torch.bfloat16 if dt == "bf16" else torch.float32
conv = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(dev)) if dt == "bf16" \
    else (lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev))
prof = sv.Profile.from_dict(synth.load_profile())
L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device=dev)
gp = sv.GraphPipeline(B, k, V, tdt, prof, L, seed=1, offset0=0)
for d, s in zip((gp.D, gp.C, gp.T), (x["D"], x["C"], x["T"])):
    d.copy_(conv(s))
gp.tok.copy_(torch.from_numpy(x["tok"]).to(dev))
gp.capture()
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
buf = (ctypes.c_ulonglong * 32)()
acc = {}
R = 30
for it in range(R + 3):
    flush.add_(1)
    torch.cuda.synchronize()
    for r in readers:
        r(None)
    gp.replay()
    torch.cuda.synchronize()
    ev = {}
    for r in readers:
        r(buf)
        for slot in range(16):
            s0, s1 = buf[2 * slot], buf[2 * slot + 1]
            if s1 and s0 != 2 ** 64 - 1:
                ev[slot] = (s0, s1)
            elif s1:  # end-only marker
                ev[slot] = (s1, s1)
            elif s0 != 2 ** 64 - 1:  # start-only marker
                ev[slot] = (s0, s0)
    t0 = min(v[0] for v in ev.values())
    if it >= 3:
        for slot, (a, b) in ev.items():
            acc.setdefault(slot, []).append(((a - t0) / 1e3, (b - t0) / 1e3))
print(f"B={B} k={k} V={V} {dt}: kernel start / end (us from the step's first kernel start), mean of {R} replays")
for slot in sorted(acc, key=lambda s: np.mean([v[0] for v in acc[s]])):
    st = np.mean([v[0] for v in acc[slot]]); en = np.mean([v[1] for v in acc[slot]])
    print(f"  {names.get(slot, slot):10s} start {st:7.1f}  end {en:7.1f}  span {en - st:6.1f}")

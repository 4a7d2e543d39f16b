import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch, synth
import paper_2509_24328_b200 as sv
from paper_2509_24328_b200 import _lib
name = sys.argv[1]; B = int(sys.argv[2])
_lib._lib = None
_lib.load(os.path.join(os.path.dirname(sv.__file__), "variants", f"libsv_{name}.so"))
x = synth.make_inputs(B, 8, 152064, "bf16", seed=1)
D = torch.from_numpy(x["D"]).view(torch.bfloat16).cuda(); C = torch.from_numpy(x["C"]).view(torch.bfloat16).cuda()
tok = torch.from_numpy(x["tok"]).cuda()
prof = sv.Profile.from_dict(synth.load_profile())
o = sv.sv_score(D, C, tok, 1.0, 1.0, prof)
torch.cuda.synchronize()
print(name, B, "ok", o["S"][0, :3].tolist())

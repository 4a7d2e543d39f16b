"""NEXT-4: the GPU profile builder + information-gain report against the CPU
form in oracle/profile.py (itself pinned by tests/test_oracle_pins.py: S L281 edges, S L290 /
L296 fallbacks).  Edges are order statistics of the same fp32 samples, so they must agree
exactly; counts exactly; cell means (GPU fixed-point 2^-32 sums) and entropies to 1e-9."""
import numpy as np
import pytest

import synth
import sv_helpers as H
from oracle import profile as oprof

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2509_24328_b200 as sv
    sv.load_library()
    return sv


def _check(sv, S, A, X, ns, na, xb=10):
    g = sv.sv_profile_build(torch.as_tensor(S, device="cuda"), torch.as_tensor(A, device="cuda"),
                            torch.as_tensor(X, device="cuda"), ns, na, xb)
    S64, A64, X64 = (np.asarray(v, dtype=np.float32).astype(np.float64) for v in (S, A, X))
    ref = oprof.build_profile(S64, A64, X64, ns, na)
    assert np.array_equal(g["s_edges"].cpu().numpy().astype(np.float64), np.asarray(ref["s_edges"]))
    assert np.array_equal(g["a_edges"].cpu().numpy().astype(np.float64), np.asarray(ref["a_edges"]))
    assert np.array_equal(g["counts"].cpu().numpy(), np.asarray(ref["counts"]))
    assert np.allclose(g["cells"].cpu().numpy(), np.asarray(ref["cells"]), rtol=1e-9, atol=1e-9)
    sb = np.array([oprof.bin_of(ref["s_edges"], v) for v in S64])
    ab = np.array([oprof.bin_of(ref["a_edges"], v) for v in A64])
    ig = oprof.info_gain(X64, sb, ab, xb)
    for key, v in ig.items():
        assert abs(g["info"][key] - v) <= 1e-9 * max(1.0, abs(v)), (key, g["info"][key], v)
    return g


def test_profile_from_gpu_pipeline_records(sv):
    """Records of a GPU profiling run: S, A from sv_score, X = accept_ratio with gamma = k."""
    B, k, V = 64, 8, 32000
    x = synth.make_inputs(B, k, V, "bf16", seed=2718)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    sc = sv.sv_score(D, C, tok, 1.0, 1.0, prof)
    gam = torch.full((B,), k, dtype=torch.int32, device="cuda")
    ver = sv.sd_verify(D, T, tok, gam, sc["draft_m"], sc["draft_l"], sc["draft_ptok"], 1.0, 1.0, 3, 0, 0)
    S, A, X = (t.reshape(-1).cpu().numpy() for t in (sc["S"], sc["A"], ver["accept_ratio"]))
    g = _check(sv, S, A, X, 20, 15)
    assert g["n_s"] == 20 and g["counts"].sum().item() == B * k


@pytest.mark.parametrize("N,ns,na", [(1, 5, 5), (7, 4, 3), (20000, 20, 15), (4096, 64, 64)])
def test_profile_ties_and_sizes(sv, N, ns, na):
    rng = np.random.default_rng(N + ns)
    S = np.round(rng.random(N), 2).astype(np.float32)       # many duplicates: collapsed edges
    A = np.minimum(1.0, rng.random(N) * 1.3).astype(np.float32)  # mass at A = 1
    X = rng.random(N).astype(np.float32)
    _check(sv, S, A, X, ns, na)

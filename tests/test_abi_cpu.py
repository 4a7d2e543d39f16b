"""CPU checks of the boundary (-m "not gpu"): libsv.so builds for sm_100a, loads, and exports
every symbol include/sv.h declares; host-side argument validation rejects bad calls
without launching anything (no GPU needed for those paths)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2509_24328_b200 import _lib, build
    build.build()
    return _lib.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sv.h")).read()
    return re.findall(r"SV_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)


def test_header_declares_the_abi():
    names = declared_symbols()
    for want in ("sv_score", "sv_schedule", "sd_verify", "sv_workspace_bytes", "sv_status_string"):
        assert want in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2509_24328_b200", "libsv.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    assert set(declared_symbols()) <= exported


def test_sm100a_cubin_embedded():
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2509_24328_b200", "libsv.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_validation_without_gpu(lib):
    from paper_2509_24328_b200 import _lib
    assert lib.sv_status_string(0) == b"ok"
    assert lib.sv_workspace_bytes(80, 8, 152064, _lib.SV_BF16) > 0
    assert lib.sv_workspace_bytes(80, 17, 152064, _lib.SV_BF16) == 0
    L = _lib.SvLogits(0, _lib.SV_BF16, 0, 0, 0)
    # NULL tensor pointer -> invalid argument, nothing launched
    st = lib.sv_score(ctypes.byref(L), ctypes.byref(L), None, 1, 1, 100, 1.0, 1.0, None,
                      None, None, None, None, None, None, None, None, None, 0, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    st = lib.sv_schedule(None, 1, 1, None, 0, 0, 1, None, None, None, None, None, 0, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    # k out of range
    st = lib.sv_schedule(ctypes.c_void_p(16), 1, 17, ctypes.c_void_p(16), 20, 0, 1, ctypes.c_void_p(16),
                         None, None, None, None, 0, None)
    assert st == _lib.SV_ERR_INVALID_ARG


def test_library_configured_by_arguments_only():
    # SURVEY §5 / include/sv.h determinism promise: no environment variables, no tuning globals
    csrc = os.path.join(ROOT, "paper_2509_24328_b200", "csrc")
    for f in os.listdir(csrc):
        with open(os.path.join(csrc, f)) as fh:
            src = fh.read()
        assert "getenv" not in src and "environ" not in src, f
    with open(os.path.join(ROOT, "paper_2509_24328_b200", "__init__.py")) as fh:
        assert "os.environ" not in fh.read()


def test_product_has_no_cpu_fallback():
    # the package never imports the oracle, and compute calls refuse CPU tensors
    import torch

    import paper_2509_24328_b200 as sv
    pkg = os.path.join(ROOT, "paper_2509_24328_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, fn)).read().replace("fp64 oracle", "")
    with pytest.raises(sv.SvError):
        sv.sv_score(torch.zeros(1, 1, 8), torch.zeros(1, 1, 8), torch.zeros(1, 1, dtype=torch.int32))


def test_wrappers_enforce_element_types_and_extents():
    """The C ABI takes untyped pointers, so the binding checks what the kernels assume:
    int32 tokens / gamma, T with k + 1 rows, C shaped like D, fp32 normalisers, int64 row pointers.
    These checks run before any CUDA call (no GPU needed)."""
    import torch

    import paper_2509_24328_b200 as sv
    D = torch.zeros(2, 3, 16)
    ok_tok = torch.zeros(2, 3, dtype=torch.int32)
    with pytest.raises(sv.SvError, match="int32"):
        sv.sv_score(D, D, torch.zeros(2, 3, dtype=torch.int64))
    with pytest.raises(sv.SvError, match="shape"):
        sv.sv_score(D, torch.zeros(2, 3, 15), ok_tok)
    with pytest.raises(sv.SvError, match="dtype"):
        sv.sv_score(D, D.double(), ok_tok)
    f32 = torch.zeros(2, 3)
    g = torch.zeros(2, dtype=torch.int32)
    with pytest.raises(sv.SvError, match="shape"):  # T with k rows instead of k + 1
        sv.sd_verify(D, torch.zeros(2, 3, 16), ok_tok, g, f32, f32, f32)
    T = torch.zeros(2, 4, 16)
    with pytest.raises(sv.SvError, match="int32"):
        sv.sd_verify(D, T, ok_tok, g.long(), f32, f32, f32)
    with pytest.raises(sv.SvError, match="float32"):
        sv.sd_verify(D, T, ok_tok, g, f32.double(), f32, f32)
    with pytest.raises(sv.SvError, match="int64"):
        sv.sd_verify_ragged(D, torch.zeros(8, 16), torch.zeros(2, dtype=torch.int32), ok_tok, g, f32, f32, f32)
    with pytest.raises(sv.SvError, match="float32"):
        sv.sv_schedule(torch.zeros(2, 3, dtype=torch.float64), torch.zeros(5, dtype=torch.float64))
    with pytest.raises(sv.SvError, match="out"):  # a caller-provided output of the wrong type
        sv.sv_score(D, D, ok_tok, out={"S": torch.zeros(2, 3, dtype=torch.float64)})


def test_host_validation_of_the_widened_abi(lib):
    """NEXT-2/3/4 and vocab-sharded entry points reject bad arguments on the host, before any
    CUDA call (so this runs without a GPU)."""
    from paper_2509_24328_b200 import _lib
    P = ctypes.c_void_p(16)  # a non-NULL dummy: validation fails before any dereference
    L = _lib.SvLogits(16, _lib.SV_BF16, 0, 0, 0)
    # filters: top_k outside [0, 32] unsupported, top_p outside (0, 1] or no filter at all invalid
    for top_k, top_p, want in ((-1, 0.9, _lib.SV_ERR_UNSUPPORTED), (33, 0.9, _lib.SV_ERR_UNSUPPORTED),
                               (0, 1.0, _lib.SV_ERR_INVALID_ARG), (20, 0.0, _lib.SV_ERR_INVALID_ARG),
                               (20, 1.5, _lib.SV_ERR_INVALID_ARG)):
        f = _lib.SvFilter(top_k, top_p)
        st = lib.sv_score_filtered(ctypes.byref(L), ctypes.byref(L), P, 2, 2, 100, 1.0, 1.0, ctypes.byref(f), None,
                                   None, None, None, None, None, None, P, 1 << 20, None)
        assert st == want, (top_k, top_p, st)
    assert lib.sv_filter_workspace_bytes(80, 8) > 0 and lib.sv_filter_workspace_bytes(80, 17) == 0
    # filtered verify: the optional draft logits must match the target's dtype; gamma is required
    f = _lib.SvFilter(0, 0.9)
    Lf = _lib.SvLogits(16, _lib.SV_F32, 0, 0, 0)
    st = lib.sd_verify_filtered(ctypes.byref(L), ctypes.byref(Lf), P, P, 2, 2, 100, 1.0, ctypes.byref(f), 0, 0, 0,
                                P, P, None, None, None, P, 1 << 20, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    st = lib.sd_verify_filtered(ctypes.byref(L), None, P, None, 2, 2, 100, 1.0, ctypes.byref(f), 0, 0, 0,
                                P, P, None, None, None, P, 1 << 20, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    # ragged verify: missing row pointers / short row stride
    st = lib.sd_verify_ragged(ctypes.byref(L), P, 99, P, P, P, P, P, P, 2, 2, 100, 1.0, 1.0, 0, 0, None, 0,
                              P, P, None, None, None, P, 1 << 30, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    st = lib.sd_verify_ragged(ctypes.byref(L), P, 100, None, P, P, P, P, P, 2, 2, 100, 1.0, 1.0, 0, 0, None, 0,
                              P, P, None, None, None, P, 1 << 30, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    # profile builder: bins beyond 64, empty input, small workspace
    assert lib.sv_profile_workspace_bytes(100, 65, 10, 10) == 0
    assert lib.sv_profile_workspace_bytes(0, 20, 15, 10) == 0
    st = lib.sv_profile_build(P, P, P, 100, 20, 15, 10, P, P, P, P, P, None, P, 16, None)
    assert st == _lib.SV_ERR_WORKSPACE
    # vocab-sharded: G < 1, rank out of range (any G * chunks merges: no lane limit)
    assert lib.sv_shard_xch_bytes(0, 80, 8, 19008, _lib.SV_BF16) > 0
    assert lib.sv_shard_xch_bytes(4, 80, 8, 19008, _lib.SV_BF16) == 0
    st = lib.sv_shard_score_p2(ctypes.byref(L), ctypes.byref(L), P, 2, 2, 100, 1.0, 1.0, P, 0, P, None)
    assert st == _lib.SV_ERR_INVALID_ARG
    st = lib.sv_shard_verify_finish(ctypes.byref(L), ctypes.byref(L), 2, 2, 100, 0, 1.0, 1.0, P, 2, 2, P, None,
                                    None, P, 1 << 30, None)
    assert st == _lib.SV_ERR_INVALID_ARG

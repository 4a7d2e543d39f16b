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
    # bf16 V=152064 -> cluster of 8 CTAs, 76 KB of (D, C) per CTA
    assert lib.sv_cluster_size(152064, _lib.SV_BF16) == 8
    assert lib.sv_cluster_size(32000, _lib.SV_F32) == 4
    assert lib.sv_cluster_size(10_000_000, _lib.SV_F32) == 0
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

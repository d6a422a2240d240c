"""The C-ABI library loads on a CPU-only host and exports every symbol the
public header declares; the ctypes binding covers all of them. No compute."""
import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pint_abi.h")
LIB = os.path.join(ROOT, "paper_2110_10762_b200", "libpint_b200.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pint_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_hot_path_entry_points():
    names = declared()
    for must in ("pint_ctx_create", "pint_op_create", "pint_op_apply_batch", "pint_correct",
                 "pint_coarse_init", "pint_sync_sweep"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build with python -m paper_2110_10762_b200.build"
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB]).decode()
    exported = set(re.findall(r"\bT (pint_[a-z_0-9]+)$", out, flags=re.M))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_is_complete():
    from paper_2110_10762_b200 import _native
    lib = _native.load_library()
    assert lib.pint_abi_version() == 1
    assert set(declared()) <= set(_native.SIGNATURES)
    # struct layout matches the header (8-byte aligned, no implicit padding)
    assert ctypes.sizeof(_native.OpDesc) == 4 * 4 + 8 * 3 + 8 * 3 + 8 * 4 + 8 * 2 + 4 * 2
    assert ctypes.sizeof(_native.OpInfo) == 8 * 2 + 4 * 6 + 8 * 4 + 4 * 4


def test_library_is_sm100a_code():
    out = subprocess.check_output(["cuobjdump", "--list-elf", LIB]).decode()
    assert "sm_100a" in out


def test_no_device_reports_a_clean_error():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2110_10762_b200 import _native
    lib = _native.load_library()
    h = ctypes.c_void_p()
    rc = lib.pint_ctx_create(0, ctypes.byref(h))
    assert rc != 0
    assert lib.pint_last_error(None)

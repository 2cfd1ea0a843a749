"""CPU-side checks of the boundary: libfairserve.so builds for sm_100a, loads, and
exports every function include/fairserve.h declares (no compute without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fairserve.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2411_15997_b200 import build
    return build.build()


def test_header_declares_the_five_calls():
    names = _declared()
    for f in ("fs_build_app_profiles", "fs_act_throttle", "fs_wsc_step", "fs_wsc_replay", "fs_sweep"):
        assert f in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fs_\w+)", out))
    assert set(_declared()) <= exported


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_strerror_without_gpu(libpath):
    lib = ctypes.CDLL(libpath)
    lib.fs_strerror.restype = ctypes.c_char_p
    assert lib.fs_strerror(-3) == b"FS_E_ORDER"
    h = ctypes.c_void_p()
    # no GPU here: context creation must fail loudly (no CPU fallback)
    import torch
    if not torch.cuda.is_available():
        assert lib.fs_ctx_create(0, None, ctypes.byref(h)) == -8


def test_binding_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_15997_b200 import fairserve as F
    with pytest.raises(Exception):
        F.Context(0)

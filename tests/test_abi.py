"""The C-ABI library builds, loads and exports every symbol include/twopass.h declares
(-m "not gpu": no compute calls, no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "twopass.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(\w+)\s*\(", src, flags=re.M)
    return sorted({n for n in names if n not in ("if", "sizeof")})


@pytest.fixture(scope="module")
def so():
    from paper_2001_04438_b200 import build
    return build.build()


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ["softmax_f32", "softmax_bf16_f32", "softmax3_recompute_f32", "softmax3_reload_f32",
              "softmax_f32_partial", "softmax_f32_finish", "softmax_workspace_bytes", "softmax_f32_host"]:
        assert n in names


def test_library_exports_every_declared_symbol(so):
    lib = ctypes.CDLL(so)
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_exports_are_c_linkage(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for n in declared_functions():
        assert n in syms, f"{n} not exported unmangled"


def test_library_is_built_for_sm100a(so):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_only_entry_points_without_gpu(so):
    lib = ctypes.CDLL(so)
    lib.softmax_workspace_bytes.restype = ctypes.c_size_t
    lib.softmax_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64]
    assert lib.softmax_workspace_bytes(0, 5) == 0
    assert lib.softmax_workspace_bytes(256, 800000) > 256 * 49 * 8
    lib.softmax_status_str.restype = ctypes.c_char_p
    assert lib.softmax_status_str(1) == b"invalid argument"
    # argument errors are decided on the host, before any CUDA call
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.tp_debug_op.argtypes = [ctypes.c_int, vp, vp, vp, vp, i64, vp]
    dummy = ctypes.c_void_p(16)
    assert lib.tp_debug_op(9, dummy, None, dummy, dummy, 32, None) == 1   # unknown op
    assert lib.tp_debug_op(8, dummy, None, dummy, dummy, 31, None) == 1   # warp value: whole warps only
    assert lib.tp_debug_op(0, None, None, dummy, dummy, 4, None) == 1     # missing input


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    import paper_2001_04438_b200 as tp
    monkeypatch.setattr(tp, "_SO", str(tmp_path / "missing.so"))
    monkeypatch.setattr(tp, "_lib", None)
    with pytest.raises(ImportError):
        tp.lib()

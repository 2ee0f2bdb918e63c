"""CPU checks of the C-ABI boundary: libactc.so builds for sm_100a, loads
without a GPU, and exports every entry point include/actc.h declares."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2111_09562_b200", "libactc.so")
HDR = os.path.join(ROOT, "include", "actc.h")


def _ensure_built():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_2111_09562_b200", "csrc"), "-j8"])


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"\b(actc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("actc_compress_plan", "actc_compress_encode", "actc_decompress", "actc_lbar", "actc_mean_abs"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    _ensure_built()
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2111_09562_b200 import _lib

    assert sorted(_lib.EXPORTED_SYMBOLS) == declared_symbols()


def test_library_is_sm100a():
    _ensure_built()
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_version_call_without_gpu():
    _ensure_built()
    from paper_2111_09562_b200 import _lib

    assert _lib.lib().actc_version() == 1

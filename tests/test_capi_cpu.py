"""C-ABI library loads and exports every symbol include/exa.h declares (CPU)."""

import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "exa.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(exa_\w+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_2510_12897_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(syms)


def test_struct_layouts_match_header():
    from paper_2510_12897_b200 import _lib

    assert ctypes.sizeof(_lib.SegDesc) == 16
    # 16+16 int64 offsets, 3 int64, 16 int32 voff, 8 int32 scalars, 3 int64
    assert ctypes.sizeof(_lib.TermDesc) == 8 * 32 + 8 * 3 + 4 * 16 + 4 * 8 + 8 * 3


def test_nvrtc_available_and_compiles_sm100a():
    from paper_2510_12897_b200 import _lib

    assert _lib.nvrtc_version().startswith("12.")
    cub = _lib.jit_compile('extern "C" __global__ void k(double* a) { a[threadIdx.x] *= 2.0; }',
                           ("-arch=sm_100a",))
    assert cub[:4] == b"\x7fELF"

"""The C-ABI library loads on CPU and exports every symbol include/mmk.h declares (no compute
calls without a GPU), and the host-side error mapping follows the reference's classes."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "mmk.h"
LIB = ROOT / "paper_2502_00937_b200" / "libmmk.so"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(mmk_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("mmk_tile_plan", "mmk_preprocess", "mmk_gemm_bf16", "mmk_layernorm", "mmk_attention_varlen_bf16",
              "mmk_embed_tokens", "mmk_pack_mllama", "mmk_pack_drop_cls", "mmk_version", "mmk_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "libmmk.so not built (run __graft_entry__.build())"
    lib = ctypes.CDLL(str(LIB))
    for s in declared_symbols():
        assert hasattr(lib, s), s
    from paper_2502_00937_b200 import _lib
    assert set(_lib.SIGNATURES) >= set(declared_symbols())
    assert _lib.version().startswith("mmk")


def test_argument_errors_map_to_reference_exceptions():
    # shape validation happens before any device work, so it is callable without a GPU
    from paper_2502_00937_b200 import _lib
    from paper_2502_00937_b200.core import SpecError
    rc = _lib.lib.mmk_tile_plan(None, None, -1, 560, 1601, 4, 0, 0, None, None, None, None, None, None, None)
    with pytest.raises(SpecError):
        _lib.check(rc)
    rc = _lib.lib.mmk_attention_varlen_bf16(None, None, None, 1, 16, 16, 16, 72, 0.1, None, None)
    with pytest.raises(_lib.ProfileError):
        _lib.check(rc)
    rc = _lib.lib.mmk_gemm_bf16(None, 64, None, 64, 128, 100, 64, 0, None, None, 100, 1.0, None, 0, None)
    with pytest.raises(_lib.ProfileError):
        _lib.check(rc)


def test_header_is_plain_c_and_links():
    """include/mmk.h compiles as C11 and a C client links against libmmk.so (no GPU needed)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None or not LIB.exists():
        pytest.skip("gcc or libmmk.so missing")
    ex = Path(__file__).resolve().parent.parent / "examples"
    r = subprocess.run(["make", "-C", str(ex), "-s", "-B"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    (ex / "c_abi_demo").unlink()

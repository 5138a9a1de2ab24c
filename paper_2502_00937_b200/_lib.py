"""ctypes binding of libmmk.so — the C-ABI boundary (include/mmk.h).

There is no fallback: if the library is missing the import fails loudly.  Status codes map to
the reference's exception classes: MMK_ERR_ARG -> SpecError (core.py:26-27),
MMK_ERR_UNSUPPORTED -> ProfileError (profiles.py:23-24), MMK_ERR_CUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .core import SpecError
from .profiles import ProfileError

LIB_PATH = Path(os.environ.get("MMK_LIB", Path(__file__).resolve().parent / "libmmk.so"))


class MMKError(RuntimeError):
    """CUDA failure inside libmmk."""


_V = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F = ctypes.c_float

SIGNATURES = {
    "mmk_version": ([], ctypes.c_char_p),
    "mmk_last_error": ([], ctypes.c_char_p),
    "mmk_tile_plan": ([_V, _V, _I32, _I32, _I32, _I32, _I32, _I32, _V, _V, _V, _V, _V, _V, _V], _I32),
    "mmk_tile_index": ([_V, _I32, _V, _V, _V], _I32),
    "mmk_seq_offsets": ([_V, _I32, _I32, _V, _V], _I32),
    "mmk_preprocess": ([_V, _V, _I32, _V, _V, _V, _V, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _V, _V, _V, _V],
                       _I32),
    "mmk_gemm_bf16": ([_V, _I64, _V, _I64, _I32, _I32, _I32, _I32, _V, _V, _I64, _F, _V, _I64, _V], _I32),
    "mmk_gemm_bf16_ln": ([_V, _I64, _V, _I64, _I32, _I32, _I32, _I32, _V, _V, _I64, _F, _V, _I64, _V, _V, _V, _V],
                         _I32),
    "mmk_ln_stats_finalize": ([_V, _I32, _I32, _F, _I32, _V, _V], _I32),
    "mmk_layernorm_bf16": ([_V, _V, _I32, _I32, _V, _V, _F, _V], _I32),
    "mmk_qk_rmsnorm": ([_V, _I32, _I32, _I64, _V, _V, _F, _V], _I32),
    "mmk_pack_pixel_shuffle": ([_V, _I32, _I32, _I32, _I32, _I32, _V, _V], _I32),
    "mmk_layernorm": ([_V, _V, _I32, _I32, _I32, _V, _V, _F, _V, _V, _V, _V, _I32, _I32, _V], _I32),
    "mmk_attention_workspace_size": ([], _I64),
    "mmk_attention_varlen_bf16": ([_V, _V, _V, _I32, _I32, _I32, _I32, _I32, _F, _V, _V], _I32),
    "mmk_embed_tokens": ([_V, _V, _V, _V, _I32, _I32, _I32, _V, _V, _F, _V, _F, _V, _F, _I32, _V, _V, _F, _V, _V],
                         _I32),
    "mmk_pack_mllama": ([_V, _V, _I32, _I32, _I32, _V, _V], _I32),
    "mmk_pack_mllama_peer": ([_V, _V, _I32, _I32, _I32, _V, _V], _I32),
    "mmk_pack_drop_cls": ([_V, _I32, _I32, _I32, _I32, _I32, _V, _V], _I32),
    "mmk_checksum_bf16": ([_V, _I64, _V, _V], _I32),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"libmmk.so not found at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback for the image path)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.mmk_last_error().decode()
    if rc == 1:
        raise SpecError(msg)
    if rc == 2:
        raise ProfileError(msg)
    raise MMKError(msg)


def version() -> str:
    return lib.mmk_version().decode()

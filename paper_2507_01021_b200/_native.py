"""ctypes binding of the C ABI in include/dictamux_b200.h.

The library is built in-tree (paper_2507_01021_b200/_lib/libdictamux_b200.so,
see build.py). There is no CPU fallback: if the library or a CUDA device is
missing, every call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libdictamux_b200.so"
# (A/B experiments: DM_LIB points at another build of the same sources)
LIB_PATH = Path(os.environ.get("DM_LIB", LIB_PATH))

EXPORTS = (
    "dm_last_error", "dm_version", "dm_fill_normal_bf16", "dm_logmel", "dm_logmel_operand",
    "dm_gemm_bf16_f32", "dm_whisper_create", "dm_whisper_destroy",
    "dm_whisper_encode", "dm_whisper_encode_lengths", "dm_whisper_admit", "dm_whisper_release", "dm_whisper_set_prompt",
    "dm_whisper_set_active", "dm_whisper_step", "dm_whisper_read", "dm_whisper_read_async",
    "dm_whisper_debug", "dm_whisper_stats", "dm_whisper_time_kernel",
    "dm_ctc_create", "dm_ctc_destroy", "dm_ctc_transcribe", "dm_ctc_read", "dm_ctc_debug",
    "dm_vad_classify",
)


class DmError(RuntimeError):
    """A C-ABI call returned a non-zero status (message from dm_last_error)."""


class WhisperConfigC(C.Structure):
    _fields_ = [("d_model", C.c_int), ("enc_layers", C.c_int),
                ("dec_layers", C.c_int), ("heads", C.c_int), ("ffn", C.c_int),
                ("n_mels", C.c_int), ("vocab", C.c_int), ("eot", C.c_int),
                ("prompt", C.c_int * 8), ("prompt_len", C.c_int),
                ("max_slots", C.c_int), ("max_encode_batch", C.c_int),
                ("num_pages", C.c_int), ("decode_groups", C.c_int),
                ("persistent_decode", C.c_int), ("fuse_ln", C.c_int)]


class CtcConfigC(C.Structure):
    _fields_ = [("hidden", C.c_int), ("layers", C.c_int), ("heads", C.c_int), ("ffn", C.c_int),
                ("vocab", C.c_int), ("max_batch", C.c_int), ("max_samples", C.c_int)]


_lib = None
_lock = threading.Lock()
P = C.c_void_p


def load(build_if_missing: bool = False):
    """Load (and optionally build) the shared library; raises if unavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if not build_if_missing:
                raise DmError(f"native library missing: {LIB_PATH} "
                              "(run `python -m paper_2507_01021_b200.build`)")
            from .build import build
            build()
        lib = C.CDLL(str(LIB_PATH))
        for name in EXPORTS:
            if not hasattr(lib, name):
                raise DmError(f"{LIB_PATH} does not export {name}")
        lib.dm_last_error.restype = C.c_char_p
        lib.dm_version.restype = C.c_int
        sig = {
            "dm_fill_normal_bf16": [P, C.c_uint64, C.c_uint64, C.c_float, C.c_float, P],
            "dm_logmel": [P, P, P, C.c_int, C.c_int, P, P],
            "dm_logmel_operand": [P, P, P, C.c_int, C.c_int, P, P, P],
            "dm_gemm_bf16_f32": [P, P, P, P, C.c_int, C.c_int, C.c_int, P],
            "dm_whisper_create": [C.POINTER(WhisperConfigC), P, P, C.c_int,
                                  C.POINTER(C.c_void_p)],
            "dm_whisper_destroy": [P],
            "dm_whisper_encode": [P, P, P, P, C.c_int, P, P],
            "dm_whisper_encode_lengths": [P, P, P, P, P, C.c_int, P, P],
            "dm_whisper_admit": [P, P, P, C.c_int, P],
            "dm_whisper_release": [P, P, C.c_int],
            "dm_whisper_set_prompt": [P, P, C.c_int, P],
            "dm_whisper_set_active": [P, P, C.c_int, P],
            "dm_whisper_step": [P, C.c_int, P],
            "dm_whisper_read": [P, P, P, P, P],
            "dm_whisper_read_async": [P, P, P, P, P],
            "dm_whisper_debug": [P, C.c_int, P, C.c_size_t, P],
            "dm_whisper_stats": [P, P, C.c_int],
            "dm_whisper_time_kernel": [P, C.c_int, C.c_int, C.c_int, P, P],
            "dm_ctc_create": [C.POINTER(CtcConfigC), P, P, C.c_int, C.POINTER(C.c_void_p)],
            "dm_ctc_destroy": [P],
            "dm_ctc_transcribe": [P, P, P, P, C.c_int, P],
            "dm_ctc_read": [P, P, P, P, P],
            "dm_ctc_debug": [P, C.c_int, P, C.c_size_t, P],
            "dm_vad_classify": [P, P, P, C.c_int, C.c_double, P, P],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.dm_last_error().decode(errors="replace") if _lib else "?"
        raise DmError(f"dictamux_b200 error {rc}: {msg}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args))

"""ctypes binding of libhs.so (the C ABI declared in include/hs.h).

The product path has no fallback: if the shared library is missing or no
sm_100 device is visible, calls raise instead of computing anything on the
CPU.  Status codes map to the reference's exception types
(pkg/src/hybridserve/errors.py).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, IntegrityFault, ScenarioError

_LIB_PATH = Path(__file__).resolve().parent / "libhs.so"

HS_OK, HS_E_CONFIG, HS_E_INTEGRITY, HS_E_CAPACITY, HS_E_CUDA = 0, 1, 2, 3, 4
PAGE_TOKENS = 64

_vp, _i, _f, _fp, _ip = C.c_void_p, C.c_int, C.c_float, C.c_void_p, C.c_void_p

# name -> argtypes (all return int)
_SIGNATURES: dict[str, list] = {
    "hs_last_error": [C.c_char_p, _i],
    "hs_device_ok": [],
    "hs_op_gemm_bf16": [_vp, _i, _i, _vp, _i, _i, _fp, _i, C.POINTER(C.c_int), _vp],
    "hs_op_splitk_reduce": [_fp, _i, _i, _i, _fp, _vp],
    "hs_op_gemm_bf16_pair": [_vp, _i, _i, _vp, _i, _i, _fp, _i, C.POINTER(C.c_int), _vp],
    "hs_op_relayout_blocked": [_vp, _vp, _i, _i, _vp],
    "hs_op_gemm_bf16_blocked": [_vp, _i, _i, _vp, _i, _i, _fp, _i, C.POINTER(C.c_int), _vp],
    "hs_op_decode_attention": [_vp, _i, _i, _i, _i, _i, _vp, _i, _i, _ip, _i, _ip, _i, _fp, _fp,
                               _vp],
    "hs_op_decode_attention_fused": [_vp, _i, _i, _i, _i, _i, _vp, _i, _i, _ip, _i, _ip, _i, _i,
                                     _ip, _fp, _fp, _ip, _vp, _i, _vp],
    "hs_op_decode_combine": [_fp, _fp, _ip, _i, _i, _i, _i, _vp, _i, _fp, _vp],
    "hs_op_prefill_attention": [_vp, _i, _i, _i, _i, _i, _vp, _i, _i, _ip, _i, _ip, _i, _vp, _i,
                                _vp],
    "hs_op_embed": [_ip, _i, _vp, _i, _fp, _vp],
    "hs_op_rmsnorm": [_fp, _i, _i, _fp, _f, _vp, _i, _vp],
    "hs_op_residual_add_norm": [_fp, _i, _i, _i, _fp, _fp, _f, _vp, _i, _vp],
    "hs_op_qkv_rope_scatter": [_fp, _i, _i, _i, _i, _i, _fp, _fp, _ip, _ip, _ip, _vp, _i, _vp, _i,
                               _i, _i, _ip, _i, _vp, _i, _vp],
    "hs_op_silu_mul": [_fp, _i, _i, _i, _vp, _i, _vp],
    "hs_op_argmax": [_fp, _i, _i, _i, _ip, _fp, _vp],
    "hs_op_lse_merge": [_vp, _fp, _i, _i, _i, _i, _i, _i, _vp, _i, _vp],
    "hs_host_attention": [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _fp, _i],
    # a remote CPU host process (cpu_host.py): model cfg, bind address, port, threads, max slots
    "hs_cpu_host_serve": [_vp, C.c_char_p, _i, _i, _i],
}

_lib = None


class HsError(RuntimeError):
    """A CUDA-side failure inside libhs (HS_E_CUDA)."""


def lib_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Load libhs.so once; raise if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise HsError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (the serving step has no CPU fallback)"
        )
    lib = C.CDLL(str(_LIB_PATH))
    lib.hs_version.restype = C.c_char_p
    lib.hs_version.argtypes = []
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    _lib = lib
    return lib


# entry points bound with non-int return types or custom argtypes elsewhere
_SPECIAL = ["hs_version", "hs_stream", "hs_cpu_busy_seconds", "hs_wall_seconds",
            "hs_launch_count", "hs_profile", "hs_profile_read", "hs_probe_dense",
            "hs_probe_decode", "hs_probe_prefill", "hs_probe_gemm", "hs_probe_dense_mode",
            "hs_probe_gemm_stream", "hs_probe_pcie", "hs_tp_export", "hs_tp_open"]


def exported_symbols() -> list[str]:
    from . import runtime  # noqa: F401  (registers the step-level signatures)

    return sorted(set(_SPECIAL) | set(_SIGNATURES))


def last_error() -> str:
    buf = C.create_string_buffer(512)
    load().hs_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = "libhs", request_id=None, layer=None) -> None:
    if rc == HS_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == HS_E_CONFIG:
        raise ConfigError(msg)
    if rc == HS_E_INTEGRITY:
        raise IntegrityFault(msg, request_id, layer)
    if rc == HS_E_CAPACITY:
        raise ScenarioError(msg)
    raise HsError(msg)


def call(name: str, *args, what: str | None = None) -> None:
    check(getattr(load(), name)(*args), what or name)


def require_device() -> None:
    """Fail loudly unless an sm_100 device is visible to libhs."""
    if os.environ.get("HS_SKIP_DEVICE_CHECK"):
        return
    if not load().hs_device_ok():
        raise HsError("libhs needs a CUDA device of compute capability 10.x (B200)")

"""ctypes binding of ``libastraea_b200.so`` (C ABI: include/astraea_b200.h).

This is the only place Python touches the native library. There is no CPU
fallback: if the library is missing or no CUDA device is present, every
device entry point raises, loudly. Torch is used for device memory, pinned
host memory and streams only; the arithmetic happens in the sm_100a
kernels behind these calls.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path



class DeviceError(RuntimeError):
    """The native CUDA library returned a non-zero status, or it / the
    sm_100 device is missing (there is no CPU fallback)."""

LIB_PATH = Path(os.environ.get("ASTRAEA_LIB", Path(__file__).resolve().parent.parent / "lib" / "libastraea_b200.so"))

SWAP_KERNEL = 0
SWAP_DMA = 1
SWAP_STAGED = 2
EPI_NONE = 0
EPI_RESIDUAL = 1


class KvGeometry(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("block_tokens", ctypes.c_int32),
        ("num_blocks", ctypes.c_int32),
    ]


class Epilogue(ctypes.Structure):
    """astraea_epilogue (include/astraea_b200.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("residual_dev", ctypes.c_void_p),
        ("ssq_out_dev", ctypes.c_void_p),
        ("ssq_in_dev", ctypes.c_void_p),
        ("ssq_in_parts", ctypes.c_int32),
        ("rms_dim", ctypes.c_int32),
        ("rms_eps", ctypes.c_float),
        ("pool_dev", ctypes.c_void_p),
        ("geo", KvGeometry),
        ("layer", ctypes.c_int32),
        ("num_q_heads", ctypes.c_int32),
        ("positions_dev", ctypes.c_void_p),
        ("slots_dev", ctypes.c_void_p),
        ("rope_theta", ctypes.c_float),
        ("rope_table_dev", ctypes.c_void_p),
        ("argmax_keys_dev", ctypes.c_void_p),
        ("argmax_col_offset", ctypes.c_int32),
    ]


class GemmPhase(ctypes.Structure):
    """astraea_gemm_phase (include/astraea_b200.h)."""

    _fields_ = [
        ("A", ctypes.c_void_p),
        ("lda", ctypes.c_int32),
        ("W", ctypes.c_void_p),
        ("ldw", ctypes.c_int32),
        ("C", ctypes.c_void_p),
        ("ldc", ctypes.c_int32),
        ("N", ctypes.c_int32),
        ("K", ctypes.c_int32),
        ("epi", Epilogue),
    ]


EPI_SILU = 2
EPI_QKV_ROPE = 3
EPI_ARGMAX = 4
PHASE_GEMM = 0
PHASE_ATTN = 1


class AttnPhase(ctypes.Structure):
    """astraea_attn_phase (include/astraea_b200.h)."""

    _fields_ = [
        ("pool_dev", ctypes.c_void_p),
        ("geo", KvGeometry),
        ("layer", ctypes.c_int32),
        ("num_q_heads", ctypes.c_int32),
        ("q_dev", ctypes.c_void_p),
        ("q_row_stride", ctypes.c_int32),
        ("table_dev", ctypes.c_void_p),
        ("max_blocks", ctypes.c_int32),
        ("ctx_dev", ctypes.c_void_p),
        ("scale", ctypes.c_float),
        ("out_dev", ctypes.c_void_p),
    ]


class StepPhase(ctypes.Structure):
    """astraea_step_phase (include/astraea_b200.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("gemm", GemmPhase),
        ("a_from", ctypes.c_int32),
        ("epi_from", ctypes.c_int32),
        ("pool_dev", ctypes.c_void_p),
        ("geo", KvGeometry),
        ("layer", ctypes.c_int32),
        ("num_q_heads", ctypes.c_int32),
        ("q_dev", ctypes.c_void_p),
        ("q_row_stride", ctypes.c_int32),
        ("table_dev", ctypes.c_void_p),
        ("max_blocks", ctypes.c_int32),
        ("ctx_dev", ctypes.c_void_p),
        ("scale", ctypes.c_float),
        ("out_dev", ctypes.c_void_p),
        ("qkv_from", ctypes.c_int32),
    ]

_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_f32 = ctypes.c_float
_i32p = ctypes.POINTER(ctypes.c_int32)
_geo = ctypes.POINTER(KvGeometry)

# name -> (restype, argtypes); must match include/astraea_b200.h exactly.
SIGNATURES = {
    "astraea_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "astraea_abi_version": (ctypes.c_int, []),
    "astraea_kv_block_bytes": (_sz, [_geo]),
    "astraea_kv_bytes_per_token": (_sz, [_geo]),
    "astraea_alloc_create": (ctypes.c_int, [_i32, ctypes.POINTER(_vp)]),
    "astraea_alloc_destroy": (ctypes.c_int, [_vp]),
    "astraea_alloc_take": (ctypes.c_int, [_vp, _i32, _i32p]),
    "astraea_alloc_give": (ctypes.c_int, [_vp, _i32p, _i32]),
    "astraea_alloc_free_count": (_i32, [_vp]),
    "astraea_kv_swap_out": (ctypes.c_int, [_geo, _vp, _i32p, _i32, _i32, _vp, ctypes.c_int, _vp]),
    "astraea_kv_swap_in": (ctypes.c_int, [_geo, _vp, _i32p, _i32, _i32, _vp, ctypes.c_int, _vp]),
    "astraea_kv_copy_blocks": (ctypes.c_int, [_geo, _vp, _i32p, _i32p, _i32, _vp]),
    "astraea_block_table_build": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "astraea_rope_kv_append": (ctypes.c_int, [_geo, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _f32, _vp]),
    "astraea_decode_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "astraea_paged_decode_attention": (
        ctypes.c_int, [_geo, _vp, _i32, _vp, _i32, _i32, _i32, _vp, _i32, _vp, _f32, _vp, _vp, _sz, _vp]),
    "astraea_paged_prefill_attention": (
        ctypes.c_int, [_geo, _vp, _i32, _vp, _i32, _vp, _i32, _i32, _i32, _vp, _i32, _vp, _f32, _vp, _vp]),
    "astraea_gemm_workspace_bytes": (_sz, [_i32, _i32, _i32]),
    "astraea_gemm_bf16": (
        ctypes.c_int, [_vp, _i32, _vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _sz, _vp]),
    "astraea_gemm_bf16_ex": (
        ctypes.c_int, [_vp, _i32, _vp, _i32, _vp, _i32, _i32, _i32, _i32, ctypes.POINTER(Epilogue), _vp, _sz, _vp]),
    "astraea_debug_gemm_trace": (ctypes.c_int, [_vp, _i32, _i32]),
    "astraea_debug_prefill_trace": (ctypes.c_int, [_vp]),
    "astraea_rope_table": (ctypes.c_int, [_vp, _i32, _i32, _f32, _vp, _vp]),
    "astraea_gemm_chain_workspace_bytes": (_sz, [_i32, _i32, ctypes.POINTER(GemmPhase)]),
    "astraea_gemm_chain": (ctypes.c_int, [_i32, _i32, ctypes.POINTER(GemmPhase), _vp, _sz, _vp]),
    "astraea_gemm_chain_attn": (
        ctypes.c_int, [_i32, _i32, ctypes.POINTER(AttnPhase), ctypes.POINTER(_i32), _i32, ctypes.POINTER(GemmPhase),
                       _vp, _sz, _vp]),
    "astraea_step_program_bytes": (_sz, [_i32]),
    "astraea_step_workspace_bytes": (_sz, [_i32, _i32, ctypes.POINTER(StepPhase)]),
    "astraea_step_program_build": (ctypes.c_int, [_i32, _i32, ctypes.POINTER(StepPhase), _vp, _sz, _vp, _sz]),
    "astraea_step_launch": (ctypes.c_int, [_i32, _i32, _vp, _vp, _i32, _vp]),
    "astraea_debug_step_trace": (ctypes.c_int, [_vp]),
    "astraea_decode_advance": (
        ctypes.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "astraea_row_ssq": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "astraea_rmsnorm": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _f32, _vp]),
    "astraea_silu_mul": (ctypes.c_int, [_vp, _vp, _i32, _i32, _vp]),
    "astraea_embedding": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "astraea_argmax": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp]),
}

_LIB = None


def load(path: os.PathLike | None = None):
    """Load and type the library (no device needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise DeviceError(
            f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback."
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().astraea_status_string(status).decode()
        raise DeviceError(f"{what} failed with status {status}: {msg}")


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    if _CUDA_OK:
        return _LIB
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 data path has no CPU fallback")
    major, minor = torch.cuda.get_device_capability()
    if major != 10:
        raise DeviceError(f"need an sm_100 (B200) device, found sm_{major}{minor}")
    lib = load()
    _CUDA_OK = True
    return lib


def ptr(t) -> int:
    """Device (or pinned host) address of a torch tensor, None -> 0."""
    return 0 if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def i32_array(values) -> ctypes.Array:
    arr = (ctypes.c_int32 * len(values))(*values)
    return arr

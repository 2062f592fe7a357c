"""ctypes binding of libsikv_b200.so (the C ABI declared in include/sikv_b200.h).

The library is built in-tree by ``paper_2603_14224_b200.build``; there is no fallback: if
the shared object is missing or no CUDA device is present, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# SIKV_LIB names an alternative in-tree build (A/B experiments); default: the shipped library
LIB_PATH = os.path.join(HERE, os.environ.get("SIKV_LIB", "libsikv_b200.so"))

IN_F32, IN_F64, IN_BF16 = 0, 1, 2
_DT = {torch.float32: IN_F32, torch.float64: IN_F64, torch.bfloat16: IN_BF16}

P = C.c_void_p
I = C.c_int
I64 = C.c_int64
SZ = C.c_size_t

_SIGS = {
    "sikv_last_error": (C.c_char_p, []),
    "sikv_abi_version": (I, []),
    "sikv_encode_workspace_bytes": (SZ, [I64, I64, I64]),
    "sikv_encode": (I, [P, P, I, I64, I64, I64, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                        P, P, P, SZ, P, P]),
    "sikv_window_sinks_workspace_bytes": (SZ, [I64, I64, I]),
    "sikv_window_sinks": (I, [P, I, I64, I64, I64, P, P, I, I, I, P, P, SZ, P]),
    "sikv_pack16": (I, [P, P, I, I64, I64, P, P, P, P, P]),
    "sikv_gather_rows": (I, [P, P, I, I64, I64, I64, P, I64, P, P, P, I, P]),
    "sikv_append": (I, [P, P, I, I64, I64, P, P, P, I64, I64, I, P, P]),
    "sikv_decode_smem_bytes": (I, [I64, I, I, I, I]),
    "sikv_decode_default_cap": (I, [I64, I, I]),
    "sikv_decode_step": (I, [P, P, P, P, P, I, P, I, P, I, P, I64, I64, I, I, I, P, P, P, I, P, P, P, SZ, P, I, I, P]),
    "sikv_decode_step_x": (I, [P, P, P, P, P, I, P, I, P, I, P, I64, I64, I, I, I, P, P, P, I, P, P, P, SZ, P, I, I,
                               P, P]),
    "sikv_exchange_wait": (I, [P, C.c_uint64, P]),
    "sikv_ipc_handle": (I, [P, P, P]),
    "sikv_ipc_open": (I, [P, P]),
    "sikv_ipc_close": (I, [P]),
    "sikv_decode_workspace_bytes": (SZ, [I64, I64]),
    "sikv_decode_workspace_bytes_k": (SZ, [I64, I64, I, I]),
    "sikv_decode_last_kernel": (I, []),
    "sikv_forced_blocks": (I, [I, I64]),
    "sikv_forced_block_words": (I, []),
    "sikv_pack_forced": (I, [P, P, I, P, P, I64, P, I, P, I64, P, I, I, I, P, P]),
    "sikv_append_forced": (I, [P, P, I, I64, P, P, P, P, P, I, P, P, I64, P, P, I, P, P]),
    "sikv_score_fast": (I, [P, P, P, I, I64, I64, I, P, P]),
    "sikv_debug_set_decode_profile": (I, [P]),
    "sikv_debug_set_attend_skip": (I, [I]),
    "sikv_build_lut_f64": (I, [P, P, I64, I, I, P, P]),
    "sikv_score_f64": (I, [P, P, I64, I, I64, P, P]),
    "sikv_topk_workspace_bytes": (SZ, [I64, I64]),
    "sikv_topk": (I, [P, I, I64, I64, P, I, I, P, P, I, P, P]),
    "sikv_dequant_rows": (I, [P, P, P, P, P, P, P, P, P, P, I, I, I, I64, I64, I64, P, I64, I, P, P]),
    "sikv_attend_f64_workspace_bytes": (SZ, [I64, I, I]),
    "sikv_attend_f64": (I, [P, P, P, P, P, P, P, P, P, P, I, I, I, I64, I64, I64, P, I, P, P, I, P, I, P,
                            P, P, P, I64, P, P, P, P]),
    "sikv_center": (I, [P, I, I64, I64, I64, P, P, P]),
}

MAX_PEERS = 8


class Exchange(C.Structure):
    """sikv_exchange (include/sikv_b200.h): the fused multi-GPU output exchange."""
    _fields_ = [("npeers", C.c_int), ("out", P * MAX_PEERS), ("flag", P * MAX_PEERS), ("unit_gid", P)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2603_14224_b200.build`")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if "SIKV_LIB" in os.environ and not hasattr(h, name):
                continue              # an older A/B build without this entry point
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def ptr(t) -> P | None:
    if t is None:
        return None
    if isinstance(t, int):
        return P(t)
    return P(t.data_ptr())


def stream() -> P:
    return P(torch.cuda.current_stream().cuda_stream)


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}; expected float32, float64 or bfloat16") from None


def call(name: str, *args) -> int:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().sikv_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 3:
            raise NotImplementedError(msg)
        raise RuntimeError(msg)
    return rc


_CUDA_SEEN = False


def require_cuda() -> torch.device:
    global _CUDA_SEEN
    if not _CUDA_SEEN:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_14224_b200 needs a CUDA device (B200, sm_100a); none is visible")
        _CUDA_SEEN = True
    return torch.device("cuda", torch.cuda.current_device())


STATUS_MESSAGES = (
    (1, "group min/max exceed the 16-bit parameter range"),
    (2, "alpha does not dominate |keys_norm|; stats were computed elsewhere"),
    (4, "contains non-finite entries"),
    (16, "values exceed the float16 range of the fast decode path"),
    (32, "recent buffer full"),
)


def raise_status(status: torch.Tensor, what: str = "input") -> None:
    """Read the device status word (one sync) and raise the reference's ValueError."""
    s = int(status.item())
    for bit, msg in STATUS_MESSAGES:
        if s & bit:
            raise ValueError(f"{what} {msg}" if bit == 4 else msg)

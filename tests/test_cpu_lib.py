"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/sikv_b200.h
declares, and its host-side argument validation works without a GPU."""

import ctypes
import os
import re

import pytest

from paper_2603_14224_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sikv_b200.h")).read()
    return sorted(set(re.findall(r"\b(sikv_\w+)\s*\(", src)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_lib._SIGS) <= set(syms)


def test_host_queries():
    lib = _lib.lib()
    assert lib.sikv_abi_version() == 8
    assert lib.sikv_encode_workspace_bytes(4, 4096, 128) > 0
    assert lib.sikv_topk_workspace_bytes(1, 1000) == 3 * 32 * 4
    cap = lib.sikv_decode_default_cap(32768, 2048, 64)
    assert 2048 < cap <= 2 * 2048 + 1024
    assert lib.sikv_decode_smem_bytes(32768, 2048, 64, 4, cap) <= 113 * 1024
    assert lib.sikv_forced_blocks(64, 0) == 4
    assert lib.sikv_forced_block_words() == 2 * 32 * 32 + 32


def test_argument_validation_without_gpu():
    with pytest.raises(ValueError, match="null"):
        _lib.call("sikv_decode_step", *([None] * 5), 0, None, 1, None, 0, None, 1, 10, 4, 1, 0, None, None, None,
                  0, None, None, None, 0, None, 0, 0, None)
    with pytest.raises(NotImplementedError, match="query heads"):
        _lib.call("sikv_decode_step", *([_lib.ptr(8)] * 5), 0, None, 1, None, 0, _lib.ptr(8), 1, 10, 9, 1, 0,
                  _lib.ptr(8), None, None, 0, None, None, None, 0, None, 0, 0, None)
    with pytest.raises(ValueError, match="kernel must be"):
        _lib.call("sikv_decode_step", *([_lib.ptr(8)] * 5), 0, None, 1, None, 0, _lib.ptr(8), 1, 10, 4, 1, 0,
                  _lib.ptr(8), None, None, 0, None, None, None, 0, None, 0, 2, None)
    with pytest.raises(ValueError, match="null"):
        _lib.call("sikv_append_forced", None, None, 0, 1, None, None, None, None, None, 0, None, None, 16, None,
                  None, 1, None, None)
    with pytest.raises(ValueError, match="non-negative"):
        _lib.call("sikv_topk", _lib.ptr(8), 0, 1, 10, None, 0, -1, _lib.ptr(8), _lib.ptr(8), 10, _lib.ptr(8), None)


def test_product_path_needs_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2603_14224_b200 as sk
    with pytest.raises(RuntimeError, match="CUDA"):
        sk.encode_keys([[1.0, 2.0, 3.0, 4.0]])

"""The C-ABI library loads without a GPU and exports every declared symbol;
the host-side block allocator (pure C++) behaves like the reference's
token accounting at block granularity."""

import re
from pathlib import Path

import pytest

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu.ops import BlockAllocator
from paper_2512_14142_b200.gpu.lib import DeviceError

HEADER = Path(__file__).resolve().parent.parent / "include" / "astraea_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"ASTRAEA_API\s+[\w\s\*]+?\b(astraea_\w+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared()
    assert "astraea_kv_swap_out" in names and "astraea_gemm_bf16" in names
    assert len(names) >= 24


def test_library_exports_every_declared_symbol():
    lib = L.load()
    for name in declared():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    assert sorted(L.SIGNATURES) == declared()


def test_status_strings():
    lib = L.load()
    assert lib.astraea_status_string(0) == b"ok"
    assert b"KV blocks" in lib.astraea_status_string(-2)
    assert lib.astraea_abi_version() == 1


def test_geometry_sizes_match_baseline():
    lib = L.load()
    g8 = L.KvGeometry(32, 8, 128, 16, 1)
    assert lib.astraea_kv_bytes_per_token(g8) == 131072          # Llama-3-8B
    assert lib.astraea_kv_block_bytes(g8) == 2 * 1024 * 1024
    assert lib.astraea_kv_bytes_per_token(L.KvGeometry(80, 1, 128, 16, 1)) == 40960  # 70B TP8
    assert lib.astraea_kv_bytes_per_token(L.KvGeometry(4, 2, 64, 16, 1)) == 2048     # small


def test_allocator_lifo_and_exhaustion():
    a = BlockAllocator(8)
    first = a.take(3)
    assert first == [0, 1, 2] and a.free == 5
    with pytest.raises(DeviceError):
        a.take(6)
    assert a.free == 5  # nothing taken on failure
    a.give(first)
    assert a.take(1) == [0]  # most recently freed first


def test_allocator_rejects_double_free():
    a = BlockAllocator(4)
    ids = a.take(2)
    a.give(ids)
    with pytest.raises(DeviceError):
        a.give([ids[0]])
    with pytest.raises(DeviceError):
        a.give([7])
    x = a.take(2)
    with pytest.raises(DeviceError):
        a.give([x[0], x[0]])
    assert a.free == 2


def test_device_calls_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(DeviceError):
        L.require_cuda()

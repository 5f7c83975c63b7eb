"""The C-ABI library builds, loads on a CPU-only box and exports every symbol that
include/heap.h declares (no compute calls here: there is no GPU)."""
import ctypes
import os
import re

import pytest

from paper_2405_07079_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "heap.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(heap_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    _native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTS)


def test_workspace_bytes_and_argument_checks():
    L = _native.lib()
    assert L.heap_workspace_bytes(1 << 20, 16, 4, 1024, 1024) > 0
    assert L.heap_workspace_bytes(1 << 20, 24, 4, 1024, 1024) == 0      # align not a power of two
    assert L.heap_workspace_bytes((1 << 20) + 8, 16, 4, 1024, 1024) == 0  # arena not a multiple
    assert L.heap_workspace_bytes(1 << 20, 16, 11, 1024, 1024) == 0      # bad policy
    assert L.heap_workspace_bytes(1 << 20, 16, 0, 1024, 1024) == 0
    for pol in range(1, 11):
        assert L.heap_workspace_bytes(1 << 20, 16, pol, 1024, 1024) > 0, pol
    for pol in (1, 2, 3, 4, 8):                                           # HEAP_PARTIAL_FREE flag
        assert L.heap_workspace_bytes(1 << 20, 16, pol | 0x100, 1024, 1024) > \
            L.heap_workspace_bytes(1 << 20, 16, pol, 1024, 1024), pol
    for pol in (5, 6, 7, 9, 10):                                          # needs address coalescing
        assert L.heap_workspace_bytes(1 << 20, 16, pol | 0x100, 1024, 1024) == 0, pol
    assert L.heap_workspace_bytes(1 << 20, 16, 4 | 0x200, 1024, 1024) == 0  # unknown flag
    assert L.heap_workspace_bytes((1 << 36) + (1 << 5), 16, 4, 1024, 1024) == 0  # > 2^32 units
    assert L.heap_workspace_bytes(1 << 36, 16, 4, 1024, 1024) > 0        # exactly 2^32 units
    h = ctypes.c_void_p()
    assert L.heap_create(1 << 20, 24, 4, 1024, 1024, None, 0, None, ctypes.byref(h)) == -1
    assert L.heap_free_batch(None, None, 0, None) == -1
    assert L.heap_free_batch_handles(None, None, 0, None, 0, None) == -1
    assert L.heap_step(None, None, None, 0, 0, None, None, 0, None) == -1
    assert L.heap_strerror(-3) == b"metadata capacity exceeded in a batch"


def test_product_path_has_no_oracle_import():
    """The product package never imports the oracle."""
    pkg = os.path.dirname(_native.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                s = open(os.path.join(root, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", s).replace("oracle/", ""), f


def test_binding_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2405_07079_b200 import Heap
    with pytest.raises(RuntimeError):
        Heap(1 << 20, 16, 4, 1024, 1024)

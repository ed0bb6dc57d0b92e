"""The C-ABI library loads and exports every entry point include/geopart_b200.h declares.

No compute calls without a GPU; the one host-side helper (gp_hilbert_cell_key_host)
shares the kernel's transpose code and is checked against the oracle here.
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "geopart_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def native():
    from paper_1805_01208_b200 import build

    build.build()
    from paper_1805_01208_b200 import _native

    return _native


def test_header_declares_the_minimum_export_set():
    names = set(declared())
    for must in ["gp_box_minmax", "gp_hilbert_keys", "gp_sort_pairs", "gp_sort_workspace_bytes",
                 "gp_gather_points", "gp_gather_rows", "gp_compact_active", "gp_assign_round",
                 "gp_movement_fold", "gp_scatter_by_gid", "gp_audit", "gp_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(native):
    lib = ctypes.CDLL(native.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
        assert name in native.EXPORTED, f"{name} not bound in _native.py"


def test_abi_version(native):
    assert native.lib.gp_abi_version() == 2


def test_struct_layouts_match_header(native):
    a, f = ctypes.c_size_t(0), ctypes.c_size_t(0)
    native.lib.gp_args_sizes(ctypes.byref(a), ctypes.byref(f))
    assert a.value == ctypes.sizeof(native.AssignArgs)
    assert f.value == ctypes.sizeof(native.FoldArgs)


@pytest.mark.parametrize("d,depth", [(2, 1), (2, 5), (2, 31), (3, 1), (3, 4), (3, 20)])
def test_host_cell_key_matches_oracle(native, d, depth):
    from oracle import geographer_oracle as O

    rng = np.random.default_rng(d * 100 + depth)
    cells = rng.integers(0, 1 << depth, size=(500, d)).astype(np.uint64)
    want = O.hilbert_from_cells(cells, depth)
    arr = (ctypes.c_uint32 * 3)()
    for i in range(cells.shape[0]):
        for j in range(d):
            arr[j] = int(cells[i, j])
        got = native.lib.gp_hilbert_cell_key_host(arr, d, depth)
        assert got == int(want[i])


def test_errors_are_reported_not_raised(native):
    rc = native.lib.gp_hilbert_keys(None, 10, 4, 4, 1, None, 20, None, None, 0, None)
    assert rc == 1
    assert b"unsupported dimension" in native.lib.gp_last_error()
    rc = native.lib.gp_hilbert_keys(None, 10, 3, 3, 1, None, 21, None, None, 0, None)
    assert rc == 1 and b"depth" in native.lib.gp_last_error()


@pytest.mark.parametrize("d", [2, 3])
def test_hilbert_fsm_tables_match_transpose(native, d):
    """The kernel's table form of the key (several levels per lookup) agrees with the
    transpose of geometry.py:135-179 at every depth (host-only check)."""
    assert native.lib.gp_hilbert_fsm_selfcheck(d) == 0, native.lib.gp_last_error()

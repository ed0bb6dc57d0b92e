"""ctypes binding of the C ABI in include/geopart_b200.h.

There is no CPU fallback: importing this module loads libgeopart_b200.so and
raises if it is missing, so a GPU box without the built extension fails
loudly instead of silently running something else.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GP_LIB_PATH: load a tuning variant built by `python -m paper_1805_01208_b200.build
# --variant NAME -DX=Y` instead (experiments only)
LIB_PATH = os.environ.get("GP_LIB_PATH") or os.path.join(_HERE, "libgeopart_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1805_01208_b200.build` "
        "(there is no CPU fallback)"
    )
lib = C.CDLL(LIB_PATH)

i32, i64, u32, u64, f64, vp, sz = (C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double,
                                   C.c_void_p, C.c_size_t)


class AssignArgs(C.Structure):
    _fields_ = [
        ("X", vp), ("ldx", i64), ("d", i32), ("k", i32), ("order3", i32), ("wmode", i32),
        ("w", vp), ("wscale", f64), ("list", vp), ("m", i64), ("a", vp), ("ublb", vp),
        ("centers", vp), ("infl", vp), ("inv2_lo", vp), ("inv2_hi", vp), ("ub_eval", vp),
        ("ub_norm", vp), ("lb_par", vp), ("block_w", vp), ("counters", vp),
        ("group_list", vp), ("group_count", vp), ("group_cap", i32), ("group_shift", i32),
        ("workspace", vp), ("workspace_bytes", sz), ("scan_regions", i32), ("grid_n", i32),
        ("grid_start", vp), ("grid_items", vp), ("grid_lo", f64 * 3), ("grid_h", f64),
        ("inv2_min", f64), ("unit_boxes", vp), ("unit_shift", i32), ("flags", i32),
        ("lb_rpar", vp), ("lb_rshift", i32), ("bound_scale", C.c_float), ("inv2_min_dev", vp),
        ("split_event", vp),
    ]


class FoldArgs(C.Structure):
    _fields_ = [
        ("X", vp), ("ldx", i64), ("d", i32), ("k", i32), ("order3", i32), ("wmode", i32),
        ("w", vp), ("a", vp), ("n_local", i64), ("pos0", i64), ("n_global", i64),
        ("centers", vp), ("weights_only", i32), ("sums", vp), ("wsum", vp), ("extent", vp),
        ("objective", vp), ("workspace", vp), ("workspace_bytes", sz), ("list", vp), ("m", i64),
    ]


_SIGS = {
    "gp_last_error": (C.c_char_p, []),
    "gp_abi_version": (C.c_int, []),
    "gp_host_is_pinned": (C.c_int, [vp]),
    "gp_args_sizes": (None, [C.POINTER(sz), C.POINTER(sz)]),
    "gp_box_minmax": (C.c_int, [vp, i64, C.c_int, i64, i64, vp, vp, vp]),
    "gp_weight_probe": (C.c_int, [vp, i64, vp, vp]),
    "gp_hilbert_keys": (C.c_int, [vp, i64, C.c_int, i64, i64, vp, C.c_int, vp, vp, u32, vp]),
    "gp_hilbert_cell_key_host": (u64, [C.POINTER(u32), C.c_int, C.c_int]),
    "gp_hilbert_fsm_selfcheck": (C.c_int, [C.c_int]),
    "gp_sort_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_sort_pairs": (C.c_int, [vp, vp, vp, vp, i64, C.c_int, vp, sz, vp]),
    "gp_gather_points": (C.c_int, [vp, i64, i64, C.c_int, vp, i64, vp, i64, vp, C.c_int, vp,
                                   vp]),
    "gp_gather_rows": (C.c_int, [vp, i64, C.c_int, vp, C.c_int, vp, vp]),
    "gp_compact_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_compact_active": (C.c_int, [vp, i64, i64, vp, vp, vp, sz, vp]),
    "gp_compact_candidates": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, sz, vp]),
    "gp_sample_ranks_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_sample_ranks": (C.c_int, [C.POINTER(u64), i64, vp, vp, sz, vp]),
    "gp_assign_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_assign_round": (C.c_int, [C.POINTER(AssignArgs), vp]),
    "gp_rebase_bounds": (C.c_int, [C.POINTER(AssignArgs), vp]),
    "gp_update_maps": (C.c_int, [vp, vp, vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_int, f64,
                                 vp]),
    "gp_group_boxes": (C.c_int, [vp, i64, C.c_int, vp, i64, C.c_int, vp, vp]),
    "gp_group_candidates": (C.c_int, [vp, i64, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_int,
                                      C.c_int, vp, vp, C.c_int, vp]),
    "gp_audit": (C.c_int, [C.POINTER(AssignArgs), vp, vp]),
    "gp_fold_workspace_bytes": (C.c_int, [i64, i64, i64, C.c_int, C.POINTER(sz)]),
    "gp_movement_fold": (C.c_int, [C.POINTER(FoldArgs), vp]),
    "gp_fold_stats": (C.c_int, [vp]),
    "gp_lb_remap": (C.c_int, [vp, C.c_int, vp]),
    "gp_region_maps": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, i64, vp, vp, vp, C.c_int, f64,
                                 vp]),
    "gp_scan_stats": (C.c_int, [vp, C.c_int]),
    "gp_fold_export": (C.c_int, [C.POINTER(FoldArgs), vp, vp, vp, vp]),
    "gp_fold_combine_bytes": (C.c_int, [C.c_int, C.POINTER(sz)]),
    "gp_fold_combine": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, sz,
                                  vp]),
    "gp_scatter_by_gid": (C.c_int, [vp, vp, i64, vp, vp]),
    "gp_deliver_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_deliver_permutation": (C.c_int, [vp, vp, i64, vp, vp, sz, vp]),
    "gp_gather_state": (C.c_int, [vp, i64, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp,
                                  vp]),
    "gp_scatter_state": (C.c_int, [vp, i64, vp, vp, vp, vp, vp]),
    "gp_gather_ranks": (C.c_int, [vp, vp, i64, vp, vp]),
    "gp_center_grid_workspace_bytes": (C.c_int, [C.c_int, C.POINTER(sz)]),
    "gp_center_grid": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(f64), f64, C.c_int, vp, vp, vp,
                                 sz, vp]),
    "gp_balance_decide": (C.c_int, [vp, C.c_int, f64, f64, C.c_int, vp, vp, vp, vp]),
    "gp_sfc_cut_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_sfc_cut": (C.c_int, [vp, vp, i64, C.c_int, f64, vp, vp, sz, vp]),
    "gp_predict": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp]),
    # formats and evaluation either side of the path (csrc/textio.cu, csrc/graphs.cu)
    "gp_parse_number_host": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(i64)]),
    "gp_text_index_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_text_index": (C.c_int, [vp, i64, C.c_int, vp, vp, sz, vp]),
    "gp_text_tokens": (C.c_int, [vp, i64, C.c_int, vp, i64, i64, vp, vp, vp, vp, vp]),
    "gp_metis_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_metis_lines": (C.c_int, [vp, vp, i64, vp, i64, vp, vp, sz, vp]),
    "gp_metis_offsets": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, vp, vp, vp, sz, vp]),
    "gp_metis_fill": (C.c_int, [vp, vp, vp, vp, i64, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp]),
    "gp_table_values": (C.c_int, [vp, i64, vp, vp, i64, C.c_int, vp, vp, vp]),
    "gp_format_ints_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_format_ints_plan": (C.c_int, [vp, i64, vp, vp, sz, vp]),
    "gp_format_ints_write": (C.c_int, [vp, i64, vp, vp, vp]),
    "gp_graph_check_workspace_bytes": (C.c_int, [i64, C.POINTER(sz)]),
    "gp_graph_check": (C.c_int, [vp, vp, vp, i64, i64, vp, vp, vp, sz, vp]),
    "gp_edge_cut_workspace_bytes": (C.c_int, [i64, i64, C.POINTER(sz)]),
    "gp_edge_cut": (C.c_int, [vp, vp, vp, f64, vp, i64, i64, vp, vp, sz, vp]),
    "gp_comm_volumes": (C.c_int, [vp, vp, vp, i64, C.c_int, vp, vp, vp]),
    "gp_block_weights_workspace_bytes": (C.c_int, [i64, C.c_int, C.POINTER(sz)]),
    "gp_block_weights": (C.c_int, [vp, vp, i64, C.c_int, f64, vp, vp, sz, vp]),
    "gp_block_bfs": (C.c_int, [vp, vp, vp, i64, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp]),
    "gp_block_level_top": (C.c_int, [vp, vp, i64, C.c_int, vp, vp, vp, vp, vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


def _verify_layouts():
    a, f = sz(0), sz(0)
    lib.gp_args_sizes(C.byref(a), C.byref(f))
    if a.value != C.sizeof(AssignArgs) or f.value != C.sizeof(FoldArgs):
        raise ImportError(f"struct layout mismatch: C {a.value}/{f.value} vs ctypes "
                          f"{C.sizeof(AssignArgs)}/{C.sizeof(FoldArgs)}")


_verify_layouts()


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib.gp_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'geopart_b200'}: error {rc}: {msg}")


# kernels launched per API call (bench.py's gpu_launches claim); CUB's sort is
# counted as one histogram pass plus one launch per 8-bit digit pass
KERNELS_PER_CALL = {
    "gp_box_minmax": 2, "gp_weight_probe": 1, "gp_hilbert_keys": 1, "gp_sort_pairs": 9,
    "gp_gather_points": 1, "gp_gather_rows": 1, "gp_compact_active": 1, "gp_compact_candidates": 1,
    "gp_assign_round": 2, "gp_rebase_bounds": 1, "gp_audit": 1, "gp_movement_fold": 13,
    "gp_scatter_by_gid": 1, "gp_deliver_permutation": 4, "gp_gather_ranks": 1,
    "gp_group_boxes": 1,
    "gp_group_candidates": 1, "gp_sample_ranks": 170, "gp_gather_state": 1, "gp_scatter_state": 1, "gp_update_maps": 3, "gp_region_maps": 1, "gp_lb_remap": 1, "gp_fold_export": 1, "gp_fold_combine": 3,
    "gp_sfc_cut": 3, "gp_predict": 1, "gp_balance_decide": 1, "gp_center_grid": 3,
    "gp_text_index": 2, "gp_text_tokens": 1, "gp_metis_lines": 3, "gp_metis_offsets": 2,
    "gp_metis_fill": 1, "gp_table_values": 3, "gp_format_ints_plan": 2,
    "gp_format_ints_write": 1, "gp_graph_check": 22, "gp_edge_cut": 2, "gp_comm_volumes": 2,
    "gp_block_weights": 2, "gp_block_bfs": 1, "gp_block_level_top": 1,
}
_launches = [0]
calls: dict[str, int] = {}   # API calls by name (tools/kprof.py)


def reset_launch_count() -> None:
    _launches[0] = 0


def launch_count() -> int:
    return _launches[0]


def count(name: str) -> None:
    _launches[0] += KERNELS_PER_CALL.get(name, 0)
    calls[name] = calls.get(name, 0) + 1


def call(name: str, *args) -> None:
    count(name)
    check(getattr(lib, name)(*args), name)


def size_query(name: str, *args) -> int:
    out = sz(0)
    check(getattr(lib, name)(*args, C.byref(out)), name)
    return int(out.value)

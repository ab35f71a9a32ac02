"""ctypes binding of ``libspamm_b200.so`` (the C ABI in ``include/spamm_b200.h``).

The library is built in-tree by ``csrc/build.sh`` (``__graft_entry__.build()``).
There is no fallback of any kind: if the library is missing or no CUDA device is
present, the first call raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPAMM_B200_LIB: another build of the same library (A/B comparisons of kernel variants)
LIB_PATH = os.environ.get("SPAMM_B200_LIB") or os.path.join(_HERE, "csrc", "libspamm_b200.so")

SPAMM_OK, SPAMM_EINVAL, SPAMM_ECUDA, SPAMM_EWORKSPACE = 0, 1, 2, 3
FINE4, COARSE16 = 0, 1

vp, i32, i64, f32, f64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_size_t


class TreeView(C.Structure):
    """``spamm_tree_view``."""

    _fields_ = [("m", i32), ("n", i32), ("depth", i32), ("nleaf", i32),
                ("keys", vp), ("values", vp), ("values_t", vp),
                ("slot", vp), ("slot_t", vp), ("norm", vp), ("norm_t", vp), ("sub", vp), ("sub_t", vp)]


class PlanBuffers(C.Structure):
    """``spamm_plan_buffers``."""

    _fields_ = [("steps", vp), ("c_keys", vp), ("tile_off", vp), ("tile_order", vp), ("chain", vp),
                ("step_capacity", i64),
                ("leaf_capacity", i64), ("counts", vp)]


class ProductBuffers(C.Structure):
    """``spamm_product_buffers``."""

    _fields_ = [("values", vp), ("values_t", vp), ("leaf_sq", vp), ("slot", vp), ("slot_t", vp), ("norm", vp),
                ("norm_t", vp), ("leaf_sq_grid", vp), ("sq_levels", vp), ("depth", i32)]


class ArenaLayout(C.Structure):
    """``spamm_arena_layout`` (byte offsets into the single allocation of spamm_multiply_arena)."""

    _fields_ = [(n, i64) for n in ("counts", "steps", "c_keys", "tile_off", "tile_order", "chain", "plan_ws_bytes",
                                   "values", "values_t", "leaf_sq", "slot", "slot_t", "norm", "norm_t", "leaf_sq_grid",
                                   "sq_levels", "total")]


class HostOperands(C.Structure):
    """``spamm_host_operands``: leaf blocks in pinned host memory, flag scratch on the device."""

    _fields_ = [("a_blocks", vp), ("a_nleaf", i64), ("a_flags", vp), ("b_blocks", vp), ("b_nleaf", i64), ("b_flags", vp),
                ("fetched", vp)]


REC = 272           # floats per stored leaf record: 256 values + 16 sub-block norms
STEP_WORDS = 16     # uint32 words per step record (struct spamm_step)
PLAN_COUNTS = 32
UNIT_EXTRA = 8192   # SPAMM_UNIT_EXTRA: tile_order holds leaf_capacity + UNIT_EXTRA units, then the chain flags


# every symbol include/spamm_b200.h declares: (restype, argtypes)
SIGNATURES = {
    "spamm_abi_version": (C.c_int, []),
    "spamm_level_offset_of": (i64, [C.c_int]),
    "spamm_error_string": (C.c_char_p, [C.c_int]),
    "spamm_launch_count": (i64, []),
    "spamm_leaf_norms_dense": (C.c_int, [vp, i64, i64, i64, C.c_int, vp, vp, vp, vp]),
    "spamm_scan_workspace_bytes": (sz, [i64]),
    "spamm_assign_slots": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, sz, vp]),
    "spamm_pack_leaves": (C.c_int, [vp, i64, i64, i64, C.c_int, vp, i64, vp, vp, vp, vp]),
    "spamm_build_interior": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int, vp]),
    "spamm_leaf_norms_packed": (C.c_int, [vp, i64, vp, vp, vp]),
    "spamm_leaves_from_blocks": (C.c_int, [vp, i64, vp, vp, vp, vp]),
    "spamm_subnorm_tails": (C.c_int, [vp, i64, vp, vp, vp]),
    "spamm_mark_touched": (C.c_int, [C.POINTER(PlanBuffers), vp, vp, vp]),
    "spamm_gather_blocks": (C.c_int, [vp, vp, i64, C.c_int, vp, vp, vp, vp]),
    "spamm_transpose_records": (C.c_int, [vp, i64, vp, vp]),
    "spamm_sparsify_leaves": (C.c_int, [vp, vp, vp, i64, C.c_float, vp, vp]),
    "spamm_index_leaves": (C.c_int, [vp, vp, i64, C.c_int, vp, vp, vp, vp, vp, vp]),
    "spamm_subrange_grids": (C.c_int, [vp, vp, C.c_int, vp, vp, vp]),
    "spamm_to_dense": (C.c_int, [C.POINTER(TreeView), vp, i64, vp]),
    "spamm_plan_workspace_bytes": (sz, [C.c_int, i64, i64]),
    "spamm_plan": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), f64, i32, i32,
                             C.POINTER(PlanBuffers), vp, sz, vp]),
    "spamm_plan_row_counts": (C.c_int, [C.POINTER(PlanBuffers), C.c_int, vp, vp]),
    "spamm_execute": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), C.POINTER(PlanBuffers), i64, i64,
                                f64, f32, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
    "spamm_execute_gates": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), C.POINTER(PlanBuffers), i64, i64,
                                      f64, vp, vp, vp, vp, vp, vp]),
    "spamm_multiply": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), f64, C.c_int, C.c_int, f32, i32, i32,
                                 C.POINTER(PlanBuffers), vp, sz, C.POINTER(ProductBuffers), vp]),
    "spamm_multiply_arena_layout": (C.c_int, [C.c_int, C.c_int, i64, i64, C.POINTER(ArenaLayout)]),
    "spamm_multiply_arena": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), f64, C.c_int, C.c_int, f32, i32, i32,
                                       C.c_int, i64, i64, vp, sz, vp, sz, vp]),
    "spamm_multiply_host": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), f64, C.c_int, C.c_int, f32, i32, i32,
                                      C.POINTER(PlanBuffers), vp, sz, C.POINTER(ProductBuffers), C.POINTER(HostOperands), vp]),
    "spamm_multiply_arena_host": (C.c_int, [C.POINTER(TreeView), C.POINTER(TreeView), f64, C.c_int, C.c_int, f32, i32, i32,
                                            C.c_int, i64, i64, vp, sz, vp, sz, C.POINTER(HostOperands), vp]),
    "spamm_exchange_allgather": (C.c_int, [vp, vp, vp, vp, i64, vp, vp, vp, vp]),
    "spamm_union_leaves": (C.c_int, [vp, vp, i64, C.c_int, vp, vp, vp, vp, vp, vp, sz, vp]),
    "spamm_compose": (C.c_int, [vp, vp, vp, vp, i64, f32, f32, C.c_int, C.c_int, vp, vp]),
}

_lib = None


def lib():
    """The loaded library.  Raises RuntimeError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(paper_1203_1692_b200 has no CPU or PyTorch fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.spamm_abi_version() != 2:
            raise RuntimeError("libspamm_b200.so ABI version mismatch; rebuild it")
        _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    """Map a status code to the reference's exceptions (ValueError for bad arguments)."""
    if rc == SPAMM_OK:
        return
    msg = f"{what}: {lib().spamm_error_string(rc).decode()}"
    if rc == SPAMM_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(lib().spamm_launch_count())


def level_offset(t: int) -> int:
    return 0 if t == 0 else 4 + ((1 << (2 * t)) - 4) // 3


def level_total(depth: int) -> int:
    """Elements of a level buffer holding levels 0..depth."""
    return level_offset(depth) + (1 << (2 * depth))

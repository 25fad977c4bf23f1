"""ctypes binding of libgcb200.so (the C-ABI in ``include/gcb200.h``).

There is no CPU fallback: if the library or a CUDA device is missing every
device entry point raises :class:`DeviceError` instead of computing anything
on the host.  Status codes map onto the reference's exception classes
(``greencross/errors.py:4-35``).
"""

import ctypes
import os

from .errors import ConfigError, DeviceError, GeometryError, GreencrossError, StateError

LIB_PATH = os.environ.get("GC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgcb200.so")

c_i64 = ctypes.c_int64
c_p = ctypes.c_void_p


class GcGeom(ctypes.Structure):
    _fields_ = [("corners", c_p), ("gram", c_p), ("tri_vid", c_p), ("xq", c_p),
                ("wq", c_p), ("nt", c_i64), ("mq", c_i64), ("wq_host", c_p),
                ("normals", c_p), ("kernel", c_i64), ("vstar_ptr", c_p), ("vstar_ent", c_p),
                ("bq", c_p), ("basis", c_i64), ("verts", c_p), ("nodes6", c_p), ("nrm6", c_p),
                ("gq", c_p), ("nq", c_p)]


class GcRules(ctypes.Structure):
    _fields_ = [("table", c_p * 4), ("npts", c_i64 * 4)]


class GcQueue(ctypes.Structure):
    _fields_ = [("tasks", c_p * 4), ("cap", c_i64 * 4), ("count", c_p)]


# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGNATURES = {
    "gc_abi_version": [],
    "gc_last_error": [],
    "gc_launch_count": [],
    "gc_reset_launch_count": [],
    "gc_surface_points": [c_p, c_i64, c_p, c_i64, c_p, c_p],
    "gc_chart_pack": [c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_pair_eval": [ctypes.POINTER(GcGeom), ctypes.POINTER(GcRules), ctypes.c_int, c_i64,
                     c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_assemble_blocks": [ctypes.POINTER(GcGeom), c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p,
                           ctypes.POINTER(GcQueue), c_p, c_p],
    "gc_singular_flush": [ctypes.POINTER(GcGeom), ctypes.POINTER(GcRules),
                          ctypes.POINTER(GcQueue), c_p, ctypes.POINTER(c_i64), c_p],
    "gc_singular_flush_async": [ctypes.POINTER(GcGeom), ctypes.POINTER(GcRules),
                                ctypes.POINTER(GcQueue), c_p, c_p, c_p],
    "gc_batched_transpose": [c_i64, c_p, c_p, c_p, c_p],
    "gc_block_tree": [c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_i64, ctypes.c_double,
                      ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(c_p), ctypes.POINTER(c_i64)],
    "gc_block_tree_fetch": [c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_bt_level_bytes": [c_i64, ctypes.POINTER(c_i64)],
    "gc_bases_scan_bytes": [c_i64, ctypes.POINTER(c_i64)],
    "gc_bases_R": [c_i64] + [c_p] * 6 + [c_i64, c_i64] + [c_p] * 4 + [c_p],
    "gc_bases_scan": [c_i64] + [c_p] * 7 + [c_i64, c_p, c_p, c_i64, c_p],
    "gc_bases_rows": [c_i64] + [c_p] * 8 + [c_i64, c_i64, c_i64, c_i64] + [c_p] * 7 + [c_p],
    "gc_bases_post": [c_i64, c_p, c_i64] + [c_p] * 6 + [c_i64] + [c_p] * 7 + [c_i64, c_p],
    "gc_h2_blocks_bytes": [c_i64, ctypes.POINTER(c_i64)],
    "gc_h2_blocks": [c_i64] + [c_p] * 14 + [c_i64, c_i64, ctypes.c_int32, ctypes.c_int32] + [c_p] * 6
                    + [c_i64, c_p],
    "gc_bt_leaves_bytes": [c_i64, ctypes.POINTER(c_i64)],
    "gc_bt_leaves": [c_i64] + [c_p] * 11 + [c_i64, c_p],
    "gc_bt_level": [c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_i64, ctypes.c_int32] + [c_p] * 10
                   + [ctypes.c_double, ctypes.c_int32] + [c_p] * 14 + [c_i64, c_p],
    "gc_green_box_rules": [ctypes.c_int, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_green_factor": [ctypes.POINTER(GcGeom), ctypes.c_int, c_i64, c_i64, c_p, c_p, c_p,
                        c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_aca": [c_i64, c_p, c_i64, ctypes.c_double, c_i64, c_p, c_p, c_p, c_p, c_p, c_i64, c_p],
    "gc_gather": [c_p, c_p, c_i64, c_p, c_p],
    "gc_scatter": [c_p, c_p, c_i64, c_p, c_p],
    "gc_scatter2": [c_p, c_p, c_p, c_i64, c_p, c_p],
    "gc_expand_ranges": [c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_tier_compose": [c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_tier_tile": [],
    "gc_graph_retarget": [c_p, c_p, ctypes.c_int32, ctypes.c_int32, c_p, c_p, c_p],
    "gc_gather_inv": [c_p, c_p, c_i64, c_p, c_p],
    "gc_plan_create": [c_i64, c_p, c_i64, c_p, c_i64, c_p, c_p],
    "gc_plan_run": [c_p, c_p, c_p, c_p],
    "gc_plan_run_host": [c_p, c_p, c_p, c_i64, c_p, c_p],
    "gc_plan_destroy": [c_p],
    "gc_scatter2_inv": [c_p, c_p, c_p, c_i64, c_p, c_p],
    "gc_block_transpose": [c_i64, c_p, c_p, c_p, c_p],
    "gc_panelmv": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_p, c_p, ctypes.c_int32,
                   ctypes.c_int32, c_p, c_p],
    "gc_lin_pairs": [ctypes.POINTER(GcGeom), c_p, c_p, c_i64, c_p, c_p, c_p, ctypes.POINTER(GcQueue), c_p, c_p],
    "gc_lin_singular": [ctypes.POINTER(GcGeom), ctypes.POINTER(GcRules), ctypes.POINTER(GcQueue), c_p,
                        ctypes.POINTER(c_i64), c_p],
    "gc_lin_gather": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_curved_singular": [ctypes.POINTER(GcGeom), ctypes.POINTER(GcRules), ctypes.POINTER(GcQueue), c_i64,
                           c_p, ctypes.POINTER(c_i64), c_p],
    "gc_curved_pairs": [ctypes.POINTER(GcGeom), c_p, c_i64, c_p, c_i64, c_i64, c_p, c_p],
    "gc_tree_boxes": [c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_tree_sort_bytes": [c_i64, c_i64, ctypes.POINTER(c_i64)],
    "gc_tree_axis": [c_i64, c_p, c_p, c_p, c_p],
    "gc_tree_split": [c_i64, c_p, c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_p],
    "gc_tree_split_small": [c_i64, c_p, c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_p],
    "gc_lin_pairs_blocks": [ctypes.POINTER(GcGeom), c_p, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p,
                            ctypes.POINTER(GcQueue), c_p, c_p],
    "gc_col_pairs_blocks": [ctypes.POINTER(GcGeom), c_p, c_p, c_p, c_i64, c_p, c_p, c_i64, c_i64, c_p, c_p, c_p,
                            c_p, c_p, c_p, c_p],
    "gc_col_pairs": [ctypes.POINTER(GcGeom), c_p, c_p, c_p, c_i64, c_p, c_p, c_i64, c_p, c_p, c_p, c_p],
    "gc_dot": [c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_cg_pq": [c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_cg_update": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_krylov_partials": [],
    "gc_priority_range": [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
    "gc_cgnr_step": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "gc_cgnr_dir": [c_i64, c_p, c_p, c_p, c_p, c_p],
    "gc_scale_inv_norm": [c_i64, c_p, c_p, c_p],
    "gc_axpy_neg": [c_i64, c_p, c_p, c_p],
    "gc_nccl_unique_id": [c_p],
    "gc_nccl_comm_init": [c_p, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(c_p)],
    "gc_nccl_comm_destroy": [c_p],
    "gc_nccl_all_gather": [c_p, c_p, c_i64, c_p, c_p],
    "gc_host_norm3": [c_p, c_i64, c_p, ctypes.c_int],
    "gc_dfma_probe": [c_i64, c_i64, c_i64, c_p, c_p],
}
_RESTYPES = {"gc_last_error": ctypes.c_char_p, "gc_launch_count": ctypes.c_uint64,
             "gc_tier_tile": ctypes.c_int64,
             "gc_reset_launch_count": None, "gc_krylov_partials": ctypes.c_int64}

EXPORTED = tuple(_SIGNATURES)
ABI_VERSION = 3

_lib = None


def load():
    """Load (once) and type the library; raises DeviceError if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError("native library %s is missing; run "
                              "`python -m paper_1810_08429_b200.build_native`" % LIB_PATH)
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        if lib.gc_abi_version() != ABI_VERSION:
            raise DeviceError("libgcb200 ABI %d, expected %d" % (lib.gc_abi_version(), ABI_VERSION))
        _lib = lib
    return _lib


_ERRORS = {1: ConfigError, 2: GeometryError, 3: DeviceError, 4: StateError}


def check(rc):
    if rc != 0:
        msg = load().gc_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, GreencrossError)(msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def launch_count():
    return int(load().gc_launch_count())

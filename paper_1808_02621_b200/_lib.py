"""ctypes binding of ``libhybridpath.so`` (the C ABI in ``include/hybridpath.h``).

There is no CPU fallback: if the library is missing the import of any device
op raises. ``symbols()`` lists every exported entry point so the CPU test suite
can check the ABI without a GPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# HP_LIB overrides the library path (A/B of two builds of the same sources)
LIB_PATH = Path(os.environ.get("HP_LIB") or Path(__file__).resolve().parent / "lib" /
                "libhybridpath.so")

HP_OPT = {"sgd": 0, "adagrad": 1, "adam": 2}
HP_DTYPE = {"float32": 0, "bfloat16": 1, "float16": 2}

vp = C.c_void_p
i32, i64, u64, f32, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_size_t


class Optim(C.Structure):
    _fields_ = [("kind", i32), ("lr", f32), ("beta1", f32), ("beta2", f32),
                ("one_minus_beta1", f32), ("one_minus_beta2", f32), ("eps", f32),
                ("lr_t", f32), ("agg_scale", f32), ("lr_t_table", vp), ("step_ctr", vp),
                ("table_len", i32)]


class Slab(C.Structure):
    _fields_ = [("w", vp), ("s0", vp), ("s1", vp), ("part_base", vp), ("V", i64), ("P", i32),
                ("D", i32)]


# name -> (restype, argtypes)
SIGNATURES = {
    "hp_version": (C.c_int, []),
    "hp_last_error": (C.c_char_p, []),
    "hp_device_sm_count": (C.c_int, []),
    "hp_launch_count": (i64, []),
    "hp_debug_set_profile": (None, [vp]),
    "hp_debug_set_cluster_threads": (None, [C.c_int]),
    "hp_debug_set_rowstream": (None, [C.c_int]),
    "hp_debug_set_pdl": (None, [C.c_int]),
    "hp_debug_set_rs_ctas": (None, [C.c_int]),
    "hp_debug_set_owner_stream": (None, [C.c_int]),
    "hp_debug_set_combine_blocks": (None, [C.c_int]),
    "hp_debug_set_reduce_b": (None, [C.c_int]),
    "hp_debug_set_dar_blocks": (None, [C.c_int]),
    "hp_debug_set_dar_buckets": (None, [C.c_int]),
    "hp_debug_set_dar_deep": (None, [C.c_int]),
    "hp_debug_set_dar_tma": (None, [C.c_int]),
    "hp_debug_set_dar_rg_tma": (None, [C.c_int]),
    "hp_debug_set_dar_rg_blocks": (None, [C.c_int]),
    "hp_debug_set_owner_waves": (None, [C.c_int]),
    "hp_debug_set_spans": (None, [vp]),
    "hp_apply_plan": (C.c_int, [vp, i64, Slab, Optim, vp, sz, vp]),
    "hp_apply_plan_build": (C.c_int, [vp, i64, Slab, vp, sz, vp]),
    "hp_dedup_ws_bytes": (sz, [i64, i32, i32, i32]),
    "hp_sort_dedup_route": (C.c_int, [vp, vp, i64, i32, i64, i32, vp, i32, vp, vp, vp, vp, vp, vp,
                                      vp, sz, vp]),
    "hp_dedup_plan": (C.c_int, [vp, i64, i32, i64, i32, vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
    "hp_plan_status": (C.c_int, [vp, vp, vp]),
    "hp_merge_apply": (C.c_int, [vp, vp, i64, Slab, Optim, vp, sz, vp]),
    "hp_local_apply": (C.c_int, [vp, vp, i64, Slab, Optim, vp, sz, vp]),
    "hp_gather_rows": (C.c_int, [Slab, vp, i64, vp, vp, vp]),
    "hp_stitch": (C.c_int, [vp, vp, i64, i32, vp, vp]),
    "hp_init_rows": (C.c_int, [vp, i64, i64, i32, u64, f32, vp]),
    "hp_fill": (C.c_int, [vp, i64, f32, vp]),
    "hp_step_counter_inc": (C.c_int, [vp, vp]),
    "hp_allgather": (C.c_int, [vp, vp, vp, i64, vp]),
    "hp_dense_reduce_bcast": (C.c_int, [vp, vp, vp, i64, i32, f32, i32, vp]),
    "hp_dense_allreduce_scale_cast": (C.c_int, [vp, vp, vp, i64, i32, f32, vp]),
    "hp_dense_allreduce_scale_cast_ex": (C.c_int, [vp, vp, i32, vp, i64, i32, f32, vp, vp]),
    "hp_nccl_unique_id_bytes": (C.c_int, []),
    "hp_nccl_get_unique_id": (C.c_int, [vp]),
    "hp_comm_init": (C.c_int, [C.POINTER(vp), i32, i32, vp]),
    "hp_comm_destroy": (C.c_int, [vp]),
    "hp_comm_size": (C.c_int, [vp]),
    "hp_comm_status": (C.c_int, [vp, vp]),
    "hp_alltoall_counts": (C.c_int, [vp, vp, vp, vp]),
    "hp_exchange_push": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i32, vp]),
    "hp_exchange_pull": (C.c_int, [vp, vp, vp, vp, vp, i32, vp]),
    "hp_xchg_window_bytes": (sz, [i32, i32, i64, i64]),
    "hp_xchg_create": (C.c_int, [C.POINTER(vp), i32, i32, i32, i64, i64, vp, C.POINTER(vp)]),
    "hp_xchg_open_peer": (C.c_int, [vp, i32, vp]),
    "hp_xchg_destroy": (C.c_int, [vp]),
    "hp_xchg_push": (C.c_int, [vp, vp, vp, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
    "hp_xchg_merge_apply": (C.c_int, [vp, Slab, Optim, i32, vp]),
    "hp_xchg_wait": (C.c_int, [vp, i32, vp]),
    "hp_xchg_plan": (C.c_int, [vp, vp, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
    "hp_xchg_push_plan": (C.c_int, [vp, vp, i64, i64, i32, vp, vp, vp, vp, sz, vp, vp]),
    "hp_xchg_stitch": (C.c_int, [vp, vp, i64, vp, i32, vp]),
    "hp_xchg_status": (C.c_int, [vp, vp, vp]),
    "hp_xchg_recv_counts": (C.c_int, [vp, vp, vp]),
    "hp_dar_create": (C.c_int, [C.POINTER(vp), i32, i32, i64, i32, vp, C.POINTER(vp)]),
    "hp_dar_open_peer": (C.c_int, [vp, i32, vp]),
    "hp_dar_destroy": (C.c_int, [vp]),
    "hp_dar_set_mode": (C.c_int, [vp, i32]),
    "hp_dar_set_in_dtype": (C.c_int, [vp, i32]),
    "hp_dar_set_split": (C.c_int, [vp, vp]),
    "hp_nvls_allreduce": (C.c_int, [vp, vp, i64, i32, i32, i32, f32, vp, vp, vp]),
    "hp_dar_allreduce": (C.c_int, [vp, vp, f32, vp]),
    "hp_dar_status": (C.c_int, [vp, vp, vp]),
    "hp_debug_nvlink_bench": (C.c_int, [vp, i32, i32, i32, vp]),
    "hp_debug_fence_bench": (C.c_int, [vp, i32, i32, i32, i32, vp]),
    "hp_xchg_debug_sig": (C.c_int, [vp, vp, vp]),
    "hp_debug_set_wait_timeout": (None, [C.c_longlong]),
    "hp_debug_set_fuse_tree": (None, [C.c_int]),
    "hp_debug_set_split_long": (None, [C.c_int]),
    "hp_debug_set_long_b8": (None, [C.c_int]),
    "hp_debug_set_cbcast": (None, [C.c_int]),
    "hp_debug_set_long_tma": (None, [C.c_int]),
    "hp_debug_set_comb_lite": (None, [C.c_int]),
    "hp_debug_set_reduce_bps": (None, [C.c_int]),
    "hp_debug_set_launch_prio": (None, [C.c_int]),
    "hp_debug_set_bcast_tma": (None, [C.c_int]),
    "hp_graph_instantiate": (C.c_int, [vp, i32, C.POINTER(vp)]),
    "hp_plan_stitch": (C.c_int, [vp, sz, i64, i32, i64, i32, vp, vp, vp]),
    "hp_apply_plan_pull": (C.c_int, [vp, i64, Slab, Optim, vp, vp, sz, vp, vp]),
    "hp_xchg_ret_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "hp_xchg_pull": (C.c_int, [vp, vp, i64, i64, i32, vp, vp, vp, vp]),
    "hp_xchg_stitch_plan": (C.c_int, [vp, vp, sz, i64, i64, i32, vp, i32, vp]),
    "hp_graph_launch": (C.c_int, [vp, vp]),
    "hp_graph_destroy": (C.c_int, [vp]),
    "hp_err_host_alloc": (C.c_int, [i32, C.POINTER(vp), C.POINTER(vp)]),
    "hp_err_host_free": (C.c_int, [vp]),
    "hp_err_collect": (C.c_int, [vp, vp, i32, vp, vp]),
    "hp_plan_err_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "hp_xchg_err_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "hp_xchg_window_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "hp_xchg_set_peer_ptr": (C.c_int, [vp, i32, vp]),
    "hp_dar_err_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "hp_dar_window_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "hp_dar_set_peer_ptr": (C.c_int, [vp, i32, vp]),
}

_lib = None


class HybridPathError(RuntimeError):
    pass


def load() -> C.CDLL:
    """Load (once) and type the library; raises if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise HybridPathError(
            f"{LIB_PATH} not found: build it with `python -m paper_1808_02621_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("HP_LIB") and not hasattr(lib, name):
            continue  # A/B against an older build: tolerate entry points it lacks
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().hp_last_error().decode(errors="replace")
        raise HybridPathError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def symbols() -> list:
    return sorted(SIGNATURES)

"""ctypes binding of libvrgeom.so (include/vrgeom.h).  There is no CPU fallback: every
compute entry point raises if the CUDA extension or a CUDA device is missing."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvrgeom.so")
ABI_VERSION = 4  # VRGEOM_ABI_VERSION of include/vrgeom.h this binding was written against

VR_NAIVE, VR_WARP, VR_SORT, VR_HASH, VR_PHASH = range(5)
STRATEGY_IDS = {"naive": VR_NAIVE, "warp": VR_WARP, "sort": VR_SORT, "hash": VR_HASH, "phash": VR_PHASH}

(VR_OK, VR_ERR_UNKNOWN_STRATEGY, VR_ERR_BAD_BATCH, VR_ERR_TABLE_BELOW_BUDGET, VR_ERR_OVER_BUDGET,
 VR_ERR_HASH_FULL, VR_ERR_WARP_NO_PROGRESS, VR_ERR_WARP_WIDTH, VR_ERR_UNALIGNED, VR_ERR_BAD_CONFIG,
 VR_ERR_UNSUPPORTED, VR_ERR_CUDA, VR_ERR_CAPACITY, VR_ERR_WORKSPACE, VR_ERR_PRIM_OVER_BUDGET,
 VR_ERR_VERTEX_RANGE) = range(16)

VR_FLAG_NO_BUDGET = 0x100
VR_FLAG_CONTIGUOUS = 0x200
VR_FLAG_STATIC = 0x400
VR_FLAG_NO_FUSE = 0x800

VR_SHADER_NONE, VR_SHADER_IDENTITY, VR_SHADER_POSITION = range(3)

(VR_STAT_INDICES, VR_STAT_INVOCATIONS, VR_STAT_BATCHES, VR_STAT_ROUNDS, VR_STAT_PROBES_FAST,
 VR_STAT_PROBES_SLOW, VR_STAT_PROBE_MAX_CHAIN, VR_STAT_ERROR) = range(8)
VR_STATS_WORDS = 16
VR_PROFILE_STAGES = 4
PROFILE_STAGE_NAMES = ("init", "dedup", "offset_scan", "shade_finalize")
# vr_last_kernel_path() values that are ONE kernel for dedup + output offsets + shading
KERNEL_PATH_NAMES = {
    2: "fused static warp kernel (dedup + look-back + shade)",
    3: "persistent tile kernel (stage + dedup + decoupled look-back/shade)",
}


class NativeLibraryError(RuntimeError):
    """libvrgeom.so is missing or no CUDA device is visible."""


class BatchConfigC(C.Structure):
    _fields_ = [("batch_size", C.c_int32), ("max_unique", C.c_int32), ("max_indices", C.c_int32),
                ("warp_width", C.c_int32), ("block_size", C.c_int32), ("primitive_size", C.c_int32)]


class HashConfigC(C.Structure):
    _fields_ = [("table_size", C.c_uint32), ("multiplier", C.c_uint32), ("max_fast_probes", C.c_uint32)]


class ShaderC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("has_matrix", C.c_int32), ("matrix", C.c_float * 16),
                ("d_positions4", C.c_void_p), ("d_attributes", C.c_void_p), ("attr_words", C.c_int32),
                ("vertex_count", C.c_int32), ("d_batch_vertex_base", C.c_void_p), ("extra_cycles", C.c_int32)]


class OutputsC(C.Structure):
    _fields_ = [("d_batch_round_off", C.c_void_p), ("d_round_uid_off", C.c_void_p),
                ("d_round_prims", C.c_void_p), ("d_unique_ids", C.c_void_p),
                ("d_assembly_map", C.c_void_p), ("d_shaded4", C.c_void_p),
                ("d_shaded_attr", C.c_void_p), ("d_shade_counts", C.c_void_p), ("d_stats", C.c_void_p),
                ("cap_unique", C.c_int64), ("cap_rounds", C.c_int64), ("d_stream_xyz", C.c_void_p)]


class CacheConfigC(C.Structure):
    _fields_ = [("num_processors", C.c_int32), ("wave_width", C.c_int32), ("capacity", C.c_int32),
                ("primitive_size", C.c_int32)]


VR_WALK_MAX_GAUSSIANS = 8


class WalkConfigC(C.Structure):
    _fields_ = [("grid_w", C.c_int32), ("grid_h", C.c_int32), ("max_move_distance", C.c_int32),
                ("kept_moves", C.c_int32), ("n_gaussians", C.c_int32), ("reserved", C.c_int32),
                ("gaussians", (C.c_double * 4) * VR_WALK_MAX_GAUSSIANS)]


_lib = None

_SIGNATURES = {
    "vr_abi_version": (C.c_int, []),
    "vr_status_string": (C.c_char_p, [C.c_int]),
    "vr_device_count": (C.c_int, []),
    "vr_check_batch_config": (C.c_int, [C.POINTER(BatchConfigC)]),
    "vr_check_hash_config": (C.c_int, [C.POINTER(HashConfigC)]),
    "vr_static_batch_count": (C.c_int64, [C.c_int64, C.POINTER(BatchConfigC)]),
    "vr_static_offsets": (C.c_int, [C.c_int64, C.POINTER(BatchConfigC), C.c_void_p, C.c_void_p]),
    "vr_dynamic_workspace_bytes": (C.c_size_t, [C.c_int64, C.POINTER(BatchConfigC)]),
    "vr_dynamic_batches": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(BatchConfigC), C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_dynamic_batches_draws": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(BatchConfigC), C.c_void_p, C.c_int32,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_dynamic_group_count": (C.c_int64, [C.c_int64, C.POINTER(BatchConfigC)]),
    "vr_dynamic_group_indices": (C.c_int64, [C.POINTER(BatchConfigC)]),
    "vr_dynamic_table_words": (C.c_int64, [C.c_int64, C.POINTER(BatchConfigC)]),
    "vr_dynamic_range_tables": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(BatchConfigC), C.c_int64, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_dynamic_range_offsets": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(BatchConfigC), C.c_int64, C.c_int64, C.c_void_p,
                                           C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_batch_vertex_base": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                       C.c_void_p]),
    "vr_output_bounds": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.POINTER(BatchConfigC),
                                   C.POINTER(HashConfigC), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "vr_run_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int64, C.c_int64, C.POINTER(BatchConfigC),
                                            C.POINTER(HashConfigC)]),
    "vr_run": (C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                         C.c_int32, C.POINTER(BatchConfigC), C.POINTER(HashConfigC), C.POINTER(ShaderC),
                         C.POINTER(OutputsC), C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_dynamic_batch_bound": (C.c_int64, [C.c_int64, C.POINTER(BatchConfigC), C.c_int32]),
    "vr_run_counted": (C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                 C.POINTER(BatchConfigC), C.POINTER(HashConfigC), C.POINTER(ShaderC), C.POINTER(OutputsC),
                                 C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_profile_enable": (C.c_int, [C.c_int]),
    "vr_last_launch_count": (C.c_int, []),
    "vr_last_kernel_path": (C.c_int, []),
    "vr_debug_reload_knobs": (C.c_int, []),
    "vr_profile_read": (C.c_int, [C.POINTER(C.c_float), C.c_int]),
    "vr_expand_stream": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_pack_xyz": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vr_pack_bytes": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vr_expand_sources": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_ideal_counts": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vr_cache_workspace_bytes": (C.c_size_t, [C.c_int64, C.POINTER(CacheConfigC)]),
    "vr_simulate_cache": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(CacheConfigC), C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_size_t, C.c_void_p]),
    "vr_walk_likelihoods": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(WalkConfigC), C.c_void_p, C.c_void_p, C.c_void_p]),
    "vr_walk_advance": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_uint64, C.c_int64,
                                  C.c_void_p, C.c_void_p]),
    "vr_walk_pack": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
}


def exported_symbols():
    """Every entry point include/vrgeom.h declares."""
    return tuple(_SIGNATURES)


def lib():
    """Load libvrgeom.so (built in-tree by __graft_entry__.build()).  Raises loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`; "
                "this package has no CPU fallback")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.vr_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libvrgeom.so ABI version mismatch")
        _lib = handle
    return _lib


def require_cuda():
    """The hot path runs on a B200 or not at all."""
    handle = lib()
    if handle.vr_device_count() < 1:
        raise NativeLibraryError("no CUDA device visible: the geometry stage has no CPU fallback")
    return handle


def status_string(status: int) -> str:
    return lib().vr_status_string(status).decode()

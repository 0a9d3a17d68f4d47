"""ctypes binding of the C-ABI in include/wgpf.h (libwgpf.so, sm_100a).

Loading fails loudly when the library cannot be built or loaded, and context
creation fails when no CUDA device is present: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _build

HIST_BINS = 64

EVENT_DTYPE = np.dtype(
    [("start", "<u8"), ("end", "<u8"), ("region", "<u4"), ("iteration", "<u4"),
     ("block_index", "<u4"), ("warp_group", "<u4")])
RECORD_DTYPE = np.dtype([("tag", "<u4"), ("payload", "<u4")])
INTERVAL_DTYPE = np.dtype([("region_id", "<u4"), ("iteration", "<u4"),
                           ("start", "<u8"), ("end", "<u8"),
                           ("start_pos", "<u8"), ("end_pos", "<u8")])
DECODED_DTYPE = np.dtype([("block_index", "<u4"), ("warp_group", "<u4"),
                          ("dropped_records", "<u4"), ("pad", "<u4"),
                          ("offset", "<u8"), ("count", "<u8")])

EV_WAIT = 0x80000000
EV_CORRECTED = 0x40000000
EV_REGION_MASK = 0x7FFFF

F_STATS_ONLY = 0x1
F_EXACT_MEAN = 0x2
F_FORCE_GENERAL = 0x4
F_NO_STATS = 0x8

OK, E_BUFFER = 0, 12


class Warnings(C.Structure):
    _fields_ = [("dropped_heads", C.c_uint32), ("truncated_tails", C.c_uint32),
                ("flagged_preconditions", C.c_uint32),
                ("malformed_groups", C.c_uint32)]


class RegionStat(C.Structure):
    _fields_ = [("label", C.c_char_p), ("warp_group", C.c_uint32),
                ("kind", C.c_uint32), ("count", C.c_uint64), ("min", C.c_uint64),
                ("max", C.c_uint64), ("sum", C.c_uint64), ("mean", C.c_double),
                ("first_event", C.c_uint64), ("hist", C.c_uint64 * HIST_BINS)]


class Profile(C.Structure):
    _fields_ = [("count_ms", C.c_float), ("scan_ms", C.c_float),
                ("emit_ms", C.c_float), ("general_ms", C.c_float),
                ("finalize_ms", C.c_float), ("total_ms", C.c_float),
                ("launches", C.c_uint32), ("general_streams", C.c_uint32),
                ("overlap_chunks", C.c_uint32), ("reserved", C.c_uint32)]


class CpStage(C.Structure):
    _fields_ = [("label", C.c_char_p), ("mean", C.c_uint64), ("steady", C.c_uint64),
                ("warp_group", C.c_uint32), ("pad", C.c_uint32)]


class Overlap(C.Structure):
    _fields_ = [("blocks", C.c_uint64), ("span", C.c_uint64),
                ("busy", C.c_uint64 * 2), ("both", C.c_uint64),
                ("bubble", C.c_uint64 * 2)]


F_PROFILE = 0x10


class ScopeOp(C.Structure):
    _fields_ = [("op", C.c_uint32), ("pad", C.c_uint32), ("trips", C.c_uint64),
                ("label", C.c_char_p)]


class LowerCfg(C.Structure):
    _fields_ = [("name", C.c_char_p), ("strategy", C.c_uint32),
                ("signature_bits", C.c_int), ("iteration_signature", C.c_int),
                ("global_buffer", C.c_int), ("slots_total", C.c_uint64),
                ("smem_capacity", C.c_uint64)]


class Lowered(C.Structure):
    _fields_ = [("slots_per_stream", C.c_uint64), ("smem_bytes_per_cta", C.c_uint64),
                ("n_regions", C.c_uint32), ("pad", C.c_uint32)]


OP_START, OP_END, OP_LOOP, OP_ENDLOOP = 0, 1, 2, 3

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Loads (building if needed) libwgpf.so."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # WGPF_LIB_OVERRIDE: an alternative build of the same ABI (A/B runs)
        path = os.environ.get("WGPF_LIB_OVERRIDE") or _build.build()
        L = C.CDLL(path)
        vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
        sig = {
            "wgpf_abi_version": ([], i32),
            "wgpf_create": ([i32, vp, C.POINTER(vp)], i32),
            "wgpf_destroy": ([vp], None),
            "wgpf_set_stream": ([vp, vp], i32),
            "wgpf_last_error": ([vp], C.c_char_p),
            "wgpf_error_category": ([i32], C.c_char_p),
            "wgpf_set_plan": ([vp, u64, u32, C.POINTER(C.c_char_p), u32], i32),
            "wgpf_replay_device": ([vp, vp, u64, u64, u64, u64, vp, u64, u32,
                                    C.POINTER(u64), C.POINTER(Warnings)], i32),
            "wgpf_replay_image": ([vp, vp, u64, u64, vp, u64, u32, C.POINTER(u64),
                                   C.POINTER(Warnings)], i32),
            "wgpf_decode_image": ([vp, vp, u64, vp, u64, C.POINTER(u64), vp, u64,
                                   C.POINTER(u64)], i32),
            "wgpf_unwrap_clock": ([vp, vp, u64, vp], i32),
            "wgpf_pair_records": ([vp, vp, u64, vp, u64, C.POINTER(u64),
                                   C.POINTER(u32), C.POINTER(u32)], i32),
            "wgpf_replay_intervals": ([vp, vp, u64, u32, u32, u64, vp, u64,
                                       C.POINTER(u64), C.POINTER(Warnings)], i32),
            "wgpf_stats_get": ([vp, C.POINTER(RegionStat), u32, C.POINTER(u32)], i32),
            "wgpf_region_stats": ([vp, vp, u64, i32, u32, C.POINTER(RegionStat), u32,
                                   C.POINTER(u32)], i32),
            "wgpf_stats_packed_bytes": ([vp], u64),
            "wgpf_stats_export": ([vp, vp], i32),
            "wgpf_stats_merge": ([vp, vp, u32], i32),
            "wgpf_synth_body": ([vp, vp, u32, u64, u64, u64], i32),
            "wgpf_last_profile": ([vp, C.POINTER(Profile)], i32),
            "wgpf_critical_path": ([vp, vp, u64, i32, C.POINTER(C.c_char_p),
                                    C.POINTER(C.c_char_p), u32, u64, i32, i32,
                                    C.POINTER(CpStage), u32, C.POINTER(u32),
                                    C.POINTER(u64), u64, C.POINTER(u32), u32,
                                    C.POINTER(u32), C.POINTER(u64)], i32),
            "wgpf_export_chrome_trace": ([vp, vp, u64, i32, C.c_double, vp, u64,
                                          C.POINTER(u64)], i32),
            "wgpf_overlap_counters": ([vp, vp, u64, i32, vp, u32,
                                       C.POINTER(Overlap)], i32),
            "wgpf_profile_bytes": ([u64, u32, u64], u64),
            "wgpf_allreduce_stats": ([vp, vp], i32),
            "wgpf_align_events": ([vp, vp, u64, i32, vp, u64, C.c_double,
                                   C.POINTER(C.c_double)], i32),
            "wgpf_collect": ([vp, vp, u64, vp, vp, u64, C.POINTER(u64)], i32),
            "wgpf_lower_scopes": ([C.POINTER(ScopeOp), C.POINTER(u32), u32,
                                   C.POINTER(LowerCfg), C.POINTER(u32),
                                   C.POINTER(Lowered), C.c_char_p, u64], i32),
        }
        override = bool(os.environ.get("WGPF_LIB_OVERRIDE"))
        for name, (args, res) in sig.items():
            if override and not hasattr(L, name):
                continue  # (an older build under A/B: entry points it lacks)
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def loaded_path() -> str:
    return _build.LIB


def ptr(a) -> int:
    """Address of a numpy array / torch tensor / int."""
    if a is None:
        return 0
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"cannot take the address of {type(a)}")

"""P1 -- the device instrumentation runtime (include/wgpf_device.cuh) and its
workloads: a scope-program self-test, the per-record cost microbenchmark and
the instrumented tcgen05/TMA bf16 GEMM (config 2).  Thin ctypes layer over
libwgpf_p1.so; the profile buffers these kernels leave in HBM are KPFT bodies
that the P2 decoder (trace.Context.replay_device) reads in place.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _build

_lib = None

# scope-program self-test regions (csrc_p1/p1_selftest.cu)
SELFTEST_LABELS = ["kernel", "outer", "inner", "async", "async.wait"]
# GEMM scopes (csrc_p1/gemm_tcgen05.cu)
GEMM_LABELS = ["tile", "tma.stall", "tma.issue", "mma.stall", "mma.issue",
               "epi.stall", "epi.ld", "epi.st"]
GEMM_WARPS = 6
GEMM_SLOTS = 64
# attention scopes (csrc_p1/attn_tcgen05.cu), the fa3 fixture's names
ATTN_LABELS = ["Load K", "Load K.wait", "Load V", "Load V.wait",
               "GEMM0.c0", "GEMM0.c0.wait", "Softmax.c0", "GEMM1.c0",
               "GEMM0.c1", "GEMM0.c1.wait", "Softmax.c1", "GEMM1.c1"]
ATTN_WARPS = 10          # stream = warp: 0 K producer, 1 V producer, 2-5 c0, 6-9 c1
ATTN_SLOTS = 64
ATTN_ROLE_OF_WARP = [0, 0] + [1] * 8  # producer / consumer roles (overlap counters)
# barrier edges of the attention kernel (perfmodel.hpp:258-313 derives them
# from the program's arrive/wait pairs): a landed tile gates the consumer
# GEMM that reads it; a consumed tile frees the slot the next load fills.
ATTN_BARRIER_EDGES = [("Load K.wait", "GEMM0.c0"), ("Load K.wait", "GEMM0.c1"),
                      ("Load V.wait", "GEMM1.c0"), ("Load V.wait", "GEMM1.c1"),
                      ("GEMM0.c0.wait", "Load K"), ("GEMM0.c1.wait", "Load K"),
                      ("GEMM0.c0.wait", "Load V"), ("GEMM0.c1.wait", "Load V")]
CTA_TIMING_DTYPE = np.dtype([("smid", "<u4"), ("streams", "<u4"),
                             ("gt_start", "<u8"), ("gt_end", "<u8"),
                             ("clk_start", "<u4"), ("clk_end", "<u4")])


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        # WGPF_P1_LIB_OVERRIDE: an alternative build of the same ABI (A/B runs)
        L = C.CDLL(os.environ.get("WGPF_P1_LIB_OVERRIDE") or _build.build_p1())
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        L.wgpf_p1_selftest.argtypes = [vp, u32, u32, u32, u32, vp, vp]
        L.wgpf_p1_selftest.restype = i32
        L.wgpf_p1_selftest_auto.argtypes = [vp, u32, u32, u32, u32, vp]
        L.wgpf_p1_selftest_auto.restype = i32
        L.wgpf_p1_selftest_capi.argtypes = [vp, u32, u32, u32, u32, vp]
        L.wgpf_p1_selftest_capi.restype = i32
        L.wgpf_p1_record_cost.argtypes = [u32, u32, i32, vp, vp]
        L.wgpf_p1_record_cost.restype = i32
        L.wgpf_p1_flush_cost.argtypes = [u32, u32, u32, i32, vp, vp, vp]
        L.wgpf_p1_flush_cost.restype = i32
        L.wgpf_gemm_bf16.argtypes = [vp, vp, vp, u32, u32, u32, i32, vp, vp, vp]
        L.wgpf_gemm_bf16.restype = i32
        L.wgpf_gemm_profile_bytes.argtypes = [u32, u32]
        L.wgpf_gemm_profile_bytes.restype = u64
        L.wgpf_gemm_ctas.argtypes = [u32, u32]
        L.wgpf_gemm_ctas.restype = u32
        L.wgpf_gemm_smem_bytes.argtypes = [i32]
        L.wgpf_gemm_smem_bytes.restype = u32
        L.wgpf_attn_bf16.argtypes = [vp, vp, vp, vp, u32, u32, C.c_float, i32, i32,
                                     vp, vp, vp]
        L.wgpf_attn_bf16.restype = i32
        L.wgpf_attn_profile_bytes.argtypes = [u32, u32]
        L.wgpf_attn_profile_bytes.restype = u64
        L.wgpf_attn_smem_bytes.argtypes = [i32, i32]
        L.wgpf_attn_smem_bytes.restype = u32
        L.wgpf_p1_run_program.argtypes = [vp, u32, u32, u32, i32, i32, u32, vp, vp, vp,
                                          vp]
        L.wgpf_p1_run_program.restype = i32
        L.wgpf_p1_loop_entry.argtypes = [u32, u32, u32, i32, vp, vp]
        L.wgpf_p1_accuracy.argtypes = [u32, u32, u32, u32, i32, vp, u32, vp, vp, u32, vp]
        L.wgpf_p1_accuracy.restype = i32
        L.wgpf_p1_loop_entry.restype = i32
        _lib = L
    return _lib


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed (status {rc})")


def stream_stride(cap: int) -> int:
    return 16 + 8 * cap


def selftest(profile_ptr: int, ctas: int, warps: int, cap: int, iters: int,
             timing_ptr: int = 0, stream: int = 0) -> None:
    _check(lib().wgpf_p1_selftest(C.c_void_p(profile_ptr), ctas, warps, cap, iters,
                                  C.c_void_p(timing_ptr), C.c_void_p(stream)),
           "wgpf_p1_selftest")


def selftest_auto(profile_ptr: int, ctas: int, warps: int, cap: int, iters: int,
                  stream: int = 0) -> None:
    """The selftest program instrumented through the device pass helpers
    (wgpf_dev::Scope / AsyncOp, include/wgpf_device.cuh)."""
    _check(lib().wgpf_p1_selftest_auto(C.c_void_p(profile_ptr), ctas, warps, cap, iters,
                                       C.c_void_p(stream)), "wgpf_p1_selftest_auto")


def selftest_capi(profile_ptr: int, ctas: int, warps: int, cap: int, iters: int,
                  stream: int = 0) -> None:
    """The selftest program through the C-style device API (wgpf_init /
    wgpf_record_op / wgpf_finalize, include/wgpf_device.cuh)."""
    _check(lib().wgpf_p1_selftest_capi(C.c_void_p(profile_ptr), ctas, warps, cap, iters,
                                       C.c_void_p(stream)), "wgpf_p1_selftest_capi")


def selftest_store_log(iters: int) -> list:
    """The (start, region) sequence one warp stores (vgpu.hpp:269-271)."""
    k, o, i, a, w = range(5)
    log = [(1, k)]
    for _ in range(iters):
        log += [(1, o), (1, i), (0, i), (0, o), (1, a), (0, a), (1, w), (0, w)]
    log.append((0, k))
    return log


def flush_cost(ctas: int, threads: int, nbytes: int, bulk: bool, profile_ptr: int,
               cycles_ptr: int, stream: int = 0) -> None:
    """FinalizeOp cost microbenchmark (csrc_p1/p1_selftest.cu k_flush_cost):
    cycles per CTA to copy an nbytes profile buffer out with vector stores or
    one cp.async.bulk."""
    _check(lib().wgpf_p1_flush_cost(ctas, threads, nbytes, int(bulk), C.c_void_p(profile_ptr),
                                    C.c_void_p(cycles_ptr), C.c_void_p(stream)),
           "wgpf_p1_flush_cost")


def record_cost(n: int, warps: int, record: bool, cycles_ptr: int,
                stream: int = 0) -> None:
    _check(lib().wgpf_p1_record_cost(n, warps, int(record), C.c_void_p(cycles_ptr),
                                     C.c_void_p(stream)), "wgpf_p1_record_cost")


def gemm(a_ptr: int, b_ptr: int, c_ptr: int, M: int, N: int, K: int,
         instrument: bool = False, profile_ptr: int = 0, timing_ptr: int = 0,
         stream: int = 0) -> None:
    _check(lib().wgpf_gemm_bf16(C.c_void_p(a_ptr), C.c_void_p(b_ptr),
                                C.c_void_p(c_ptr), M, N, K, int(instrument),
                                C.c_void_p(profile_ptr), C.c_void_p(timing_ptr),
                                C.c_void_p(stream)), "wgpf_gemm_bf16")


def gemm_profile_bytes(M: int, N: int) -> int:
    return int(lib().wgpf_gemm_profile_bytes(M, N))


def gemm_ctas(M: int, N: int) -> int:
    """CTAs of the persistent GEMM grid (min(tiles, SMs)); one profile
    segment of GEMM_WARPS streams each."""
    return int(lib().wgpf_gemm_ctas(M, N))


def gemm_smem_bytes(instrument: bool) -> int:
    return int(lib().wgpf_gemm_smem_bytes(int(instrument)))


def attention(q_ptr: int, k_ptr: int, v_ptr: int, o_ptr: int, BH: int, S: int,
              scale: float = 0.0, kv_stages: int = 2, instrument: bool = False,
              profile_ptr: int = 0, timing_ptr: int = 0, stream: int = 0) -> None:
    """O = softmax(Q K^T scale) V, bf16 [BH, S, 128]; S % 256 == 0."""
    _check(lib().wgpf_attn_bf16(C.c_void_p(q_ptr), C.c_void_p(k_ptr), C.c_void_p(v_ptr),
                                C.c_void_p(o_ptr), BH, S, scale, kv_stages,
                                int(instrument), C.c_void_p(profile_ptr),
                                C.c_void_p(timing_ptr), C.c_void_p(stream)),
           "wgpf_attn_bf16")


def attn_profile_bytes(BH: int, S: int) -> int:
    return int(lib().wgpf_attn_profile_bytes(BH, S))


def attn_smem_bytes(instrument: bool, kv_stages: int = 2) -> int:
    return int(lib().wgpf_attn_smem_bytes(int(instrument), kv_stages))


def kpft_v2(body: bytes | np.ndarray, n_streams: int) -> bytes:
    """wgpf_collect: a KPFT v2 header in front of a flushed device body."""
    b = body.tobytes() if isinstance(body, np.ndarray) else bytes(body)
    return b"KPFT" + struct.pack("<HHQ", 2, 0, n_streams) + b


def kpft_v1(body: bytes | np.ndarray, n_streams: int) -> bytes:
    assert n_streams <= 0xFFFF
    b = body.tobytes() if isinstance(body, np.ndarray) else bytes(body)
    return b"KPFT" + struct.pack("<HH", 1, n_streams) + b


# ---- buffer planning (lower.hpp:142-188) --------------------------------------

def _pow2_floor(v: int) -> int:
    p = 1
    while p * 2 <= v:
        p *= 2
    return p


def plan_slots(num_regions: int, trip_counts, num_warp_groups: int, strategy,
               capacity_bytes: int):
    """plan_slots: slots per stream (warp group) of a device buffer of
    capacity_bytes without a concrete program.  Flush: two records per region
    per iteration (iterations = product of the nonzero trip counts) spread over
    the streams, rejected with a capacity-error when they do not fit; circular:
    the largest power of two that fits.  Returns a BufferPlan with no labels."""
    from .trace import BufferPlan, BufferStrategy, Error, ErrorKind
    M64 = (1 << 64) - 1
    if num_regions == 0 or num_warp_groups == 0:
        raise Error(ErrorKind.Lower, "plan_slots: inputs must be positive")
    iters = 1
    for t in trip_counts:
        iters = (iters * (t if t else 1)) & M64
    strategy = BufferStrategy(strategy)
    if strategy == BufferStrategy.Flush:
        total = (2 * num_regions * iters) & M64
        per = max(1, ((total + num_warp_groups - 1) & M64) // num_warp_groups)
        need = (per * num_warp_groups * 8) & M64
        if need > capacity_bytes:
            raise Error(ErrorKind.Capacity,
                        f"flush sizing needs {need} bytes, capacity is {capacity_bytes}")
        return BufferPlan(per, strategy, [])
    slots = capacity_bytes // (8 * num_warp_groups)
    if slots == 0:
        raise Error(ErrorKind.Capacity, "circular sizing: capacity too small for one "
                    "slot per warp group")
    return BufferPlan(_pow2_floor(slots), strategy, [])


def signature_for(wg: int) -> int:
    """MachineConfig::signature_for (vgpu.hpp:39-45), packed (trace.hpp:42-46):
    the 12 signature bits of stream wg's tags (wgpf_dev::signature_for)."""
    return (wg % 32) | (((wg // 32) % 16) << 5) | (((wg // 512) % 8) << 9)


# ---- lowering of a scope program (lower.hpp:220-301) ---------------------------

@dataclass
class ScopePlan:
    """lower()'s result for a scope program: the BufferPlan fields and, per
    body, the dense region id of every op (None for loop ops)."""
    slots_per_stream: int
    labels: list
    region_ids: list
    smem_bytes_per_cta: int


def _scope_ops(bodies):
    from . import _lib as L
    flat, lens, keep = [], [], []
    for body in bodies:
        lens.append(len(body))
        for o in body:
            kind = o[0]
            if kind in ("start", "end"):
                lab = o[1].encode()
                keep.append(lab)
                flat.append(L.ScopeOp(L.OP_START if kind == "start" else L.OP_END, 0, 0,
                                      lab))
            elif kind == "loop":
                flat.append(L.ScopeOp(L.OP_LOOP, 0, int(o[1]), None))
            elif kind == "endloop":
                flat.append(L.ScopeOp(L.OP_ENDLOOP, 0, 0, None))
            else:
                raise ValueError(f"unknown scope op {o!r}")
    return flat, lens, keep


def lower_scopes(bodies, strategy, smem_capacity: int, slots_total: int = 0,
                 signature_bits: bool = False, iteration_signature: bool = False,
                 global_buffer: bool = False, name: str = "kernel") -> ScopePlan:
    """lower() of a scope program (C-ABI wgpf_lower_scopes): bodies[k] is
    stream role k's op list -- ("start", label), ("end", label),
    ("loop", trips), ("endloop",).  Raises trace.Error with the reference's
    kind and message (ir.hpp:347-390 loop checks, instrument.hpp:60-105
    pairing, lower.hpp:223-279 configuration, ids, slots, smem budget)."""
    from . import _lib as L
    from .trace import BufferStrategy, Error, ErrorKind
    flat, lens, _keep = _scope_ops(bodies)
    n = len(flat)
    ops = (L.ScopeOp * max(1, n))(*flat)
    blen = (C.c_uint32 * max(1, len(lens)))(*lens)
    rid = (C.c_uint32 * max(1, n))()
    cfg = L.LowerCfg(name.encode(), int(BufferStrategy(strategy)), int(signature_bits),
                     int(iteration_signature), int(global_buffer), slots_total,
                     smem_capacity)
    out = L.Lowered()
    err = C.create_string_buffer(1024)
    rc = L.lib().wgpf_lower_scopes(ops, blen, len(lens), C.byref(cfg), rid, C.byref(out),
                                   err, 1024)
    if rc != 0:
        if 1 <= rc <= 9:
            raise Error(ErrorKind(rc - 1), err.value.decode())
        raise RuntimeError(err.value.decode())
    labels = [None] * out.n_regions
    per_body, k = [], 0
    for body in bodies:
        ids = []
        for o in body:
            r = rid[k]
            k += 1
            if o[0] in ("start", "end"):
                labels[r] = o[1]
                ids.append(r)
            else:
                ids.append(None)
        per_body.append(ids)
    return ScopePlan(out.slots_per_stream, labels, per_body, out.smem_bytes_per_cta)


# device interpreter ops (csrc_p1/p1_selftest.cu k_program)
PROG_START, PROG_END, PROG_LOOP, PROG_ENDLOOP, PROG_BUSY = 0, 1, 2, 3, 4
SIG_NONE, SIG_HW, SIG_ITER = 0, 1, 2


def program_encoding(bodies, plan: ScopePlan, busy: int = 0):
    """(ops u32[n, 2], body offsets u32[n_bodies + 1]) of a lowered scope
    program for the device interpreter; `busy` inserts that many ALU steps
    after every record (so scopes have a duration)."""
    ops, offs = [], [0]
    for body, ids in zip(bodies, plan.region_ids):
        for o, r in zip(body, ids):
            if o[0] == "start":
                ops.append((PROG_START, r))
            elif o[0] == "end":
                ops.append((PROG_END, r))
            elif o[0] == "loop":
                ops.append((PROG_LOOP, int(o[1])))
            else:
                ops.append((PROG_ENDLOOP, 0))
            if busy and o[0] in ("start", "end"):
                ops.append((PROG_BUSY, busy))
        offs.append(len(ops))
    return (np.array(ops, np.uint32).reshape(-1, 2), np.array(offs, np.uint32))


def run_program(profile_ptr: int, ctas: int, n_bodies: int, cap: int, flush: bool,
                validate: bool, sig_mode: int, d_ops_ptr: int, d_offs_ptr: int,
                d_err_ptr: int = 0, stream: int = 0) -> None:
    """Runs a lowered scope program on the device: every CTA runs one warp per
    body through wgpf_dev::Recorder<pow2, flush, validate> (loops through
    wgpf_dev::Loop), then flushes its buffer (a KPFT body segment)."""
    _check(lib().wgpf_p1_run_program(C.c_void_p(profile_ptr), ctas, n_bodies, cap,
                                     int(flush), int(validate), sig_mode,
                                     C.c_void_p(d_ops_ptr), C.c_void_p(d_offs_ptr),
                                     C.c_void_p(d_err_ptr), C.c_void_p(stream)),
           "wgpf_p1_run_program")


def loop_entry_cycles(n: int, trips: int, warps: int, record: bool, cycles_ptr: int,
                      stream: int = 0) -> None:
    """Loop-entry microbenchmark (vgpu.hpp:366-369): per-warp cycles of n
    entries of an inner loop of `trips` iterations, with or without a
    START/END pair in the inner body (csrc_p1/p1_selftest.cu k_loop_entry)."""
    _check(lib().wgpf_p1_loop_entry(n, trips, warps, int(record), C.c_void_p(cycles_ptr),
                                    C.c_void_p(stream)), "wgpf_p1_loop_entry")


def loop_entry_cost(n: int = 1 << 14, warps: int = 4) -> dict:
    """Per-entry cost of entering an instrumented loop, in cycles: E = 2 (T(n,
    1) - T(n/2, 2)) / n per variant; the instrumentation's loop-entry cost is
    E(records) - E(plain) (the reference charges 5, vgpu.hpp:366-369)."""
    import torch
    out = {}
    for rec in (False, True):
        t = []
        for (m, trips) in ((n, 1), (n // 2, 2)):
            c = torch.zeros(warps, dtype=torch.int64, device="cuda")
            loop_entry_cycles(m, trips, warps, rec, c.data_ptr())
            loop_entry_cycles(m, trips, warps, rec, c.data_ptr())
            torch.cuda.synchronize()
            t.append(c.double().mean().item())
        out["records" if rec else "plain"] = {
            "entry": 2 * (t[0] - t[1]) / n, "body": (2 * t[1] - t[0]) / n}
    out["loop_entry_cost_cycles"] = out["records"]["entry"] - out["plain"]["entry"]
    out["record_pair_cycles_in_loop"] = out["records"]["body"] - out["plain"]["body"]
    return out

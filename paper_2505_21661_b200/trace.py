"""Python mirror of the reference's trace API (namespace ``wgprof``,
/root/reference/proj/include/wgprof/trace.hpp + pipeline.hpp), backed by the
sm_100a kernels through the C-ABI (include/wgpf.h).

Same names, argument meaning and error behaviour as the reference:

    ProfileRecord, encode_record, decode_record      trace.hpp:58-99
    TraceStream, GlobalTraceImage,
    serialize_image, deserialize_image              trace.hpp:105-209
    BufferPlan, BufferStrategy                       lower.hpp:42,57-73
    decode_image                                     trace.hpp:222-251  (GPU)
    unwrap_clock                                     trace.hpp:257-272  (GPU)
    pair_records                                     trace.hpp:294-346  (GPU)
    replay                                           trace.hpp:398-487  (GPU)
    replay_image                                     pipeline.hpp:66-81 (GPU)
    region_stats                                     pipeline.hpp:114-133 (GPU)
    Error / ErrorKind                                error.hpp:8-55

Events are returned as numpy structured arrays of the 32-byte ``wgpf_event``
(label replaced by the region id); ``TraceReplay.timeline()`` converts small
results to ``TimelineEvent`` objects with label strings.
"""
from __future__ import annotations

import ctypes as C
import enum
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import (EV_CORRECTED, EV_REGION_MASK, EV_WAIT, EVENT_DTYPE,
                   INTERVAL_DTYPE, RECORD_DTYPE)

START_FLAG = 0x80000000
SIGNATURE_MASK = 0xFFF
MAX_REGIONS = 1 << 19
TRACE_VERSION = 1
TRACE_MAGIC = b"KPFT"
WAIT_SUFFIX = ".wait"


# ---------------------------------------------------------------------------
# errors (error.hpp)
# ---------------------------------------------------------------------------


class ErrorKind(enum.IntEnum):
    Parse = 0
    Validate = 1
    Instrument = 2
    Lower = 3
    Capacity = 4
    Deadlock = 5
    Trace = 6
    Config = 7
    Io = 8


_CATEGORY = {ErrorKind.Parse: "parse-error", ErrorKind.Validate: "validate-error",
             ErrorKind.Instrument: "instrument-error",
             ErrorKind.Lower: "lower-error", ErrorKind.Capacity: "capacity-error",
             ErrorKind.Deadlock: "simulation-deadlock",
             ErrorKind.Trace: "trace-error", ErrorKind.Config: "config-error",
             ErrorKind.Io: "io-error"}


class Error(RuntimeError):
    """wgprof::Error(kind, message); category() is the CLI token."""

    def __init__(self, kind, message: str):
        super().__init__(message)
        self.kind = kind

    def category(self) -> str:
        if isinstance(self.kind, ErrorKind):
            return _CATEGORY[self.kind]
        return str(self.kind)


class BufferTooSmall(RuntimeError):
    def __init__(self, needed: int, message: str):
        super().__init__(message)
        self.needed = needed


def _check(ctx, rc: int, needed: int = 0) -> None:
    if rc == L.OK:
        return
    msg = L.lib().wgpf_last_error(ctx).decode()
    if 1 <= rc <= 9:
        raise Error(ErrorKind(rc - 1), msg)
    if rc == L.E_BUFFER:
        raise BufferTooSmall(needed, msg)
    raise RuntimeError(f"wgpf: {L.lib().wgpf_error_category(rc).decode()}: {msg}")


# ---------------------------------------------------------------------------
# records and images (format helpers, host side)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Signature:
    wave_slot_id: int = 0
    simd_id: int = 0
    pipe_id: int = 0

    def packed(self) -> int:
        return ((self.wave_slot_id & 0x1F) | ((self.simd_id & 0xF) << 5) |
                ((self.pipe_id & 0x7) << 9))

    @staticmethod
    def unpack(bits: int) -> "Signature":
        return Signature(bits & 0x1F, (bits >> 5) & 0xF, (bits >> 9) & 0x7)


@dataclass(frozen=True)
class ProfileRecord:
    tag: int = 0
    payload: int = 0

    def is_start(self) -> bool:
        return (self.tag & START_FLAG) != 0

    def region_id(self) -> int:
        return (self.tag >> 12) & (MAX_REGIONS - 1)

    def signature(self) -> int:
        return self.tag & SIGNATURE_MASK

    @staticmethod
    def make(is_start: bool, region: int, signature: int, clock: int) -> "ProfileRecord":
        if region >= MAX_REGIONS:
            raise Error(ErrorKind.Trace,
                        f"region id {region} overflows the 19-bit tag field")
        return ProfileRecord((START_FLAG if is_start else 0) | (region << 12) |
                             (signature & SIGNATURE_MASK), clock & 0xFFFFFFFF)


def encode_record(r: ProfileRecord) -> bytes:
    return struct.pack("<II", r.tag, r.payload)


def decode_record(b: bytes) -> ProfileRecord:
    tag, payload = struct.unpack_from("<II", b)
    return ProfileRecord(tag, payload)


def records_array(records) -> np.ndarray:
    a = np.empty(len(records), RECORD_DTYPE)
    for i, r in enumerate(records):
        a[i] = (r.tag, r.payload)
    return a


@dataclass
class TraceStream:
    block_index: int = 0
    warp_group: int = 0
    record_count: int = 0
    slot_capacity: int = 0
    slots: list = field(default_factory=list)  # ProfileRecord or RECORD_DTYPE


@dataclass
class GlobalTraceImage:
    streams: list = field(default_factory=list)


def serialize_image(img: GlobalTraceImage) -> bytes:
    """trace.hpp:158-179 (v1; > 65535 streams raise like the reference)."""
    if len(img.streams) > 0xFFFF:
        raise Error(ErrorKind.Trace, "too many streams for the image header")
    out = [TRACE_MAGIC, struct.pack("<HH", TRACE_VERSION, len(img.streams))]
    for s in img.streams:
        if len(s.slots) != s.slot_capacity:
            raise Error(ErrorKind.Trace,
                        "stream slot count does not match its declared capacity")
        out.append(struct.pack("<IIII", s.block_index, s.warp_group,
                               s.record_count, s.slot_capacity))
        sl = s.slots
        if isinstance(sl, np.ndarray):
            out.append(np.ascontiguousarray(sl, RECORD_DTYPE).tobytes())
        else:
            out.append(b"".join(encode_record(r) for r in sl))
    return b"".join(out)


def serialize_body_v2(body: np.ndarray, n_streams: int) -> bytes:
    """KPFT v2 container (this framework; u64 stream count)."""
    return TRACE_MAGIC + struct.pack("<HHQ", 2, 0, n_streams) + \
        np.ascontiguousarray(body).tobytes()


def deserialize_image(data: bytes) -> GlobalTraceImage:
    """trace.hpp:181-209 (host parse; v2 accepted as the framework container)."""
    n = len(data)
    if n < 4:
        raise Error(ErrorKind.Trace, "truncated trace image")
    if data[:4] != TRACE_MAGIC:
        raise Error(ErrorKind.Trace, "bad magic: not a trace image")
    if n < 6:
        raise Error(ErrorKind.Trace, "truncated trace image")
    (version,) = struct.unpack_from("<H", data, 4)
    if version == 1:
        if n < 8:
            raise Error(ErrorKind.Trace, "truncated trace image")
        (count,) = struct.unpack_from("<H", data, 6)
        pos = 8
    elif version == 2:
        if n < 16:
            raise Error(ErrorKind.Trace, "truncated trace image")
        (count,) = struct.unpack_from("<Q", data, 8)
        pos = 16
    else:
        raise Error(ErrorKind.Trace, f"unsupported trace version {version}")
    img = GlobalTraceImage()
    for _ in range(count):
        if pos + 16 > n:
            raise Error(ErrorKind.Trace, "truncated trace image")
        b, w, rc, cap = struct.unpack_from("<IIII", data, pos)
        pos += 16
        if pos + 8 * cap > n:
            raise Error(ErrorKind.Trace, "truncated trace image")
        slots = np.frombuffer(data, RECORD_DTYPE, cap, pos).copy()
        pos += 8 * cap
        img.streams.append(TraceStream(b, w, rc, cap, slots))
    if pos != n:
        raise Error(ErrorKind.Trace, "trailing bytes after trace image")
    return img


# ---------------------------------------------------------------------------
# plan
# ---------------------------------------------------------------------------


class BufferStrategy(enum.IntEnum):
    Circular = 0
    Flush = 1


@dataclass
class BufferPlan:
    slots_per_warp_group: int = 0
    strategy: BufferStrategy = BufferStrategy.Circular
    region_labels: list = field(default_factory=list)

    def base_offset(self, wg: int) -> int:
        return wg * self.slots_per_warp_group * 8

    def region_id(self, label: str):
        try:
            return self.region_labels.index(label)
        except ValueError:
            return None


def label_of(labels, rid: int) -> str:
    return labels[rid] if rid < len(labels) else f"region#{rid}"


@dataclass
class DeviceProgram:
    """The lowered program's side channel: what the replay and the critical
    path analysis need from `print_device_program` (lower.hpp:320-380) --
    the buffer plan (strategy, slots per stream, region table) and the
    barrier-derived candidate edges (barrier_edges, perfmodel.hpp:258-313)."""
    name: str
    num_warp_groups: int
    plan: BufferPlan
    barrier_edges: list


def parse_device_program(text: str) -> DeviceProgram:
    """Parse a `.dev` file (the reference's `print_device_program` output).

    barrier_edges: for every `arrive <b>` the label of the nearest preceding
    end `store_counter`, for every `wait <b>` the label of the nearest
    following start `store_counter` in the same warp-group body; an edge per
    (arrive, wait) pair on the same barrier with different labels, sorted and
    unique (perfmodel.hpp:258-313)."""
    import json as _json
    lines = text.splitlines()
    if not lines or not lines[0].startswith("device kernel "):
        raise Error(ErrorKind.Parse, "not a device program")
    head = lines[0].split()
    kv = dict(tok.split("=", 1) for tok in head if "=" in tok)
    labels, bodies, cur = [], [], None
    for line in lines[1:]:
        t = line.strip()
        if t.startswith("region ") and cur is None:
            labels.append(_json.loads(t[t.index('"'):]))
        elif t.startswith("wg") and t.endswith("{"):
            cur = []
            bodies.append(cur)
        elif cur is not None and t and t != "}":
            cur.append(t)

    def label(rid: int) -> str:
        return labels[rid] if rid < len(labels) else ""

    def region_of(t: str) -> int:
        return int(t.split("region=")[1].split()[0])

    arrives, waits = [], []
    for body in bodies:
        for i, t in enumerate(body):
            if t.startswith("arrive "):
                for j in range(i - 1, -1, -1):
                    if body[j].startswith("store_counter") and body[j].endswith(" end"):
                        if label(region_of(body[j])):
                            arrives.append((t.split()[1], label(region_of(body[j]))))
                        break
            elif t.startswith("wait "):
                for j in range(i + 1, len(body)):
                    if body[j].startswith("store_counter") and body[j].endswith(" start"):
                        if label(region_of(body[j])):
                            waits.append((t.split()[1], label(region_of(body[j]))))
                        break
    edges = sorted({(a, w) for b1, a in arrives for b2, w in waits if b1 == b2 and a != w})
    strategy = (BufferStrategy.Circular if kv.get("strategy") == "circular"
                else BufferStrategy.Flush)
    plan = BufferPlan(int(kv.get("slots_per_wg", 0)), strategy, labels)
    return DeviceProgram(head[2], int(kv.get("wgs", 0)), plan, edges)


def is_wait_marker(label: str) -> bool:
    return len(label) > len(WAIT_SUFFIX) and label.endswith(WAIT_SUFFIX)


# ---------------------------------------------------------------------------
# results
# ---------------------------------------------------------------------------


@dataclass
class TimelineEvent:
    region: str
    block_index: int
    warp_group: int
    iteration: int
    start: int
    end: int
    kind: str  # "exec" | "wait"
    corrected: bool

    def duration(self) -> int:
        return self.end - self.start


def timeline(events: np.ndarray, labels) -> list[TimelineEvent]:
    out = []
    for e in events:
        r = int(e["region"])
        out.append(TimelineEvent(label_of(labels, r & EV_REGION_MASK),
                                 int(e["block_index"]), int(e["warp_group"]),
                                 int(e["iteration"]), int(e["start"]), int(e["end"]),
                                 "wait" if r & EV_WAIT else "exec",
                                 bool(r & EV_CORRECTED)))
    return out


@dataclass
class TraceReplay:
    events: np.ndarray  # EVENT_DTYPE
    dropped_heads: int = 0
    truncated_tails: int = 0
    flagged_preconditions: int = 0
    malformed_groups: int = 0
    labels: list = field(default_factory=list)

    def timeline(self) -> list[TimelineEvent]:
        return timeline(self.events, self.labels)


@dataclass
class RegionStats:
    warp_group: int
    kind: str
    count: int
    min: int
    max: int
    mean: float
    sum: int = 0
    first_event: int = 0
    hist: list = field(default_factory=list)


@dataclass
class DecodedStream:
    block_index: int
    warp_group: int
    dropped_records: int
    records: np.ndarray  # RECORD_DTYPE


@dataclass
class PairResult:
    intervals: np.ndarray  # INTERVAL_DTYPE
    dropped_heads: int = 0
    truncated_tails: int = 0


@dataclass
class ReplayResult:
    events: np.ndarray
    flagged_preconditions: int = 0
    malformed_groups: int = 0


# ---------------------------------------------------------------------------
# the GPU context
# ---------------------------------------------------------------------------


class Context:
    """One wgpf_ctx (a CUDA device + stream + plan)."""

    def __init__(self, device: int = 0, stream: int = 0):
        self.L = L.lib()
        h = C.c_void_p()
        rc = self.L.wgpf_create(device, C.c_void_p(stream), C.byref(h))
        if rc != 0:
            raise RuntimeError(
                f"wgpf_create(device={device}) failed: "
                f"{self.L.wgpf_error_category(rc).decode()} (no usable CUDA device; "
                "this framework has no CPU fallback)")
        self.h = h
        self.plan = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.L.wgpf_destroy(h)
            self.h = None

    def set_stream(self, stream: int) -> None:
        self.L.wgpf_set_stream(self.h, C.c_void_p(stream))

    def set_plan(self, plan: BufferPlan) -> None:
        if self.plan is not None and self.plan == plan:
            return
        labels = list(plan.region_labels)
        arr = (C.c_char_p * max(1, len(labels)))(*[s.encode() for s in labels])
        _check(self.h, self.L.wgpf_set_plan(self.h, int(plan.slots_per_warp_group),
                                            int(plan.strategy), arr, len(labels)))
        self.plan = BufferPlan(plan.slots_per_warp_group, plan.strategy, labels)

    # -- replay_image --------------------------------------------------------
    def replay_image_bytes(self, data: bytes, plan: BufferPlan, record_cost: int,
                           flags: int = 0, events_cap: int | None = None) -> TraceReplay:
        self.set_plan(plan)
        buf = np.frombuffer(data, np.uint8)
        if events_cap is None:
            events_cap = max(1, len(data) // 16)
        ev = np.empty(events_cap, EVENT_DTYPE)
        ne, w = C.c_uint64(), L.Warnings()
        rc = self.L.wgpf_replay_image(self.h, buf.ctypes.data, len(data), record_cost,
                                      ev.ctypes.data, events_cap, flags,
                                      C.byref(ne), C.byref(w))
        if rc == L.E_BUFFER:
            return self.replay_image_bytes(data, plan, record_cost, flags, ne.value)
        _check(self.h, rc, ne.value)
        n = 0 if flags & L.F_STATS_ONLY else ne.value
        return TraceReplay(ev[:n].copy(), w.dropped_heads, w.truncated_tails,
                           w.flagged_preconditions, w.malformed_groups,
                           list(plan.region_labels))

    def replay_device(self, body_ptr: int, body_bytes: int, n_streams: int,
                      record_cost: int, events_ptr: int = 0, events_cap: int = 0,
                      flags: int = 0, stream_base: int = 0):
        """Device-resident KPFT body -> device events.  Returns
        (n_events, Warnings)."""
        ne, w = C.c_uint64(), L.Warnings()
        rc = self.L.wgpf_replay_device(self.h, C.c_void_p(body_ptr), body_bytes,
                                       n_streams, stream_base, record_cost,
                                       C.c_void_p(events_ptr), events_cap, flags,
                                       C.byref(ne), C.byref(w))
        _check(self.h, rc, ne.value)
        return ne.value, w

    def last_profile(self) -> dict:
        p = L.Profile()
        self.L.wgpf_last_profile(self.h, C.byref(p))
        return {k: getattr(p, k) for k, _ in L.Profile._fields_}

    def stats(self) -> dict:
        """Statistics of the last replay (label -> RegionStats), label order."""
        return self._read_stats(self.L.wgpf_stats_get)

    def _read_stats(self, fn, *args) -> dict:
        cap = 256
        while True:
            out = (L.RegionStat * cap)()
            n = C.c_uint32()
            rc = fn(self.h, *args, out, cap, C.byref(n))
            if rc == L.E_BUFFER:
                cap = n.value
                continue
            _check(self.h, rc)
            res = {}
            for i in range(n.value):
                s = out[i]
                res[s.label.decode()] = RegionStats(
                    s.warp_group, "wait" if s.kind else "exec", s.count, s.min, s.max,
                    s.mean, s.sum, s.first_event, list(s.hist))
            return res

    def region_stats(self, events: np.ndarray, exact_mean: bool = True,
                     on_device_ptr: int = 0) -> dict:
        flags = L.F_EXACT_MEAN if exact_mean else 0
        if on_device_ptr:
            return self._read_stats(self.L.wgpf_region_stats, C.c_void_p(on_device_ptr),
                                    len(events), 1, flags)
        ev = np.ascontiguousarray(events, EVENT_DTYPE)
        return self._read_stats(self.L.wgpf_region_stats, C.c_void_p(ev.ctypes.data),
                                len(ev), 0, flags)

    def stats_packed_bytes(self) -> int:
        return self.L.wgpf_stats_packed_bytes(self.h)

    def stats_export(self, dst_ptr: int) -> None:
        _check(self.h, self.L.wgpf_stats_export(self.h, C.c_void_p(dst_ptr)))

    def align_events(self, events, timing: np.ndarray, cycles_per_ns: float = 0.0,
                     on_device_ptr: int = 0, n_events: int | None = None):
        """Cross-SM alignment (wgpf_align_events): events from their CTA's
        SM clock into one global cycle domain using the runtime's per-CTA
        timing records (p1.CTA_TIMING_DTYPE).  Host events: returns the
        aligned copy; device events: in place.  Returns (events, cycles_per_ns)."""
        tm = np.ascontiguousarray(timing)
        f = C.c_double()
        if on_device_ptr:
            _check(self.h, self.L.wgpf_align_events(self.h, C.c_void_p(on_device_ptr),
                                                    n_events, 1, C.c_void_p(tm.ctypes.data),
                                                    len(tm), cycles_per_ns, C.byref(f)))
            return None, f.value
        ev = np.ascontiguousarray(events, EVENT_DTYPE).copy()
        _check(self.h, self.L.wgpf_align_events(self.h, C.c_void_p(ev.ctypes.data), len(ev),
                                                0, C.c_void_p(tm.ctypes.data), len(tm),
                                                cycles_per_ns, C.byref(f)))
        return ev, f.value

    def allreduce_stats(self, nccl_comm: int) -> None:
        """Combines this rank's statistics with every rank of an NCCL
        communicator (wgpf_allreduce_stats: export, one ncclAllGather, merge)."""
        _check(self.h, self.L.wgpf_allreduce_stats(self.h, C.c_void_p(nccl_comm)))

    def stats_merge(self, gathered_ptr: int, n_ranks: int) -> None:
        _check(self.h, self.L.wgpf_stats_merge(self.h, C.c_void_p(gathered_ptr),
                                               n_ranks))

    # -- unit-level entry points ---------------------------------------------
    def decode_image_bytes(self, data: bytes, plan: BufferPlan) -> list[DecodedStream]:
        self.set_plan(plan)
        buf = np.frombuffer(data, np.uint8)
        rcap, scap = max(1, len(data) // 8), max(1, len(data) // 16)
        recs = np.empty(rcap, RECORD_DTYPE)
        ds = np.empty(scap, L.DECODED_DTYPE)
        nr, ns = C.c_uint64(), C.c_uint64()
        _check(self.h, self.L.wgpf_decode_image(self.h, buf.ctypes.data, len(data),
                                                recs.ctypes.data, rcap, C.byref(nr),
                                                ds.ctypes.data, scap, C.byref(ns)))
        out = []
        for s in ds[:ns.value]:
            a, k = int(s["offset"]), int(s["count"])
            out.append(DecodedStream(int(s["block_index"]), int(s["warp_group"]),
                                     int(s["dropped_records"]), recs[a:a + k].copy()))
        return out

    def unwrap_clock(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, np.uint32)
        out = np.empty(len(v), np.uint64)
        _check(self.h, self.L.wgpf_unwrap_clock(self.h, v.ctypes.data, len(v),
                                                out.ctypes.data))
        return out

    def pair_records(self, records: np.ndarray, region_table) -> PairResult:
        self.set_plan(BufferPlan(0, BufferStrategy.Flush, list(region_table)))
        r = np.ascontiguousarray(records, RECORD_DTYPE)
        cap = len(r) // 2 + 1
        out = np.empty(cap, INTERVAL_DTYPE)
        n, dh, tt = C.c_uint64(), C.c_uint32(), C.c_uint32()
        _check(self.h, self.L.wgpf_pair_records(self.h, r.ctypes.data, len(r),
                                                out.ctypes.data, cap, C.byref(n),
                                                C.byref(dh), C.byref(tt)))
        return PairResult(out[:n.value].copy(), dh.value, tt.value)

    def replay(self, intervals: np.ndarray, region_table, block_index: int,
               warp_group: int, record_cost: int) -> ReplayResult:
        self.set_plan(BufferPlan(0, BufferStrategy.Flush, list(region_table)))
        iv = np.ascontiguousarray(intervals, INTERVAL_DTYPE)
        cap = max(1, len(iv))
        out = np.empty(cap, EVENT_DTYPE)
        n, w = C.c_uint64(), L.Warnings()
        _check(self.h, self.L.wgpf_replay_intervals(
            self.h, iv.ctypes.data, len(iv), block_index, warp_group, record_cost,
            out.ctypes.data, cap, C.byref(n), C.byref(w)))
        return ReplayResult(out[:n.value].copy(), w.flagged_preconditions,
                            w.malformed_groups)

    def critical_path(self, events: np.ndarray, barrier_edges=(), slack: int = 132,
                      exclude_warmup: bool = True, gate_by_block: bool = False,
                      on_device_ptr: int = 0, n_events: int | None = None) -> dict:
        """analyze_critical_path (perfmodel.hpp:317-501) on the GPU.  Labels
        come from the context plan.  Returns stages / mean / steady / wg /
        binding {(gate, gated): count} / cycle / period."""
        n = len(events) if n_events is None else n_events
        if on_device_ptr:
            ptr_ev, on_dev = C.c_void_p(on_device_ptr), 1
        else:
            ev = np.ascontiguousarray(events, EVENT_DTYPE)
            ptr_ev, on_dev = C.c_void_p(ev.ctypes.data), 0
        nb = len(barrier_edges)
        src = (C.c_char_p * max(1, nb))(*[a.encode() for a, _ in barrier_edges])
        dst = (C.c_char_p * max(1, nb))(*[b.encode() for _, b in barrier_edges])
        cap = 64
        while True:
            stages = (L.CpStage * cap)()
            bind = (C.c_uint64 * (cap * cap))()
            cyc = (C.c_uint32 * cap)()
            ns, nc, period = C.c_uint32(), C.c_uint32(), C.c_uint64()
            rc = self.L.wgpf_critical_path(self.h, ptr_ev, n, on_dev, src, dst, nb,
                                           slack, int(exclude_warmup),
                                           int(gate_by_block), stages, cap,
                                           C.byref(ns), bind, cap * cap, cyc, cap,
                                           C.byref(nc), C.byref(period))
            if rc == L.E_BUFFER:
                cap = max(2 * cap, ns.value)
                continue
            _check(self.h, rc)
            S = ns.value
            labels = [stages[i].label.decode() for i in range(S)]
            binding = {(labels[a], labels[b]): bind[a * S + b]
                       for a in range(S) for b in range(S) if bind[a * S + b]}
            return dict(stages=labels, mean=[stages[i].mean for i in range(S)],
                        steady=[stages[i].steady for i in range(S)],
                        wg=[stages[i].warp_group for i in range(S)],
                        binding=binding,
                        cycle=[labels[cyc[i]] for i in range(nc.value)],
                        period=period.value)

    def overlap(self, events: np.ndarray, role_of_wg, on_device_ptr: int = 0,
                n_events: int | None = None) -> dict:
        n = len(events) if n_events is None else n_events
        roles = np.ascontiguousarray(role_of_wg, np.uint8)
        if on_device_ptr:
            ptr_ev, on_dev = C.c_void_p(on_device_ptr), 1
        else:
            ev = np.ascontiguousarray(events, EVENT_DTYPE)
            ptr_ev, on_dev = C.c_void_p(ev.ctypes.data), 0
        out = L.Overlap()
        _check(self.h, self.L.wgpf_overlap_counters(self.h, ptr_ev, n, on_dev,
                                                    C.c_void_p(roles.ctypes.data),
                                                    len(roles), C.byref(out)))
        return dict(blocks=out.blocks, span=out.span, busy=list(out.busy),
                    both=out.both, bubble=list(out.bubble))

    def export_chrome_trace(self, events: np.ndarray, cycles_per_us: float = 1000.0,
                            on_device_ptr: int = 0, n_events: int | None = None) -> str:
        """export_chrome_trace (trace.hpp:493-511), byte-identical JSON."""
        n = len(events) if n_events is None else n_events
        if on_device_ptr:
            p, dev = C.c_void_p(on_device_ptr), 1
        else:
            ev = np.ascontiguousarray(events, EVENT_DTYPE)
            p, dev = C.c_void_p(ev.ctypes.data), 0
        ln = C.c_uint64()
        _check(self.h, self.L.wgpf_export_chrome_trace(self.h, p, n, dev, cycles_per_us,
                                                       None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        _check(self.h, self.L.wgpf_export_chrome_trace(self.h, p, n, dev, cycles_per_us,
                                                       buf, ln.value + 1, C.byref(ln)))
        return buf.raw[:ln.value].decode()

    def collect(self, profile_ptr: int, n_streams: int, validate_ptr: int = 0) -> bytes:
        """Engine::image (vgpu.hpp:136-148) of a device profile: the flushed
        KPFT body checked (debug-mode pairing errors -> instrument-error,
        flush overflow -> capacity-error, the reference's texts) and copied
        out as a KPFT image (v1 up to 65,535 streams, else v2)."""
        n = C.c_uint64()
        _check(self.h, self.L.wgpf_collect(self.h, C.c_void_p(profile_ptr), n_streams,
                                           C.c_void_p(validate_ptr), None, 0,
                                           C.byref(n)))
        buf = np.empty(n.value, np.uint8)
        _check(self.h, self.L.wgpf_collect(self.h, C.c_void_p(profile_ptr), n_streams,
                                           C.c_void_p(validate_ptr),
                                           C.c_void_p(buf.ctypes.data), n.value,
                                           C.byref(n)))
        return buf.tobytes()

    def synth_body(self, dst_ptr: int, shape: int, stream0: int, n_streams: int,
                   n_long: int) -> None:
        _check(self.h, self.L.wgpf_synth_body(self.h, C.c_void_p(dst_ptr), shape,
                                              stream0, n_streams, n_long))


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ---------------------------------------------------------------------------
# reference-signature module functions
# ---------------------------------------------------------------------------


def _image_bytes(image) -> bytes:
    if isinstance(image, (bytes, bytearray, memoryview)):
        return bytes(image)
    return serialize_image(image)


def decode_image(image, plan: BufferPlan) -> list[DecodedStream]:
    """decode_image(img, plan) (trace.hpp:222)."""
    return default_context().decode_image_bytes(_image_bytes(image), plan)


def unwrap_clock(values) -> np.ndarray:
    """unwrap_clock(values) (trace.hpp:257)."""
    return default_context().unwrap_clock(values)


def pair_records(stream, region_table) -> PairResult:
    """pair_records(stream, region_table) (trace.hpp:294)."""
    if not isinstance(stream, np.ndarray):
        stream = records_array(stream)
    return default_context().pair_records(stream, region_table)


def replay(pairs: PairResult, block_index: int, warp_group: int, record_cost: int,
           region_table=()) -> ReplayResult:
    """replay(pairs, block, wg, record_cost) (trace.hpp:398); labels of the
    interval region ids come from region_table."""
    return default_context().replay(pairs.intervals, region_table, block_index,
                                    warp_group, record_cost)


def replay_image(image, plan: BufferPlan, record_cost: int) -> TraceReplay:
    """replay_image(image, plan, record_cost) (pipeline.hpp:66)."""
    return default_context().replay_image_bytes(_image_bytes(image), plan, record_cost)


def region_stats(events: np.ndarray, region_table) -> dict:
    """region_stats(events) (pipeline.hpp:114) with the reference's bit-exact
    mean recurrence; label -> RegionStats in label order."""
    ctx = default_context()
    ctx.set_plan(BufferPlan(0, BufferStrategy.Flush, list(region_table)))
    return ctx.region_stats(events, exact_mean=True)

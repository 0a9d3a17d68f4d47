"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes bindings for
  * oracle/liboracle.so            -- the C restatement (oracle/wgpf_oracle.c)
  * oracle/_ref/libwgprof_ref.so   -- the reference's own headers compiled from
                                      /root/reference (oracle/ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product package
(paper_2505_21661_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwgprof_ref.so")

EVENT_DTYPE = np.dtype(
    [("start", "<u8"), ("end", "<u8"), ("region", "<u4"), ("iteration", "<u4"),
     ("block_index", "<u4"), ("warp_group", "<u4")])
assert EVENT_DTYPE.itemsize == 32

EV_WAIT = 0x80000000
EV_CORRECTED = 0x40000000
EV_REGION_MASK = 0x7FFFF
HIST_BINS = 64


def build(force: bool = False) -> None:
    """Builds liboracle.so (always) and _ref (when /root/reference exists)."""
    args = ["make", "-s", "-f", os.path.join(HERE, "Makefile")]
    if force:
        args.append("-B")
    subprocess.run(args + ["all"], check=True)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def label_blob(labels) -> bytes:
    return b"".join(s.encode() + b"\0" for s in labels)


def split_blob(ptr, n: int, length: int) -> list[str]:
    if n == 0:
        return []
    raw = C.string_at(ptr, length)
    parts = raw.split(b"\0")
    return [p.decode() for p in parts[:n]]


def label_of(labels, rid: int) -> str:
    return labels[rid] if rid < len(labels) else f"region#{rid}"


class OracleError(Exception):
    """Mirrors wgprof::Error: .code = 1 + ErrorKind, .category, message."""

    def __init__(self, code: int, category: str, message: str):
        super().__init__(message)
        self.code = code
        self.category = category


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------


class _Status(C.Structure):
    _fields_ = [("code", C.c_int), ("category", C.c_char * 32),
                ("message", C.c_char * 1024)]

    def raise_if(self):
        if self.code:
            raise OracleError(self.code, self.category.decode(),
                              self.message.decode())


class _Plan(C.Structure):
    _fields_ = [("slots_per_warp_group", C.c_uint64), ("strategy", C.c_uint32),
                ("n_labels", C.c_uint32), ("labels", C.POINTER(C.c_char_p))]


class _ReplayOut(C.Structure):
    _fields_ = [("n_events", C.c_uint64), ("events", C.c_void_p),
                ("dropped_heads", C.c_uint32), ("truncated_tails", C.c_uint32),
                ("flagged_preconditions", C.c_uint32),
                ("malformed_groups", C.c_uint32), ("n_streams", C.c_uint64),
                ("records", C.c_uint64)]


class _DecodeOut(C.Structure):
    _fields_ = [("n_streams", C.c_uint64), ("block", C.POINTER(C.c_uint32)),
                ("wg", C.POINTER(C.c_uint32)), ("dropped", C.POINTER(C.c_uint32)),
                ("offset", C.POINTER(C.c_uint64)), ("n_records", C.c_uint64),
                ("records", C.c_void_p)]


class _Interval(C.Structure):
    _fields_ = [("region_id", C.c_uint32), ("iteration", C.c_uint32),
                ("start", C.c_uint64), ("end", C.c_uint64),
                ("start_pos", C.c_uint64), ("end_pos", C.c_uint64)]


INTERVAL_DTYPE = np.dtype([("region_id", "<u4"), ("iteration", "<u4"),
                           ("start", "<u8"), ("end", "<u8"),
                           ("start_pos", "<u8"), ("end_pos", "<u8")])


class _PairOut(C.Structure):
    _fields_ = [("n", C.c_uint64), ("iv", C.c_void_p),
                ("dropped_heads", C.c_uint32), ("truncated_tails", C.c_uint32)]


class _Stat(C.Structure):
    _fields_ = [("label", C.c_char_p), ("warp_group", C.c_uint32),
                ("kind", C.c_uint32), ("count", C.c_uint64), ("min", C.c_uint64),
                ("max", C.c_uint64), ("sum", C.c_uint64), ("mean", C.c_double),
                ("mean_exact", C.c_double), ("first_event", C.c_uint64),
                ("hist", C.c_uint64 * HIST_BINS)]


class _StatsOut(C.Structure):
    _fields_ = [("n", C.c_uint32), ("s", C.POINTER(_Stat)), ("names", C.c_void_p)]


class _CpOut(C.Structure):
    _fields_ = [("n_stages", C.c_uint32), ("stage_label", C.POINTER(C.c_char_p)),
                ("stage_mean", C.POINTER(C.c_uint64)),
                ("stage_n", C.POINTER(C.c_uint64)),
                ("stage_wg", C.POINTER(C.c_uint32)), ("n_bind", C.c_uint32),
                ("bind_src", C.POINTER(C.c_uint32)),
                ("bind_dst", C.POINTER(C.c_uint32)),
                ("bind_count", C.POINTER(C.c_uint64)), ("n_cycle", C.c_uint32),
                ("cycle", C.POINTER(C.c_uint32)), ("period", C.c_uint64),
                ("names", C.c_void_p)]


class _OverlapOut(C.Structure):
    _fields_ = [("blocks", C.c_uint64), ("span", C.c_uint64),
                ("busy", C.c_uint64 * 2), ("both", C.c_uint64),
                ("bubble", C.c_uint64 * 2)]


@dataclass
class Replay:
    events: np.ndarray
    dropped_heads: int = 0
    truncated_tails: int = 0
    flagged_preconditions: int = 0
    malformed_groups: int = 0
    n_streams: int = 0
    records: int = 0


@dataclass
class Stat:
    label: str
    warp_group: int
    kind: str
    count: int
    min: int
    max: int
    sum: int = 0
    mean: float = 0.0
    mean_exact: float = 0.0
    first_event: int = 0
    hist: list = field(default_factory=list)


class Oracle:
    """The C restatement (oracle/wgpf_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.wgpo_replay_kpft.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Plan),
                                       C.c_uint64, C.POINTER(_ReplayOut),
                                       C.POINTER(_Status)]
        L.wgpo_replay_body.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64,
                                       C.POINTER(_Plan), C.c_uint64,
                                       C.POINTER(_ReplayOut), C.POINTER(_Status)]
        L.wgpo_free_replay.argtypes = [C.POINTER(_ReplayOut)]
        L.wgpo_decode_kpft.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Plan),
                                       C.POINTER(_DecodeOut), C.POINTER(_Status)]
        L.wgpo_free_decode.argtypes = [C.POINTER(_DecodeOut)]
        L.wgpo_unwrap_clock.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.wgpo_pair_records.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Plan),
                                        C.POINTER(_PairOut), C.POINTER(_Status)]
        L.wgpo_free_pair.argtypes = [C.POINTER(_PairOut)]
        L.wgpo_replay_pairs.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Plan),
                                        C.c_uint32, C.c_uint32, C.c_uint64,
                                        C.POINTER(_ReplayOut), C.POINTER(_Status)]
        L.wgpo_region_stats.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Plan),
                                        C.POINTER(_StatsOut)]
        L.wgpo_free_stats.argtypes = [C.POINTER(_StatsOut)]
        L.wgpo_critical_path.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Plan),
                                         C.POINTER(C.c_char_p),
                                         C.POINTER(C.c_char_p), C.c_uint32,
                                         C.c_uint64, C.c_int, C.c_int,
                                         C.POINTER(_CpOut), C.POINTER(_Status)]
        L.wgpo_free_cp.argtypes = [C.POINTER(_CpOut)]
        L.wgpo_overlap.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32,
                                   C.POINTER(_OverlapOut)]

    @staticmethod
    def _plan(slots, strategy, labels):
        arr = (C.c_char_p * max(1, len(labels)))(*[s.encode() for s in labels])
        p = _Plan(slots, strategy, len(labels), arr)
        p._keep = arr
        return p

    def _replay_result(self, out: _ReplayOut) -> Replay:
        n = out.n_events
        ev = np.empty(n, EVENT_DTYPE)
        if n:
            C.memmove(ev.ctypes.data, out.events, n * 32)
        r = Replay(ev, out.dropped_heads, out.truncated_tails,
                   out.flagged_preconditions, out.malformed_groups,
                   out.n_streams, out.records)
        self.lib.wgpo_free_replay(C.byref(out))
        return r

    def replay_kpft(self, data: bytes, slots: int, strategy: int, labels,
                    record_cost: int) -> Replay:
        buf = np.frombuffer(data, np.uint8)
        plan = self._plan(slots, strategy, labels)
        out, st = _ReplayOut(), _Status()
        self.lib.wgpo_replay_kpft(buf.ctypes.data, len(data), C.byref(plan),
                                  record_cost, C.byref(out), C.byref(st))
        st.raise_if()
        return self._replay_result(out)

    def replay_body(self, body: np.ndarray, n_streams: int, slots: int,
                    strategy: int, labels, record_cost: int) -> Replay:
        body = np.ascontiguousarray(body).view(np.uint8)
        plan = self._plan(slots, strategy, labels)
        out, st = _ReplayOut(), _Status()
        self.lib.wgpo_replay_body(body.ctypes.data, body.nbytes, n_streams,
                                  C.byref(plan), record_cost, C.byref(out),
                                  C.byref(st))
        st.raise_if()
        return self._replay_result(out)

    def decode_kpft(self, data: bytes, slots: int, strategy: int):
        buf = np.frombuffer(data, np.uint8)
        plan = self._plan(slots, strategy, [])
        out, st = _DecodeOut(), _Status()
        self.lib.wgpo_decode_kpft(buf.ctypes.data, len(data), C.byref(plan),
                                  C.byref(out), C.byref(st))
        st.raise_if()
        ns = out.n_streams
        res = []
        recs = np.empty(out.n_records, np.dtype([("tag", "<u4"), ("payload", "<u4")]))
        if out.n_records:
            C.memmove(recs.ctypes.data, out.records, out.n_records * 8)
        for s in range(ns):
            a, b = out.offset[s], out.offset[s + 1]
            res.append(dict(block_index=out.block[s], warp_group=out.wg[s],
                            dropped_records=out.dropped[s], records=recs[a:b].copy()))
        self.lib.wgpo_free_decode(C.byref(out))
        return res

    def unwrap_clock(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.empty(len(v), np.uint64)
        self.lib.wgpo_unwrap_clock(v.ctypes.data, len(v), out.ctypes.data)
        return out

    def pair_records(self, records: np.ndarray, labels):
        recs = np.ascontiguousarray(records)
        plan = self._plan(0, 0, labels)
        out, st = _PairOut(), _Status()
        self.lib.wgpo_pair_records(recs.ctypes.data, len(recs), C.byref(plan),
                                   C.byref(out), C.byref(st))
        st.raise_if()
        iv = np.empty(out.n, INTERVAL_DTYPE)
        if out.n:
            C.memmove(iv.ctypes.data, out.iv, out.n * INTERVAL_DTYPE.itemsize)
        res = (iv, out.dropped_heads, out.truncated_tails)
        self.lib.wgpo_free_pair(C.byref(out))
        return res

    def replay_pairs(self, intervals: np.ndarray, labels, block: int, wg: int,
                     record_cost: int) -> Replay:
        iv = np.ascontiguousarray(intervals, dtype=INTERVAL_DTYPE)
        plan = self._plan(0, 0, labels)
        out, st = _ReplayOut(), _Status()
        self.lib.wgpo_replay_pairs(iv.ctypes.data, len(iv), C.byref(plan), block,
                                   wg, record_cost, C.byref(out), C.byref(st))
        st.raise_if()
        return self._replay_result(out)

    def region_stats(self, events: np.ndarray, labels) -> list[Stat]:
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        plan = self._plan(0, 0, labels)
        out = _StatsOut()
        self.lib.wgpo_region_stats(ev.ctypes.data, len(ev), C.byref(plan),
                                   C.byref(out))
        res = []
        for i in range(out.n):
            s = out.s[i]
            res.append(Stat(s.label.decode(), s.warp_group,
                            "wait" if s.kind else "exec", s.count, s.min, s.max,
                            s.sum, s.mean, s.mean_exact, s.first_event,
                            list(s.hist)))
        self.lib.wgpo_free_stats(C.byref(out))
        return res

    def critical_path(self, events: np.ndarray, labels, barrier_edges=(),
                      slack=132, exclude_warmup=True, gate_by_block=False):
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        plan = self._plan(0, 0, labels)
        nb = len(barrier_edges)
        src = (C.c_char_p * max(1, nb))(*[a.encode() for a, _ in barrier_edges])
        dst = (C.c_char_p * max(1, nb))(*[b.encode() for _, b in barrier_edges])
        out, st = _CpOut(), _Status()
        self.lib.wgpo_critical_path(ev.ctypes.data, len(ev), C.byref(plan), src,
                                    dst, nb, slack, int(exclude_warmup),
                                    int(gate_by_block), C.byref(out), C.byref(st))
        st.raise_if()
        stages = [out.stage_label[i].decode() for i in range(out.n_stages)]
        res = dict(
            stages=stages,
            mean=[out.stage_mean[i] for i in range(out.n_stages)],
            steady=[out.stage_n[i] for i in range(out.n_stages)],
            wg=[out.stage_wg[i] for i in range(out.n_stages)],
            binding={(stages[out.bind_src[i]], stages[out.bind_dst[i]]):
                     out.bind_count[i] for i in range(out.n_bind)},
            cycle=[stages[out.cycle[i]] for i in range(out.n_cycle)],
            period=out.period)
        self.lib.wgpo_free_cp(C.byref(out))
        return res

    def overlap(self, events: np.ndarray, role_of_wg) -> dict:
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        roles = np.ascontiguousarray(role_of_wg, dtype=np.uint8)
        out = _OverlapOut()
        self.lib.wgpo_overlap(ev.ctypes.data, len(ev), roles.ctypes.data,
                              len(roles), C.byref(out))
        return dict(blocks=out.blocks, span=out.span, busy=list(out.busy),
                    both=out.both, bubble=list(out.bubble))


# ---------------------------------------------------------------------------
# The reference itself (oracle/_ref/libwgprof_ref.so)
# ---------------------------------------------------------------------------


class _RStatus(C.Structure):
    _fields_ = [("code", C.c_int), ("category", C.c_char * 32),
                ("message", C.c_char * 1024)]

    def raise_if(self):
        if self.code:
            raise OracleError(self.code, self.category.decode(),
                              self.message.decode())


REF_EVENT_DTYPE = np.dtype([("start", "<u8"), ("end", "<u8"), ("label", "<u4"),
                            ("iteration", "<u4"), ("block", "<u4"), ("wg", "<u4"),
                            ("kind", "<u4"), ("corrected", "<u4")])


class _RStat(C.Structure):
    _fields_ = [("label", C.c_uint32), ("wg", C.c_uint32), ("kind", C.c_uint32),
                ("count", C.c_uint32), ("min", C.c_uint64), ("max", C.c_uint64),
                ("mean", C.c_double)]


class _RReplayOut(C.Structure):
    _fields_ = [("st", _RStatus), ("n_events", C.c_uint64), ("events", C.c_void_p),
                ("n_labels", C.c_uint32), ("label_blob", C.c_void_p),
                ("label_blob_len", C.c_uint64), ("dropped_heads", C.c_uint32),
                ("truncated_tails", C.c_uint32),
                ("flagged_preconditions", C.c_uint32),
                ("malformed_groups", C.c_uint32), ("n_stats", C.c_uint32),
                ("stats", C.POINTER(_RStat))]


class _RDecodeOut(C.Structure):
    _fields_ = [("st", _RStatus), ("n_streams", C.c_uint64),
                ("block", C.POINTER(C.c_uint32)), ("wg", C.POINTER(C.c_uint32)),
                ("dropped", C.POINTER(C.c_uint32)),
                ("offset", C.POINTER(C.c_uint64)), ("n_records", C.c_uint64),
                ("tags", C.POINTER(C.c_uint32)),
                ("payloads", C.POINTER(C.c_uint32))]


REF_INTERVAL_DTYPE = np.dtype([("region_id", "<u4"), ("label", "<u4"),
                               ("iteration", "<u4"), ("pad", "<u4"),
                               ("start", "<u8"), ("end", "<u8"),
                               ("start_pos", "<u8"), ("end_pos", "<u8")])


class _RPairOut(C.Structure):
    _fields_ = [("st", _RStatus), ("n", C.c_uint64), ("iv", C.c_void_p),
                ("dropped_heads", C.c_uint32), ("truncated_tails", C.c_uint32),
                ("n_labels", C.c_uint32), ("label_blob", C.c_void_p),
                ("label_blob_len", C.c_uint64)]


class _RCpOut(C.Structure):
    _fields_ = [("st", _RStatus), ("n_cycle", C.c_uint32),
                ("cycle_blob", C.c_void_p), ("cycle_blob_len", C.c_uint64),
                ("period", C.c_uint64), ("n_nodes", C.c_uint32),
                ("node_blob", C.c_void_p), ("node_blob_len", C.c_uint64),
                ("node_duration", C.POINTER(C.c_uint64)), ("n_edges", C.c_uint32),
                ("edge_src", C.POINTER(C.c_uint32)),
                ("edge_dst", C.POINTER(C.c_uint32)),
                ("n_barrier_edges", C.c_uint32),
                ("barrier_edge_blob", C.c_void_p),
                ("barrier_edge_blob_len", C.c_uint64)]


class _RBenchOut(C.Structure):
    _fields_ = [("st", _RStatus), ("seconds", C.c_double), ("records", C.c_uint64),
                ("events", C.c_uint64), ("streams", C.c_uint64)]


@dataclass
class RefReplay:
    events: np.ndarray  # REF_EVENT_DTYPE
    labels: list
    dropped_heads: int
    truncated_tails: int
    flagged_preconditions: int
    malformed_groups: int
    stats: list


class Reference:
    """The reference implementation compiled from /root/reference."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference)")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_replay_kpft.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                      C.c_char_p, C.c_uint32, C.c_uint64,
                                      C.POINTER(_RReplayOut)]
        L.ref_free_replay.argtypes = [C.POINTER(_RReplayOut)]
        L.ref_decode_kpft.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                      C.POINTER(_RDecodeOut)]
        L.ref_free_decode.argtypes = [C.POINTER(_RDecodeOut)]
        L.ref_unwrap_clock.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.ref_pair_records.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64,
                                       C.c_char_p, C.c_uint32, C.POINTER(_RPairOut)]
        L.ref_free_pair.argtypes = [C.POINTER(_RPairOut)]
        L.ref_replay_pairs.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p,
                                       C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint64, C.POINTER(_RReplayOut)]
        L.ref_critical_path_kpft.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p,
                                             C.c_uint64, C.c_uint64, C.c_int,
                                             C.POINTER(_RCpOut)]
        L.ref_free_cp.argtypes = [C.POINTER(_RCpOut)]
        L.ref_run_fixture.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p,
                                      C.POINTER(_RStatus)]
        L.ref_random_program_image.argtypes = [C.c_uint64, C.c_int, C.c_int,
                                               C.c_uint32, C.c_uint32, C.c_uint64,
                                               C.c_char_p, C.POINTER(_RStatus)]
        L.ref_bench_replay.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64,
                                       C.c_uint32, C.c_char_p, C.c_uint32,
                                       C.c_uint64, C.c_uint64, C.c_int,
                                       C.POINTER(_RBenchOut)]

    def export_chrome(self, events: np.ndarray, labels, cycles_per_us: float = 1000.0) -> str:
        """export_chrome_trace (trace.hpp:493-511) over this framework's event
        array (the reference's own JSON writer, nlohmann 3.11.3)."""
        L = self.lib
        L.ref_export_chrome.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint32,
                                        C.c_double, C.POINTER(C.c_void_p),
                                        C.POINTER(_RStatus)]
        L.ref_export_chrome.restype = C.c_int64
        L.ref_free_text.argtypes = [C.c_void_p]
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        p, st = C.c_void_p(), _RStatus()
        n = L.ref_export_chrome(ev.ctypes.data, len(ev), label_blob(labels), len(labels),
                                cycles_per_us, C.byref(p), C.byref(st))
        st.raise_if()
        try:
            return C.string_at(p, n).decode()
        finally:
            L.ref_free_text(p)

    def replay_kpft(self, data: bytes, slots: int, strategy: int, labels,
                    record_cost: int) -> RefReplay:
        buf = np.frombuffer(data, np.uint8)
        out = _RReplayOut()
        self.lib.ref_replay_kpft(buf.ctypes.data, len(data), slots, strategy,
                                 label_blob(labels), len(labels), record_cost,
                                 C.byref(out))
        try:
            out.st.raise_if()
            return self._replay(out)
        finally:
            self.lib.ref_free_replay(C.byref(out))

    def _replay(self, out) -> RefReplay:
        n = out.n_events
        ev = np.empty(n, REF_EVENT_DTYPE)
        if n:
            C.memmove(ev.ctypes.data, out.events, n * REF_EVENT_DTYPE.itemsize)
        labels = split_blob(out.label_blob, out.n_labels, out.label_blob_len)
        stats = []
        for i in range(out.n_stats):
            s = out.stats[i]
            stats.append(Stat(labels[s.label], s.wg, "wait" if s.kind else "exec",
                              s.count, s.min, s.max, mean=s.mean))
        return RefReplay(ev, labels, out.dropped_heads, out.truncated_tails,
                         out.flagged_preconditions, out.malformed_groups, stats)

    def decode_kpft(self, data: bytes, slots: int, strategy: int):
        buf = np.frombuffer(data, np.uint8)
        out = _RDecodeOut()
        self.lib.ref_decode_kpft(buf.ctypes.data, len(data), slots, strategy,
                                 C.byref(out))
        try:
            out.st.raise_if()
            res = []
            for s in range(out.n_streams):
                a, b = out.offset[s], out.offset[s + 1]
                tags = np.array([out.tags[i] for i in range(a, b)], np.uint32)
                pay = np.array([out.payloads[i] for i in range(a, b)], np.uint32)
                res.append(dict(block_index=out.block[s], warp_group=out.wg[s],
                                dropped_records=out.dropped[s], tags=tags,
                                payloads=pay))
            return res
        finally:
            self.lib.ref_free_decode(C.byref(out))

    def unwrap_clock(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.empty(len(v), np.uint64)
        self.lib.ref_unwrap_clock(v.ctypes.data, len(v), out.ctypes.data)
        return out

    def pair_records(self, tags, payloads, labels):
        t = np.ascontiguousarray(tags, dtype=np.uint32)
        p = np.ascontiguousarray(payloads, dtype=np.uint32)
        out = _RPairOut()
        self.lib.ref_pair_records(t.ctypes.data, p.ctypes.data, len(t),
                                  label_blob(labels), len(labels), C.byref(out))
        try:
            out.st.raise_if()
            iv = np.empty(out.n, REF_INTERVAL_DTYPE)
            if out.n:
                C.memmove(iv.ctypes.data, out.iv, out.n * REF_INTERVAL_DTYPE.itemsize)
            names = split_blob(out.label_blob, out.n_labels, out.label_blob_len)
            return iv, names, out.dropped_heads, out.truncated_tails
        finally:
            self.lib.ref_free_pair(C.byref(out))

    def replay_pairs(self, iv: np.ndarray, labels, block, wg, record_cost):
        """iv: REF_INTERVAL_DTYPE with .label indexing `labels`."""
        iv = np.ascontiguousarray(iv, dtype=REF_INTERVAL_DTYPE)
        out = _RReplayOut()
        self.lib.ref_replay_pairs(iv.ctypes.data, len(iv), label_blob(labels),
                                  len(labels), block, wg, record_cost, C.byref(out))
        try:
            out.st.raise_if()
            return self._replay(out)
        finally:
            self.lib.ref_free_replay(C.byref(out))

    def critical_path_kpft(self, data: bytes, dev_text: str, record_cost: int,
                           slack=132, exclude_warmup=True) -> dict:
        buf = np.frombuffer(data, np.uint8)
        out = _RCpOut()
        self.lib.ref_critical_path_kpft(buf.ctypes.data, len(data),
                                        dev_text.encode(), record_cost, slack,
                                        int(exclude_warmup), C.byref(out))
        try:
            out.st.raise_if()
            nodes = split_blob(out.node_blob, out.n_nodes, out.node_blob_len)
            be = split_blob(out.barrier_edge_blob, 2 * out.n_barrier_edges,
                            out.barrier_edge_blob_len)
            return dict(
                cycle=split_blob(out.cycle_blob, out.n_cycle, out.cycle_blob_len),
                period=out.period, nodes=nodes,
                durations=[out.node_duration[i] for i in range(out.n_nodes)],
                edges=[(out.edge_src[i], out.edge_dst[i]) for i in range(out.n_edges)],
                barrier_edges=[(be[2 * i], be[2 * i + 1])
                               for i in range(out.n_barrier_edges)])
        finally:
            self.lib.ref_free_cp(C.byref(out))

    def run_fixture(self, conf: str, kir: str, out_prefix: str) -> None:
        st = _RStatus()
        self.lib.ref_run_fixture(conf.encode(), kir.encode(), out_prefix.encode(),
                                 C.byref(st))
        st.raise_if()

    def random_program_image(self, seed, index, with_loop, num_wgs, strategy,
                             slots_total, out_prefix) -> None:
        st = _RStatus()
        self.lib.ref_random_program_image(seed, index, int(with_loop), num_wgs,
                                          strategy, slots_total,
                                          out_prefix.encode(), C.byref(st))
        st.raise_if()

    def lower_kir(self, kir: str, strategy: int, slots_total: int = 0,
                  signature_bits: bool = False, iteration_signature: bool = False,
                  global_buffer: bool = False, simulate: bool = False,
                  out_prefix: str = "") -> dict:
        """lower() (lower.hpp:220) of KIR text, optionally simulate()
        (vgpu.hpp:424): {'slots', 'labels'[, 'image', 'store_log']}; raises
        RefError with the reference's kind and message."""
        import tempfile
        L = self.lib
        L.ref_lower_kir.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_char_p, C.POINTER(_RStatus)]
        with tempfile.TemporaryDirectory() as d:
            pre = os.path.join(d, "p")
            st = _RStatus()
            L.ref_lower_kir(kir.encode(), strategy, slots_total, int(signature_bits),
                            int(iteration_signature), int(global_buffer), int(simulate),
                            pre.encode(), C.byref(st))
            st.raise_if()
            lines = open(pre + ".plan").read().split("\n")
            out = {"slots": int(lines[0]), "labels": [l for l in lines[1:-1]]}
            if simulate:
                out["image"] = open(pre + ".kpft", "rb").read()
                out["store_log"] = [[int(t, 16) for t in line.split()]
                                    for line in open(pre + ".log").read().split("\n")[:-1]]
            return out

    def bench_replay(self, body: np.ndarray, n_streams: int, slots: int,
                     strategy: int, labels, record_cost: int, chunk_streams: int,
                     nthreads: int) -> dict:
        body = np.ascontiguousarray(body).view(np.uint8)
        out = _RBenchOut()
        self.lib.ref_bench_replay(body.ctypes.data, n_streams, slots, strategy,
                                  label_blob(labels), len(labels), record_cost,
                                  chunk_streams, nthreads, C.byref(out))
        out.st.raise_if()
        return dict(seconds=out.seconds, records=out.records, events=out.events,
                    streams=out.streams)


# ---------------------------------------------------------------------------
# canonical comparison helpers
# ---------------------------------------------------------------------------

CANON_DTYPE = np.dtype([("start", "<u8"), ("end", "<u8"), ("label", "<u4"),
                        ("iteration", "<u4"), ("block", "<u4"), ("wg", "<u4"),
                        ("kind", "<u4"), ("corrected", "<u4")])


class LabelSpace:
    """Interns label strings so that events from different producers compare."""

    def __init__(self):
        self.ids: dict[str, int] = {}

    def id(self, s: str) -> int:
        if s not in self.ids:
            self.ids[s] = len(self.ids)
        return self.ids[s]


def canon_from_events(ev: np.ndarray, labels, space: LabelSpace) -> np.ndarray:
    """wgpf_event array (region ids) -> canonical label-keyed array."""
    out = np.empty(len(ev), CANON_DTYPE)
    out["start"] = ev["start"]
    out["end"] = ev["end"]
    rid = ev["region"] & EV_REGION_MASK
    uniq, inv = np.unique(rid, return_inverse=True)
    lut = np.array([space.id(label_of(labels, int(r))) for r in uniq], np.uint32)
    out["label"] = lut[inv] if len(uniq) else 0
    out["iteration"] = ev["iteration"]
    out["block"] = ev["block_index"]
    out["wg"] = ev["warp_group"]
    out["kind"] = (ev["region"] >> 31) & 1
    out["corrected"] = (ev["region"] >> 30) & 1
    return out


def canon_from_ref(ev: np.ndarray, ref_labels, space: LabelSpace) -> np.ndarray:
    out = np.empty(len(ev), CANON_DTYPE)
    for f in ("start", "end", "iteration", "block", "wg", "kind", "corrected"):
        out[f] = ev[f]
    lut = np.array([space.id(s) for s in ref_labels] or [0], np.uint32)
    out["label"] = lut[ev["label"]] if len(ev) else 0
    return out

"""Analytic overlap models on measured stage times.

Host-side mirrors of the reference's models in wgprof/perfmodel.hpp -- tiny
graphs and a handful of integers, so they stay on the host and take the GPU
results (stage means, binding edges from `Context.critical_path`) as input:

  swp_latency      perfmodel.hpp:44-68    software-pipelining latency
  ws_latency       perfmodel.hpp:97-158   warp-specialisation longest path
  roofline         perfmodel.hpp:180-187  compute / memory cycles
  overhead_model   perfmodel.hpp:196-198  Eq. 1, T_vanilla + N * cost
  load_stage_table perfmodel.hpp:202-222  "<stage> <t_load> <t_comp>" text

Same names, argument meaning, integer arithmetic (u64 wrap, i64 delta,
ceiling divisions) and `Error(kind, message)` as the reference; checked
against the reference itself in tests/test_models.py.
"""
from __future__ import annotations

import dataclasses
import enum

from .trace import Error, ErrorKind

_M64 = (1 << 64) - 1


def _u64(x: int) -> int:
    return x & _M64


def _i64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >> 63 else x


# ---- software pipelining -----------------------------------------------------

@dataclasses.dataclass
class SwpStage:
    name: str = ""
    t_load: int = 0
    t_comp: int = 0


@dataclasses.dataclass
class SwpInput:
    n_warp_groups: int = 1
    n_pipe_stages: int = 1
    n_loop: int = 1
    stages: list = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class SwpResult:
    delta: int = 0
    latency: int = 0


def swp_latency(inp: SwpInput) -> SwpResult:
    """delta = N_WG * N_pipe * sum(t_comp) - max(t_load + t_comp); compute
    bound (sum(t_comp) * N_loop) when delta >= 0, else load bound
    (ceil(max * N_loop / N_pipe))."""
    if not inp.stages or not inp.n_warp_groups or not inp.n_pipe_stages or not inp.n_loop:
        raise Error(ErrorKind.Validate, "swp_latency: inputs must be positive")
    comp = _u64(sum(s.t_comp for s in inp.stages))
    worst = max(_u64(s.t_load + s.t_comp) for s in inp.stages)
    delta = _i64(_i64(inp.n_warp_groups * inp.n_pipe_stages) * _i64(comp) - _i64(worst))
    if delta >= 0:
        return SwpResult(delta, _u64(comp * inp.n_loop))
    total = _u64(worst * inp.n_loop)
    return SwpResult(delta, _u64(total + inp.n_pipe_stages - 1) // inp.n_pipe_stages)


# ---- warp specialisation -----------------------------------------------------

class StageKind(enum.IntEnum):
    Load = 0
    Comp = 1


@dataclasses.dataclass
class WsNode:
    label: str = ""
    duration: int = 0
    kind: StageKind = StageKind.Comp


@dataclasses.dataclass
class WsInput:
    nodes: list = dataclasses.field(default_factory=list)
    edges: list = dataclasses.field(default_factory=list)  # (src, dst) indices


@dataclasses.dataclass
class WsResult:
    critical_path: list = dataclasses.field(default_factory=list)
    latency: int = 0


def ws_latency(inp: WsInput) -> WsResult:
    """Longest duration-weighted path of the stage DAG.  Ties: a node's
    successor is the first best one in edge order unless a later one with the
    same length has a smaller label (a successor only extends the path if it
    adds length or replaces an earlier choice); the start is the longest
    node, smaller label on ties."""
    n = len(inp.nodes)
    out_edges = [[] for _ in range(n)]
    for a, b in inp.edges:
        if not (0 <= a < n and 0 <= b < n):
            raise Error(ErrorKind.Validate, "ws_latency: edge index out of range")
        out_edges[a].append(b)
    # depth-first post-order with colouring; a grey successor is a cycle
    WHITE, GREY, BLACK = 0, 1, 2
    colour = [WHITE] * n
    best = [0] * n
    nxt: list = [None] * n
    for root in range(n):
        if colour[root] != WHITE:
            continue
        stack = [(root, 0)]
        colour[root] = GREY
        while stack:
            v, k = stack[-1]
            if k < len(out_edges[v]):
                stack[-1] = (v, k + 1)
                s = out_edges[v][k]
                if colour[s] == GREY:
                    raise Error(ErrorKind.Validate, "ws_latency: stage graph has a cycle")
                if colour[s] == WHITE:
                    colour[s] = GREY
                    stack.append((s, 0))
                continue
            d = inp.nodes[v].duration
            b, c = _u64(d), None
            for s in out_edges[v]:
                cand = _u64(d + best[s])
                if cand > b or (cand == b and c is not None and
                                inp.nodes[s].label < inp.nodes[c].label):
                    b, c = cand, s
            best[v], nxt[v] = b, c
            colour[v] = BLACK
            stack.pop()
    res = WsResult()
    if n == 0:
        return res
    start = 0
    for i in range(1, n):
        if best[i] > best[start] or (best[i] == best[start] and
                                     inp.nodes[i].label < inp.nodes[start].label):
            start = i
    res.latency = best[start]
    v = start
    while v is not None:
        res.critical_path.append(inp.nodes[v].label)
        v = nxt[v]
    return res


def ws_input_from_critical_path(cp: dict) -> WsInput:
    """The stage graph of a `Context.critical_path` result as ws_latency
    input -- the reference's CriticalPathAnalysis.graph
    (perfmodel.hpp:407-497): stages in label order with their mean
    durations (kind Load when the label contains "Load"); edges the binding
    cycle unfolded into a chain when there is one, else every edge binding in
    at least half of its target's steady-state instances."""
    order = sorted(range(len(cp["stages"])), key=lambda i: cp["stages"][i])
    labels = [cp["stages"][i] for i in order]
    index = {l: k for k, l in enumerate(labels)}
    nodes = [WsNode(cp["stages"][i], int(cp["mean"][i]),
                    StageKind.Load if "Load" in cp["stages"][i] else StageKind.Comp)
             for i in order]
    if cp["cycle"]:
        cyc = [index[l] for l in cp["cycle"]]
        edges = list(zip(cyc[:-1], cyc[1:]))
    else:
        steady = {cp["stages"][i]: cp["steady"][i] for i in range(len(cp["stages"]))}
        edges = sorted({(index[a], index[b]) for (a, b), cnt in cp["binding"].items()
                        if 2 * cnt >= steady[b]})
    return WsInput(nodes, edges)


# ---- roofline and instrumentation overhead -------------------------------------

@dataclasses.dataclass
class RooflineInput:
    flops: int = 0
    throughput: int = 1  # operations per cycle
    t_read: int = 0
    bytes: int = 0
    bandwidth: int = 1   # bytes per cycle


@dataclasses.dataclass
class RooflineResult:
    compute_cycles: int = 0
    memory_cycles: int = 0


def roofline(inp: RooflineInput) -> RooflineResult:
    if not inp.throughput or not inp.bandwidth:
        raise Error(ErrorKind.Validate, "roofline: rates must be positive")
    return RooflineResult(_u64(inp.flops + inp.throughput - 1) // inp.throughput,
                          _u64(inp.t_read + _u64(inp.bytes + inp.bandwidth - 1) // inp.bandwidth))


@dataclasses.dataclass
class OverheadInput:
    t_vanilla: int = 0
    n_record: int = 0
    cycle_record: int = 0


def overhead_model(inp: OverheadInput) -> int:
    """Eq. 1: T_th = T_vanilla + N_record * cycle_record (u64)."""
    return _u64(inp.t_vanilla + inp.n_record * inp.cycle_record)


# ---- stage table -------------------------------------------------------------------

_WS = " \t\n\v\f\r"  # isspace() in the C locale


def _scan_u64(line: str, pos: int):
    """istream >> uint64_t: skip blanks, optional sign, decimal digits;
    (value, next position) or None.  A minus sign negates modulo 2^64."""
    n = len(line)
    while pos < n and line[pos] in _WS:
        pos += 1
    neg = False
    if pos < n and line[pos] in "+-":
        neg = line[pos] == "-"
        pos += 1
    d0 = pos
    while pos < n and line[pos].isdigit() and line[pos].isascii():
        pos += 1
    if pos == d0:
        return None
    v = int(line[d0:pos])
    if v > _M64:
        return None
    return ((-v) & _M64 if neg else v), pos


def load_stage_table(text: str) -> list:
    """One `<stage> <t_load> <t_comp>` per line, `#` starts a comment, blank
    lines skipped; anything else is a parse-error naming the line."""
    stages = []
    for lineno, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0]
        head = line.lstrip(_WS)
        if not head:
            continue
        k = 0
        while k < len(head) and head[k] not in _WS:
            k += 1
        name, rest = head[:k], head[k:]
        a = _scan_u64(rest, 0)
        b = _scan_u64(rest, a[1]) if a else None
        if b is None:
            raise Error(ErrorKind.Parse, f"stage table line {lineno}: expected "
                        "<stage> <t_load> <t_comp>")
        stages.append(SwpStage(name, a[0], b[0]))
    return stages

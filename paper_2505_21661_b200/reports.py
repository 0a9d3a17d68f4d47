"""The reference's JSON reports on the GPU's results ("wire
the GPU binding counts into the reference report generator").

  replay_report  make_replay_report       pipeline.hpp:145-174
  model_report   detail::model_report_json pipeline.hpp:178-238
  dumps          nlohmann::ordered_json::dump(2) + "\\n" (pipeline.hpp:275-276)

Inputs are what the GPU path produces -- `Context.region_stats` (label ->
RegionStats), `Context.critical_path` (stage means, binding counts, cycle,
period), the replay warnings -- plus the simulator totals the reference
reads from its vGPU (total / vanilla cycles, records written; the simulator
itself is out of scope).  Doubles are formatted by libwgpf's Grisu2
(`wgpf_format_json_double`), so the bytes equal the reference's files.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math

from . import models as M

_WAIT = ".wait"


@dataclasses.dataclass
class SimTotals:
    """SimResult's totals (vgpu.hpp:61-68)."""
    total_cycles: int = 0
    vanilla_cycles: int = 0
    records_written: int = 0


@dataclasses.dataclass
class ModelParams:
    """config.hpp:174-179 ([model] section)."""
    pipe_stages: int = 1
    warp_groups: int = 1
    loop_iters: int = 1
    swp_stages: list = dataclasses.field(default_factory=list)  # (load, comp)


class Double(float):
    """A JSON number that is always written as a double (nlohmann keeps the
    C++ type: 0.0 stays "0.0")."""


def _llround(x: float) -> int:
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


def _fmt_double(x: float) -> str:
    from ._lib import lib
    L = lib()
    L.wgpf_format_json_double.argtypes = [C.c_double, C.c_char_p, C.c_uint64]
    L.wgpf_format_json_double.restype = C.c_int
    buf = C.create_string_buffer(40)
    n = L.wgpf_format_json_double(float(x), buf, 40)
    if n < 0:
        raise RuntimeError("wgpf_format_json_double failed")
    return buf.raw[:n].decode()


def _str(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif o < 0x20:
            out.append({8: "\\b", 9: "\\t", 10: "\\n", 12: "\\f", 13: "\\r"}.get(
                o, "\\u%04x" % o))
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _dump(v, ind: int) -> str:
    pad, inner = " " * ind, " " * (ind + 2)
    if isinstance(v, dict):
        if not v:
            return "{}"
        return "{\n" + ",\n".join(f"{inner}{_str(k)}: {_dump(x, ind + 2)}"
                                  for k, x in v.items()) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(inner + _dump(x, ind + 2) for x in v) + "\n" + pad + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if v is None:
        return "null"
    if isinstance(v, (Double, float)):
        return _fmt_double(v)
    if isinstance(v, int):
        return str(v)
    return _str(str(v))


def dumps(report: dict) -> str:
    """nlohmann ordered_json dump(2) plus the trailing newline the reference
    writes."""
    return _dump(report, 0) + "\n"


def _kind(k) -> str:
    return "wait" if str(getattr(k, "name", k)).lower().endswith("wait") else "exec"


def replay_report(kernel: str, sim: SimTotals, stats: dict, cp: dict, warnings,
                  record_cost: int) -> dict:
    """make_replay_report: regions in label order, the binding cycle (or the
    stage graph's longest path when there is none), period, warnings."""
    regions = []
    for label in sorted(stats):
        rs = stats[label]
        regions.append({"region": label, "warp_group": int(rs.warp_group),
                        "kind": _kind(rs.kind), "count": int(rs.count),
                        "mean_duration": Double(rs.mean), "min_duration": int(rs.min),
                        "max_duration": int(rs.max)})
    path = list(cp["cycle"]) or M.ws_latency(M.ws_input_from_critical_path(cp)).critical_path
    return {"kernel": kernel, "total_cycles": int(sim.total_cycles),
            "vanilla_cycles": int(sim.vanilla_cycles),
            "records_written": int(sim.records_written), "record_cost": int(record_cost),
            "regions": regions, "critical_path": path,
            "iteration_period": int(cp["period"]),
            "warnings": {"dropped_heads": int(warnings.dropped_heads),
                         "truncated_tails": int(warnings.truncated_tails),
                         "flagged_preconditions": int(warnings.flagged_preconditions),
                         "malformed_groups": int(warnings.malformed_groups)}}


def model_report(kernel: str, sim: SimTotals, stats: dict, cp: dict, record_cost: int,
                 params: ModelParams | None = None) -> dict:
    """model_report_json: the warp-specialisation model over the measured
    stage graph, Eq. 1 against the measured total, and the software-
    pipelining model on measured stage durations when stages are given."""
    ws = M.ws_latency(M.ws_input_from_critical_path(cp))
    theo = M.overhead_model(M.OverheadInput(sim.vanilla_cycles, sim.records_written,
                                            record_cost))
    rep = {"kernel": kernel,
           "ws_model": {"critical_path": ws.critical_path, "latency": ws.latency},
           "iteration_period": int(cp["period"]),
           "overhead_model": {"vanilla_cycles": int(sim.vanilla_cycles),
                              "records": int(sim.records_written),
                              "record_cost": int(record_cost), "theoretical_cycles": theo,
                              "actual_cycles": int(sim.total_cycles),
                              "ratio": Double(0.0 if theo == 0 else
                                              float(sim.total_cycles) / float(theo))}}
    if params and params.swp_stages:
        def duration(label):
            t = 0
            if label in stats:
                t += _llround(stats[label].mean)
            if label + _WAIT in stats:
                t += _llround(stats[label + _WAIT].mean)
            return t & ((1 << 64) - 1)
        si = M.SwpInput(params.warp_groups, params.pipe_stages, params.loop_iters,
                        [M.SwpStage(f"{a}/{b}", duration(a), duration(b))
                         for a, b in params.swp_stages])
        sr = M.swp_latency(si)
        rep["swp_model"] = {"stages": [{"stage": s.name, "t_load": s.t_load,
                                        "t_comp": s.t_comp} for s in si.stages],
                            "delta": sr.delta, "latency": sr.latency}
    return rep

"""The reference's JSON reports (paper_2505_21661_b200/reports.py) rebuilt
from the replay results: byte-identical to the fixtures' golden
<name>_replay.json / <name>_model.json (written by the reference's
run_pipeline).  CPU: statistics and critical path from the oracle (the GPU
path's are checked equal to the oracle's in tests/test_gpu_*.py); doubles
through libwgpf's formatter (host code)."""
import json
import os

import pytest

from conftest import FIXTURES, GOLDEN, load_fixture
from paper_2505_21661_b200 import reports as R

from test_oracle import dev_barrier_edges

# [model] sections of the fixtures' .conf files (config.hpp:174-179)
PARAMS = {
    "simple": R.ModelParams(2, 1, 50, [("Matmul.wait", "Scale")]),
    "gemm_swp": R.ModelParams(2, 1, 20, [("Load A", "MMA even"), ("Load B", "MMA odd")]),
}


def _golden(name, kind):
    return open(os.path.join(GOLDEN, "fixtures", f"{name}_{kind}.json")).read()


@pytest.mark.parametrize("name", FIXTURES)
def test_reports_byte_identical(oracle, name):
    data, slots, strategy, labels, cost, dev = load_fixture(name)
    r = oracle.replay_kpft(data, slots, strategy, labels, cost)
    stats = {s.label: s for s in oracle.region_stats(r.events, labels)}
    cp = oracle.critical_path(r.events, labels, dev_barrier_edges(dev))
    want = json.loads(_golden(name, "replay"))
    sim = R.SimTotals(want["total_cycles"], want["vanilla_cycles"], want["records_written"])
    assert R.dumps(R.replay_report(name, sim, stats, cp, r, cost)) == _golden(name, "replay")
    got = R.dumps(R.model_report(name, sim, stats, cp, cost, PARAMS.get(name)))
    assert got == _golden(name, "model")


def test_json_number_and_string_layout():
    assert R.dumps({"a": R.Double(0.0), "b": [], "c": {}, "d": -3,
                    "e": "q\"\\\n\x01é", "f": R.Double(1e16), "g": R.Double(0.1)}) == (
        '{\n  "a": 0.0,\n  "b": [],\n  "c": {},\n  "d": -3,\n'
        '  "e": "q\\"\\\\\\n\\u0001é",\n  "f": 1e+16,\n  "g": 0.1\n}\n')

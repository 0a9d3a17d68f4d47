"""GPU interval-overlap analysis (K6) against the oracle's restatement of
analyze_critical_path (perfmodel.hpp:317-501, O(n^2) gating) and the golden
fixture reports; role-overlap counters against the oracle definition."""
import json
import os

import numpy as np
import pytest

from conftest import FIXTURES, GOLDEN, load_fixture
from oracle import oracle as O
from test_oracle import dev_barrier_edges

pytestmark = pytest.mark.gpu


def T():
    from paper_2505_21661_b200 import trace
    return trace


LABELS = ["A", "A.wait", "B", "C", "C.wait", "Load K", "Load K.wait", "Z"]


def random_events(seed, n_chains=12, per_chain=60, labels=8, blocks=3, wgs=4):
    rng = np.random.default_rng(seed)
    evs = []
    it = {}
    for ch in range(n_chains):
        b, w = ch % blocks, (ch // blocks) % wgs
        t = int(rng.integers(0, 5000))
        for _ in range(per_chain):
            lab = int(rng.integers(0, labels))
            dur = int(rng.integers(0, 800))
            wait = LABELS[lab].endswith(".wait") and rng.random() < 0.8
            k = it.get(lab, 0)
            it[lab] = k + int(rng.integers(1, 3))
            region = lab | (O.EV_WAIT if wait else 0) | O.EV_CORRECTED
            evs.append((t, t + dur, region, k, b, w))
            t += dur + int(rng.integers(0, 300))
    ev = np.array(evs, O.EVENT_DTYPE)
    return ev[rng.permutation(len(ev))]


@pytest.mark.parametrize("gate_by_block", [False, True])
@pytest.mark.parametrize("seed", range(6))
def test_critical_path_vs_oracle(ctx, oracle, seed, gate_by_block):
    ev = random_events(seed)
    ctx.set_plan(T().BufferPlan(0, T().BufferStrategy.Flush, LABELS))
    edges = [("A", "C"), ("B", "Load K.wait")]
    want = oracle.critical_path(ev, LABELS, edges, gate_by_block=gate_by_block)
    got = ctx.critical_path(ev, edges, gate_by_block=gate_by_block)
    for k in ("stages", "mean", "steady", "wg", "binding", "cycle", "period"):
        assert got[k] == want[k], (k, got[k], want[k])


@pytest.mark.parametrize("name", FIXTURES)
def test_critical_path_fixtures(ctx, oracle, name):
    data, slots, strategy, labels, cost, dev = load_fixture(name)
    plan = T().BufferPlan(slots, T().BufferStrategy(strategy), labels)
    r = ctx.replay_image_bytes(data, plan, cost)
    edges = dev_barrier_edges(dev)
    got = ctx.critical_path(r.events, edges)
    want = oracle.critical_path(r.events, labels, edges)
    assert got == {k: want[k] for k in got}
    rep = json.load(open(os.path.join(GOLDEN, "fixtures", name + "_replay.json")))
    assert got["period"] == rep["iteration_period"]
    if got["cycle"]:
        assert got["cycle"] == rep["critical_path"]


def test_critical_path_missing_stage_error(ctx):
    ev = random_events(1)
    ctx.set_plan(T().BufferPlan(0, T().BufferStrategy.Flush, LABELS))
    with pytest.raises(T().Error, match='no events for stage "nope"'):
        ctx.critical_path(ev, [("A", "nope")])


@pytest.mark.parametrize("seed", range(4))
def test_overlap_counters_vs_oracle(ctx, oracle, seed):
    ev = random_events(100 + seed, n_chains=16, per_chain=80, blocks=4, wgs=4)
    roles = [0, 1, 1, 2]
    ctx.set_plan(T().BufferPlan(0, T().BufferStrategy.Flush, LABELS))
    assert ctx.overlap(ev, roles) == oracle.overlap(ev, roles)

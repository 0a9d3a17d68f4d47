"""CPU tests: pin the oracle (oracle/wgpf_oracle.c) against the reference's
golden vectors (tests/golden, regenerated from the reference by
tests/golden/gen_golden.py), the reference's own known-answer tests, and --
where the build container has it -- the reference itself."""
import json
import os

import numpy as np
import pytest

from conftest import (FIXTURES, GOLDEN, canon_golden, load_fixture,
                      load_random_set, load_synth)
from oracle import oracle as O
from oracle import synth as S
import fuzz

START = 0x80000000


def rec(is_start, region, clock, sig=0):
    return ((START if is_start else 0) | (region << 12) | sig, clock)


def recs(lst):
    a = np.empty(len(lst), np.dtype([("tag", "<u4"), ("payload", "<u4")]))
    for i, (t, p) in enumerate(lst):
        a[i] = (t, p)
    return a


def chrome_events(name, labels):
    """Chrome JSON (reference export_chrome_trace, trace.hpp:493-511) ->
    canonical events; ts/dur are cycles / 1000.0 as doubles."""
    doc = json.load(open(os.path.join(GOLDEN, "fixtures", name + ".json")))
    out = []
    for e in doc["traceEvents"]:
        s = round(e["ts"] * 1000)
        d = round(e["dur"] * 1000)
        assert s / 1000.0 == e["ts"] and d / 1000.0 == e["dur"]
        out.append((e["name"], e["pid"], e["tid"], s, s + d, e["args"]["iteration"],
                    e["args"]["kind"], e["args"]["corrected"]))
    return out


def oracle_tuples(ev, labels):
    out = []
    for e in ev:
        r = int(e["region"])
        out.append((O.label_of(labels, r & O.EV_REGION_MASK), int(e["block_index"]),
                    int(e["warp_group"]), int(e["start"]), int(e["end"]),
                    int(e["iteration"]), "wait" if r & O.EV_WAIT else "exec",
                    bool(r & O.EV_CORRECTED)))
    return out


# ---------------------------------------------------------------------------
# golden fixtures (the reference pipeline's own outputs)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_events_match_reference_chrome_trace(oracle, name):
    data, slots, strategy, labels, cost, _ = load_fixture(name)
    r = oracle.replay_kpft(data, slots, strategy, labels, cost)
    assert oracle_tuples(r.events, labels) == chrome_events(name, labels)


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_stats_match_reference_report(oracle, name):
    data, slots, strategy, labels, cost, _ = load_fixture(name)
    r = oracle.replay_kpft(data, slots, strategy, labels, cost)
    rep = json.load(open(os.path.join(GOLDEN, "fixtures", name + "_replay.json")))
    st = oracle.region_stats(r.events, labels)
    assert [s.label for s in st] == [x["region"] for x in rep["regions"]]
    for s, x in zip(st, rep["regions"]):
        assert (s.warp_group, s.kind, s.count, s.min, s.max) == (
            x["warp_group"], x["kind"], x["count"], x["min_duration"],
            x["max_duration"])
        assert s.mean == x["mean_duration"]  # bit-exact recurrence
    w = rep["warnings"]
    assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
            r.malformed_groups) == (w["dropped_heads"], w["truncated_tails"],
                                    w["flagged_preconditions"], w["malformed_groups"])


def dev_barrier_edges(dev):
    """Barrier edges of a .dev program, as perfmodel.hpp:258-313 derives them."""
    bodies, cur = [], None
    for line in dev.splitlines():
        t = line.strip()
        if t.startswith("wg") and t.endswith("{"):
            cur = []
            bodies.append(cur)
        elif cur is not None and t and t != "}":
            cur.append(t)
    labels = []
    for line in dev.splitlines():
        t = line.strip()
        if t.startswith("region "):
            labels.append(json.loads(t[t.index('"'):]))
    arrives, waits = [], []
    for body in bodies:
        for i, t in enumerate(body):
            if t.startswith("arrive "):
                for j in range(i - 1, -1, -1):
                    if body[j].startswith("store_counter") and body[j].endswith("end"):
                        rid = int(body[j].split("region=")[1].split()[0])
                        arrives.append((t.split()[1], labels[rid]))
                        break
            elif t.startswith("wait "):
                for j in range(i + 1, len(body)):
                    if body[j].startswith("store_counter") and body[j].endswith("start"):
                        rid = int(body[j].split("region=")[1].split()[0])
                        waits.append((t.split()[1], labels[rid]))
                        break
    edges = sorted({(a, w) for b1, a in arrives for b2, w in waits
                    if b1 == b2 and a != w})
    return edges


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_critical_path_matches_reference(oracle, name):
    data, slots, strategy, labels, cost, dev = load_fixture(name)
    r = oracle.replay_kpft(data, slots, strategy, labels, cost)
    cp = oracle.critical_path(r.events, labels, dev_barrier_edges(dev))
    rep = json.load(open(os.path.join(GOLDEN, "fixtures", name + "_replay.json")))
    assert cp["period"] == rep["iteration_period"]
    if cp["cycle"]:
        assert cp["cycle"] == rep["critical_path"]


def test_fixture_critical_path_vs_live_reference(oracle, reference):
    for name in FIXTURES:
        data, slots, strategy, labels, cost, dev = load_fixture(name)
        ref = reference.critical_path_kpft(data, dev, cost)
        r = oracle.replay_kpft(data, slots, strategy, labels, cost)
        assert dev_barrier_edges(dev) == ref["barrier_edges"]
        cp = oracle.critical_path(r.events, labels, ref["barrier_edges"])
        assert cp["cycle"] == ref["cycle"] and cp["period"] == ref["period"]
        assert cp["stages"] == ref["nodes"] and cp["mean"] == ref["durations"]


def test_deadlock_fixture_error_line():
    line = open(os.path.join(GOLDEN, "fixtures", "deadlock.err")).read()
    assert line.startswith("error: simulation-deadlock:") and "stuck" in line


# ---------------------------------------------------------------------------
# golden random programs (reference simulator + replay_image)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("setname", ["fidelity", "circular", "circular_flush",
                                     "replay100"])
def test_random_programs_match_reference(oracle, setname):
    n_ev = 0
    for img, slots, strategy, labels, res in load_random_set(setname):
        sp = O.LabelSpace()
        r = oracle.replay_kpft(img, slots, strategy, labels, 33)
        assert np.array_equal(O.canon_from_events(r.events, labels, sp),
                              canon_golden(res, sp))
        assert [r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups] == list(res["warnings"])
        st = oracle.region_stats(r.events, labels)
        assert [s.label for s in st] == list(res["stat_label"])
        assert [s.mean for s in st] == list(res["stat_mean"])
        assert [s.count for s in st] == list(res["stat_count"])
        assert [s.min for s in st] == list(res["stat_min"])
        assert [s.max for s in st] == list(res["stat_max"])
        assert [s.warp_group for s in st] == list(res["stat_wg"])
        n_ev += len(r.events)
    assert n_ev > 0


def test_circular_tail_equals_flush_tail(oracle):
    """test_acceptance.cpp:104-147 on the golden pairs of images."""
    circ = load_random_set("circular")
    flush = load_random_set("circular_flush")
    for (ci, cs, cst, _, _), (fi, fs, fst, _, _) in zip(circ, flush):
        t = oracle.decode_kpft(ci, cs, cst)
        f = oracle.decode_kpft(fi, fs, fst)
        for a, b in zip(t, f):
            n = min(len(b["records"]), 8)
            assert len(a["records"]) == n
            assert np.array_equal(a["records"], b["records"][len(b["records"]) - n:])


# ---------------------------------------------------------------------------
# synthetic configs 4 / 5 (slices) -- pins oracle/synth.py too
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("shape", ["mixed", "nested"])
def test_synth_slices_match_reference(oracle, shape):
    import hashlib
    g = load_synth(shape)
    if shape == "mixed":
        body, n, strategy, labels = (S.mixed_body(S.MIXED_FULL_LONG - 1024, 2048,
                                                  S.MIXED_FULL_LONG), 2048, 1,
                                     S.MIXED_LABELS)
    else:
        body, n, strategy, labels = S.nested_body(0, 1024), 1024, 0, S.NESTED_LABELS
    assert hashlib.sha256(body.tobytes()).hexdigest() == str(g["body_sha256"])
    r = oracle.replay_body(body, n, S.CAP, strategy, labels, 33)
    sp = O.LabelSpace()
    assert np.array_equal(O.canon_from_events(r.events, labels, sp),
                          O.canon_from_ref(g["events"], list(g["labels"]), sp))
    assert [r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
            r.malformed_groups] == list(g["warnings"])
    st = oracle.region_stats(r.events, labels)
    assert [s.mean for s in st] == list(g["stat_mean"])


def test_synth_known_answers(oracle):
    """producer 221->110 events / 1 tail, 222->111/0;
    consumer 221->109/3, 222->110/2; nested: 104 events, 24 heads, 24 tails."""
    for s0, long_ in ((0, 16), (16, 0)):
        body = S.mixed_body(s0, 16, long_)
        for s in range(16):
            one = body.reshape(16, -1)[s]
            r = oracle.replay_body(one, 1, S.CAP, 1, S.MIXED_LABELS, 33)
            prod = s < 4
            c = 222 if s0 + s < long_ else 221
            want = {(True, 221): (110, 1), (True, 222): (111, 0),
                    (False, 221): (109, 3), (False, 222): (110, 2)}[(prod, c)]
            assert (len(r.events), r.truncated_tails) == want
    r = oracle.replay_body(S.nested_body(0, 4), 4, S.CAP, 0, S.NESTED_LABELS, 33)
    assert (len(r.events), r.dropped_heads, r.truncated_tails) == (416, 96, 96)


def test_full_config4_event_total():
    """Config 4 totals 2^30 records and 531,791,872 events (closed form)."""
    n, n_long = S.MIXED_FULL_STREAMS, S.MIXED_FULL_LONG
    prod = lambda lo, hi: sum(1 for s in range(16) if s < 4) * 0  # noqa: E731
    del prod
    streams_long = n_long
    streams_short = n - n_long
    assert streams_long * 222 + streams_short * 221 == 1 << 30
    # per 16-stream block: 4 producers, 12 consumers
    ev_long = 4 * 111 + 12 * 110
    ev_short = 4 * 110 + 12 * 109
    assert (n_long // 16) * ev_long + (streams_short // 16) * ev_short == 531_791_872


# ---------------------------------------------------------------------------
# known answers from the reference's unit tests
# ---------------------------------------------------------------------------

def test_tag_layout_known_answers():
    """test_trace.cpp:9-27."""
    assert rec(True, 3, 1000)[0] == 0x80003000
    assert rec(False, 0, 0)[0] == 0
    assert rec(True, (1 << 19) - 1, 0, 0xFFF)[0] == 0xFFFFFFFF


def test_circular_capacity4_six_writes(oracle):
    """test_trace.cpp:82-105: slots [r4, r5, r2, r3] -> r2..r5."""
    body = np.array([0, 0, 6, 4] + [x for r in (4, 5, 2, 3)
                                    for x in rec(True, r, r)], np.uint32)
    img = S.kpft_v1(body.view(np.uint8), 1)
    d = oracle.decode_kpft(img, 4, 0)
    assert d[0]["dropped_records"] == 2
    assert [(t >> 12) & 0x7FFFF for t in d[0]["records"]["tag"]] == [2, 3, 4, 5]


def test_decode_errors(oracle):
    """test_trace.cpp:58-80,120-130 + trace.hpp:183-207,227-240."""
    body = np.array([0, 1, 0, 8] + [0] * 16, np.uint32)
    img = S.kpft_v1(body.view(np.uint8), 1)
    with pytest.raises(O.OracleError, match="does not match the buffer plan"):
        oracle.replay_kpft(img, 4, 0, [], 33)
    with pytest.raises(O.OracleError, match="truncated"):
        oracle.replay_kpft(img[:-1], 8, 0, [], 33)
    with pytest.raises(O.OracleError, match="trailing bytes"):
        oracle.replay_kpft(img + b"\0", 8, 0, [], 33)
    with pytest.raises(O.OracleError, match="bad magic"):
        oracle.replay_kpft(b"XPFT" + img[4:], 8, 0, [], 33)
    with pytest.raises(O.OracleError, match="unsupported trace version 3"):
        oracle.replay_kpft(img[:4] + b"\x03\x00" + img[6:], 8, 0, [], 33)
    over = np.array([0, 1, 9, 8] + [0] * 16, np.uint32)
    with pytest.raises(O.OracleError, match="flush stream claims"):
        oracle.replay_kpft(S.kpft_v1(over.view(np.uint8), 1), 8, 1, [], 33)


def test_unwrap_known_answers(oracle):
    """test_trace.cpp:132-141."""
    out = oracle.unwrap_clock([0xFFFFFF00, 0x00000100])
    assert out[1] - out[0] == 0x200
    assert list(oracle.unwrap_clock([10, 20, 4000])) == [10, 20, 4000]


def test_pairing_known_answers(oracle):
    """test_trace.cpp:156-214."""
    iv, dh, tt = oracle.pair_records(recs([rec(1, 0, 10), rec(0, 0, 20),
                                           rec(1, 0, 30), rec(0, 0, 40)]), ["a"])
    assert list(iv["iteration"]) == [0, 1] and dh == 0
    iv, _, _ = oracle.pair_records(recs([rec(1, 0, 10), rec(1, 1, 20), rec(0, 1, 30),
                                         rec(0, 0, 40)]), ["a", "b"])
    assert [tuple(x) for x in iv[["region_id", "start", "end"]]] == [(1, 20, 30),
                                                                      (0, 10, 40)]
    iv, dh, tt = oracle.pair_records(recs([rec(0, 0, 10)]), ["a"])
    assert len(iv) == 0 and dh == 1
    iv, dh, tt = oracle.pair_records(recs([rec(1, 0, 10)]), ["a"])
    assert len(iv) == 0 and tt == 1
    lst = [rec(1, 0, 0)]
    for i in range(1, 6):
        lst += [rec(1, 1, (i * 0x90000000) & 0xFFFFFFFF),
                rec(0, 1, (i * 0x90000000) & 0xFFFFFFFF)]
    lst.append(rec(0, 0, (5 * 0x90000000) & 0xFFFFFFFF))
    with pytest.raises(O.OracleError, match=r"2\^32"):
        oracle.pair_records(recs(lst), ["a", "b"])


def _iv(region, it, start, end, sp, ep):
    return (region, it, start, end, sp, ep)


def test_replay_known_answers(oracle):
    """test_replay.cpp:51-99."""
    iv = np.array([_iv(0, 0, 10, 150, 0, 1), _iv(1, 0, 400, 410, 2, 3)],
                  O.INTERVAL_DTYPE)
    r = oracle.replay_pairs(iv, ["G", "G.wait"], 0, 0, 33)
    w = r.events[1]
    assert (w["start"], w["end"]) == (150, 400) and w["region"] & O.EV_WAIT
    assert w["region"] & O.EV_CORRECTED
    iv = np.array([_iv(1, 0, 40, 80, 1, 2), _iv(0, 0, 10, 176, 0, 3)],
                  O.INTERVAL_DTYPE)
    r = oracle.replay_pairs(iv, ["outer", "inner"], 0, 0, 33)
    assert r.events[1]["end"] - r.events[1]["start"] == 166 - 33 - 2 * 33
    iv = np.array([_iv(0, 0, 10, 100, 0, 1), _iv(1, 0, 120, 130, 2, 3)],
                  O.INTERVAL_DTYPE)
    r = oracle.replay_pairs(iv, ["G", "G.wait"], 0, 0, 33)
    assert r.flagged_preconditions == 1
    assert not (r.events[1]["region"] & O.EV_CORRECTED)
    iv = np.array([_iv(1, 0, 120, 130, 0, 1)], O.INTERVAL_DTYPE)
    r = oracle.replay_pairs(iv, ["G", "G.wait"], 0, 0, 33)
    assert r.malformed_groups == 1 and len(r.events) == 1


def test_histogram_definition(oracle):
    """This framework's 64 half-octave bins (include/wgpf_format.h)."""
    from oracle.oracle import EVENT_DTYPE
    durs = [0, 1, 2, 3, 4, 5, 6, 7, 8, 11, 12, 15, 16, (1 << 32) - 1]
    ev = np.zeros(len(durs), EVENT_DTYPE)
    ev["end"] = durs
    st = oracle.region_stats(ev, ["r"])
    h = st[0].hist
    want = {0: 1, 1: 1, 2: 1, 3: 1, 4: 2, 5: 2, 6: 2, 7: 2, 8: 1, 63: 1}
    assert {i: v for i, v in enumerate(h) if v} == want


# ---------------------------------------------------------------------------
# fuzz: oracle == reference on edge-case images (needs oracle/_ref)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("mode", ["nested", "random"])
def test_fuzz_oracle_vs_reference(oracle, reference, mode):
    for seed in range(60):
        data, cap, strategy, labels = fuzz.random_image(
            seed, n_streams=6, cap=32, mode=mode, big_gaps=(seed % 3 == 0))
        try:
            rr = reference.replay_kpft(data, cap, strategy, labels, 33)
            rerr = None
        except O.OracleError as e:
            rr, rerr = None, (e.category, str(e))
        try:
            r = oracle.replay_kpft(data, cap, strategy, labels, 33)
            oerr = None
        except O.OracleError as e:
            r, oerr = None, (e.category, str(e))
        assert rerr == oerr, (seed, rerr, oerr)
        if rerr:
            continue
        sp = O.LabelSpace()
        assert np.array_equal(O.canon_from_events(r.events, labels, sp),
                              O.canon_from_ref(rr.events, rr.labels, sp)), seed
        assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups) == (rr.dropped_heads, rr.truncated_tails,
                                        rr.flagged_preconditions,
                                        rr.malformed_groups)
        st = oracle.region_stats(r.events, labels)
        assert [(s.label, s.warp_group, s.kind, s.count, s.min, s.max, s.mean)
                for s in st] == [(s.label, s.warp_group, s.kind, s.count, s.min,
                                  s.max, s.mean) for s in rr.stats], seed


# ---------------------------------------------------------------------------
# Chrome Trace numbers: Grisu2 as the reference's JSON library prints doubles
# ---------------------------------------------------------------------------

JSON_DIR = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/"
            "cudnn_frontend/thirdparty/nlohmann")


def test_grisu2_matches_reference_json_library(tmp_path):
    """include/wgpf_grisu2.h (shared by the host and GPU Chrome exporters)
    prints every double byte-identically to nlohmann/json 3.11.3 -- including
    the values where Grisu2 is not the shortest round trip (std::to_chars)."""
    import subprocess
    if not os.path.exists(os.path.join(JSON_DIR, "json.hpp")):
        pytest.skip("nlohmann/json header not in this image")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "grisu2_test")
    res = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"),
                          "-I", JSON_DIR, os.path.join(root, "tests", "cxx", "grisu2_test.cpp"),
                          "-o", exe], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-2000:]
    res = subprocess.run([exe, "1000000", "11"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:]


@pytest.mark.parametrize("name", FIXTURES)
def test_reference_chrome_export_entry_point(reference, oracle, name):
    """oracle/_ref's export_chrome_trace entry point reproduces the shipped
    out/<fixture>.json byte for byte from the oracle's events."""
    data, slots, strategy, labels, cost, _ = load_fixture(name)
    r = oracle.replay_kpft(data, slots, strategy, labels, cost)
    got = reference.export_chrome(r.events, labels, 1000.0)
    assert got == open(os.path.join(GOLDEN, "fixtures", name + ".json")).read()


@pytest.mark.parametrize("name", FIXTURES)
def test_device_program_side_channel(name):
    """trace.parse_device_program (the .dev side channel, lower.hpp:320-380)
    gives the fixture's plan and the barrier edges perfmodel.hpp:258-313
    derives (the test-side parser above is the independent check)."""
    from paper_2505_21661_b200 import trace as T
    data, slots, strategy, labels, cost, dev = load_fixture(name)
    dp = T.parse_device_program(dev)
    assert dp.plan.slots_per_warp_group == slots
    assert int(dp.plan.strategy) == strategy
    assert dp.plan.region_labels == labels
    assert dp.barrier_edges == dev_barrier_edges(dev)
    assert dp.num_warp_groups > 0 and dp.name

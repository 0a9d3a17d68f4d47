"""GPU parity: the sm_100a replay path (through the C-ABI) against the
reference's golden vectors, the CPU oracle, and the reference's known-answer
tests -- bit-exact on every integer output, bit-exact means in exact mode."""
import json
import os

import numpy as np
import pytest

from conftest import (FIXTURES, GOLDEN, canon_golden, load_fixture,
                      load_random_set, load_synth)
from oracle import oracle as O
from oracle import synth as S
import fuzz

pytestmark = pytest.mark.gpu

FLAG_MODES = {"fast": 0, "general": 0x4}


def T():
    from paper_2505_21661_b200 import trace
    return trace


def plan_of(slots, strategy, labels):
    t = T()
    return t.BufferPlan(slots, t.BufferStrategy(strategy), list(labels))


def same_events(ev, labels, ref_canon, space):
    return np.array_equal(O.canon_from_events(ev, labels, space), ref_canon)


# ---------------------------------------------------------------------------
# golden fixtures
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("mode", list(FLAG_MODES))
@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_replay(ctx, oracle, name, mode):
    data, slots, strategy, labels, cost, _ = load_fixture(name)
    r = ctx.replay_image_bytes(data, plan_of(slots, strategy, labels), cost,
                               flags=FLAG_MODES[mode] | 0x2)
    o = oracle.replay_kpft(data, slots, strategy, labels, cost)
    assert np.array_equal(r.events, o.events)
    rep = json.load(open(os.path.join(GOLDEN, "fixtures", name + "_replay.json")))
    w = rep["warnings"]
    assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
            r.malformed_groups) == (w["dropped_heads"], w["truncated_tails"],
                                    w["flagged_preconditions"], w["malformed_groups"])
    st = ctx.stats()
    assert list(st) == [x["region"] for x in rep["regions"]]
    for x in rep["regions"]:
        s = st[x["region"]]
        assert (s.warp_group, s.kind, s.count, s.min, s.max) == (
            x["warp_group"], x["kind"], x["count"], x["min_duration"],
            x["max_duration"])
        assert s.mean == x["mean_duration"]  # bit-exact recurrence (H1 a)


# ---------------------------------------------------------------------------
# golden random programs
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("mode", list(FLAG_MODES))
@pytest.mark.parametrize("setname", ["fidelity", "circular", "circular_flush",
                                     "replay100"])
def test_random_programs(ctx, setname, mode):
    for img, slots, strategy, labels, res in load_random_set(setname):
        r = ctx.replay_image_bytes(img, plan_of(slots, strategy, labels), 33,
                                   flags=FLAG_MODES[mode] | 0x2)
        sp = O.LabelSpace()
        assert same_events(r.events, labels, canon_golden(res, sp), sp)
        assert [r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups] == list(res["warnings"])
        st = ctx.stats()
        assert list(st) == list(res["stat_label"])
        assert [s.mean for s in st.values()] == list(res["stat_mean"])
        assert [s.count for s in st.values()] == list(res["stat_count"])
        assert [s.min for s in st.values()] == list(res["stat_min"])
        assert [s.max for s in st.values()] == list(res["stat_max"])
        assert [s.warp_group for s in st.values()] == list(res["stat_wg"])
        assert [s.kind == "wait" for s in st.values()] == list(res["stat_kind"])


# ---------------------------------------------------------------------------
# synthetic configs (slices) and the GPU synthetic generator
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("mode", list(FLAG_MODES))
@pytest.mark.parametrize("shape", ["mixed", "nested"])
def test_synth_slices(ctx, shape, mode):
    g = load_synth(shape)
    if shape == "mixed":
        body, n, strategy, labels = (S.mixed_body(S.MIXED_FULL_LONG - 1024, 2048,
                                                  S.MIXED_FULL_LONG), 2048, 1,
                                     S.MIXED_LABELS)
        img = S.kpft_v1(body, n)
    else:
        body, n, strategy, labels = S.nested_body(0, 1024), 1024, 0, S.NESTED_LABELS
        img = S.kpft_v2(body, n)  # v2 container
    r = ctx.replay_image_bytes(img, plan_of(S.CAP, strategy, labels), 33,
                               flags=FLAG_MODES[mode] | 0x2)
    sp = O.LabelSpace()
    assert same_events(r.events, labels,
                       O.canon_from_ref(g["events"], list(g["labels"]), sp), sp)
    assert [r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
            r.malformed_groups] == list(g["warnings"])
    st = ctx.stats()
    assert [s.mean for s in st.values()] == list(g["stat_mean"])
    assert [s.count for s in st.values()] == list(g["stat_count"])


@pytest.mark.parametrize("shape", [0, 1])
def test_gpu_synth_generator_matches_cpu(ctx, shape):
    import torch
    n, s0 = 3000, S.MIXED_FULL_LONG - 1500
    if shape == 1:
        s0 = 123456
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), shape, s0, n, S.MIXED_FULL_LONG)
    torch.cuda.synchronize()
    cpu = S.mixed_body(s0, n, S.MIXED_FULL_LONG) if shape == 0 else \
        S.nested_body(s0, n)
    assert np.array_equal(body.cpu().numpy(), cpu)


# ---------------------------------------------------------------------------
# fuzz vs the oracle (edge cases: crossings, out-of-table ids, duplicate
# labels, orphans, clock wraps, errors)
# ---------------------------------------------------------------------------

# record costs around the thread-per-stream kernel's bound (cost < 2^21 keeps
# cost x position in 32 bits; larger costs route to the warp-per-stream path)
COSTS = [33, 0, 1, (1 << 21) - 1, 1 << 21, (1 << 32) + 5]


@pytest.mark.parametrize("mode", ["nested", "random"])
@pytest.mark.parametrize("path", list(FLAG_MODES))
def test_fuzz_vs_oracle(ctx, oracle, mode, path):
    t = T()
    for seed in range(80):
        data, cap, strategy, labels = fuzz.random_image(
            1000 + seed, n_streams=12, cap=32 if seed % 2 else 64, mode=mode,
            big_gaps=(seed % 3 == 0))
        cost = COSTS[seed % len(COSTS)] if seed >= 40 else 33
        try:
            o = oracle.replay_kpft(data, cap, strategy, labels, cost)
            oerr = None
        except O.OracleError as e:
            o, oerr = None, (e.category, str(e))
        try:
            r = ctx.replay_image_bytes(data, plan_of(cap, strategy, labels), cost,
                                       flags=FLAG_MODES[path] | 0x2)
            gerr = None
        except t.Error as e:
            r, gerr = None, (e.category(), str(e))
        assert oerr == gerr, (seed, oerr, gerr)
        if oerr:
            continue
        assert np.array_equal(r.events, o.events), seed
        assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups) == (o.dropped_heads, o.truncated_tails,
                                        o.flagged_preconditions, o.malformed_groups)
        want = oracle.region_stats(o.events, labels)
        got = ctx.stats()
        assert list(got) == [s.label for s in want], seed
        for s in want:
            g = got[s.label]
            assert (g.warp_group, g.kind, g.count, g.min, g.max, g.sum, g.mean,
                    g.first_event, g.hist) == (s.warp_group, s.kind, s.count, s.min,
                                               s.max, s.sum, s.mean, s.first_event,
                                               s.hist), (seed, s.label)


def test_errors_match_reference_messages(ctx, oracle):
    t = T()
    body = np.array([0, 1, 0, 8] + [0] * 16, np.uint32)
    img = S.kpft_v1(body.view(np.uint8), 1)
    cases = [(img, 4, "does not match the buffer plan (4)"),
             (img[:-1], 8, "truncated trace image"),
             (img + b"\0", 8, "trailing bytes after trace image"),
             (b"XPFT" + img[4:], 8, "bad magic: not a trace image"),
             (img[:4] + b"\x03\x00" + img[6:], 8, "unsupported trace version 3")]
    for data, slots, msg in cases:
        with pytest.raises(t.Error) as ei:
            ctx.replay_image_bytes(data, plan_of(slots, 0, []), 33)
        assert ei.value.category() == "trace-error" and msg in str(ei.value)
        with pytest.raises(O.OracleError) as eo:
            oracle.replay_kpft(data, slots, 0, [], 33)
        assert str(eo.value) == str(ei.value)


# ---------------------------------------------------------------------------
# reference known answers through the C-ABI
# ---------------------------------------------------------------------------

def test_known_answers_unit_entry_points(ctx):
    t = T()
    P = t.ProfileRecord.make
    assert P(True, 3, 0, 1000).tag == 0x80003000                 # test_trace:9
    img = t.GlobalTraceImage([t.TraceStream(0, 1, 6, 4, [P(True, 4, 0, 4),
                                                         P(True, 5, 0, 5),
                                                         P(True, 2, 0, 2),
                                                         P(True, 3, 0, 3)])])
    d = ctx.decode_image_bytes(t.serialize_image(img),
                               t.BufferPlan(4, t.BufferStrategy.Circular, []))
    assert d[0].dropped_records == 2                             # test_trace:82
    assert [(int(x) >> 12) & 0x7FFFF for x in d[0].records["tag"]] == [2, 3, 4, 5]
    u = ctx.unwrap_clock([0xFFFFFF00, 0x00000100])               # test_trace:132
    assert int(u[1] - u[0]) == 0x200
    assert list(ctx.unwrap_clock([10, 20, 4000])) == [10, 20, 4000]
    pr = ctx.pair_records(t.records_array([P(True, 0, 0, 10), P(True, 1, 0, 20),
                                           P(False, 1, 0, 30), P(False, 0, 0, 40)]),
                          ["a", "b"])                            # test_trace:171
    assert [(int(a), int(b), int(c)) for a, b, c in
            pr.intervals[["region_id", "start", "end"]]] == [(1, 20, 30), (0, 10, 40)]
    pr = ctx.pair_records(t.records_array([P(False, 0, 0, 10)]), ["a"])
    assert pr.dropped_heads == 1 and len(pr.intervals) == 0
    lst = [P(True, 0, 0, 0)]
    for i in range(1, 6):
        c = (i * 0x90000000) & 0xFFFFFFFF
        lst += [P(True, 1, 0, c), P(False, 1, 0, c)]
    lst.append(P(False, 0, 0, (5 * 0x90000000) & 0xFFFFFFFF))
    with pytest.raises(t.Error, match=r"exceeds 2\^32"):      # test_trace:203
        ctx.pair_records(t.records_array(lst), ["a", "b"])
    iv = np.array([(0, 0, 10, 150, 0, 1), (1, 0, 400, 410, 2, 3)], t.INTERVAL_DTYPE)
    rr = ctx.replay(iv, ["G", "G.wait"], 0, 0, 33)             # test_replay:51
    assert (int(rr.events[1]["start"]), int(rr.events[1]["end"])) == (150, 400)
    iv = np.array([(1, 0, 40, 80, 1, 2), (0, 0, 10, 176, 0, 3)], t.INTERVAL_DTYPE)
    rr = ctx.replay(iv, ["outer", "inner"], 0, 0, 33)          # test_replay:66
    assert int(rr.events[1]["end"] - rr.events[1]["start"]) == 67
    iv = np.array([(0, 0, 10, 100, 0, 1), (1, 0, 120, 130, 2, 3)], t.INTERVAL_DTYPE)
    rr = ctx.replay(iv, ["G", "G.wait"], 0, 0, 33)             # test_replay:81
    assert rr.flagged_preconditions == 1
    iv = np.array([(1, 0, 120, 130, 0, 1)], t.INTERVAL_DTYPE)
    rr = ctx.replay(iv, ["G", "G.wait"], 0, 0, 33)             # test_replay:92
    assert rr.malformed_groups == 1 and len(rr.events) == 1


# ---------------------------------------------------------------------------
# device-resident bodies at scale
# ---------------------------------------------------------------------------

def _device_replay(ctx, shape, s0, n, flags=0):
    import torch
    labels = S.MIXED_LABELS if shape == 0 else S.NESTED_LABELS
    strategy = 1 if shape == 0 else 0
    ctx.set_plan(plan_of(S.CAP, strategy, labels))
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), shape, s0, n, S.MIXED_FULL_LONG)
    cap = n * 128
    ev = torch.empty(cap * 32, dtype=torch.uint8, device="cuda")
    ne, w = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, ev.data_ptr(),
                              cap, flags)
    return body, ev, ne, w, labels, strategy


@pytest.mark.parametrize("shape", [0, 1])
def test_device_body_vs_oracle_64k_streams(ctx, oracle, shape):
    n = 1 << 16
    s0 = S.MIXED_FULL_LONG - n // 2
    body, ev, ne, w, labels, strategy = _device_replay(ctx, shape, s0, n, 0x2)
    o = oracle.replay_body(body.cpu().numpy(), n, S.CAP, strategy, labels, 33)
    got = ev[:ne * 32].cpu().numpy().view(O.EVENT_DTYPE)
    assert ne == len(o.events)
    assert np.array_equal(got, o.events)
    assert (w.dropped_heads, w.truncated_tails, w.flagged_preconditions,
            w.malformed_groups) == (o.dropped_heads, o.truncated_tails,
                                    o.flagged_preconditions, o.malformed_groups)
    want = oracle.region_stats(o.events, labels)
    st = ctx.stats()
    for s in want:
        g = st[s.label]
        assert (g.count, g.min, g.max, g.sum, g.mean, g.warp_group, g.kind,
                g.first_event, g.hist) == (s.count, s.min, s.max, s.sum, s.mean,
                                           s.warp_group, s.kind, s.first_event,
                                           s.hist)


def test_overlapped_pass1_pass2_equals_sequential(ctx, monkeypatch):
    """The opt-in overlapped replay (WGPF_OVERLAP=1: pass 1 of chunk k+1 on a
    second stream beside k_tps on chunk k, chunked offset scans with a
    device-side running base) gives the sequential replay's events,
    warnings and statistics bit for bit."""
    import torch
    from paper_2505_21661_b200 import trace as T
    n = 1 << 16
    s0 = S.MIXED_FULL_LONG - n // 2
    body, ev, ne, w, labels, strategy = _device_replay(ctx, 0, s0, n, 0x2)
    want_ev = ev[:ne * 32].clone()
    want_st = ctx.stats()
    monkeypatch.setenv("WGPF_OVERLAP", "1")
    octx = T.Context(0)
    octx.set_plan(plan_of(S.CAP, strategy, labels))
    ev2 = torch.zeros_like(ev)
    ne2, w2 = octx.replay_device(body.data_ptr(), body.numel(), n, 33, ev2.data_ptr(),
                                 n * 128, 0x2 | 0x10)
    assert octx.last_profile()["overlap_chunks"] > 1
    assert ne2 == ne
    assert torch.equal(ev2[:ne * 32], want_ev)
    assert (w2.dropped_heads, w2.truncated_tails, w2.flagged_preconditions,
            w2.malformed_groups) == (w.dropped_heads, w.truncated_tails,
                                     w.flagged_preconditions, w.malformed_groups)
    assert octx.stats() == want_st


@pytest.mark.slow
def test_full_config4_properties(ctx, oracle):
    """Full 2^30-record config 4 on one B200: closed-form totals plus a
    sample of streams checked against the oracle event for event."""
    import torch
    n = S.MIXED_FULL_STREAMS
    body, ev, ne, w, labels, strategy = _device_replay(ctx, 0, 0, n, 0)
    assert ne == 531_791_872
    n_long = S.MIXED_FULL_LONG
    tails = (n_long // 16) * (4 * 0 + 12 * 2) + ((n - n_long) // 16) * (4 * 1 + 12 * 3)
    assert (w.dropped_heads, w.truncated_tails, w.malformed_groups) == (0, tails, 0)
    st = ctx.stats()
    assert sum(s.count for s in st.values()) == ne
    rng = np.random.default_rng(4)
    counts = np.where(np.arange(n) < n_long, 0, 0)
    del counts
    stride = S.stream_stride()
    for s in sorted(rng.choice(n, 64, replace=False)):
        s = int(s)
        one = body[s * stride:(s + 1) * stride].cpu().numpy()
        o = oracle.replay_body(one, 1, S.CAP, 1, labels, 33)
        # event offset of stream s: closed form over the 16-stream blocks
        blk, lane = divmod(s, 16)
        def per(gs):
            long_ = gs < n_long
            return (111 if long_ else 110) if gs % 16 < 4 else (110 if long_ else 109)
        off = 0
        full_long_blocks = min(blk, n_long // 16)
        off += full_long_blocks * (4 * 111 + 12 * 110)
        off += (blk - full_long_blocks) * (4 * 110 + 12 * 109)
        off += sum(per(blk * 16 + k) for k in range(lane))
        got = ev[off * 32:(off + len(o.events)) * 32].cpu().numpy().view(O.EVENT_DTYPE)
        assert np.array_equal(got, o.events), s
    del body, ev
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_full_config5_properties(ctx, oracle):
    """Full config 5 on one B200 (2^22 circular 64-deep streams, 2^30
    surviving records): closed-form totals and per-label counts, plus a
    sample of streams checked against the oracle event for event."""
    import torch
    n = S.NESTED_FULL_STREAMS
    body, ev, ne, w, labels, strategy = _device_replay(ctx, 1, 0, n, 0)
    # surviving window = writes 744..999 of S0..S63 E63..E0 repeated: 24 dropped
    # heads (E23..E0), then S0..S63 E63..E0 S0..S63 E63..E24: 104 events and
    # 24 open STARTs per stream
    per = 104
    assert ne == per * n
    assert (w.dropped_heads, w.truncated_tails, w.malformed_groups,
            w.flagged_preconditions) == (24 * n, 24 * n, 0, 0)
    st = ctx.stats()
    for k, lab in enumerate(labels):
        assert st[lab].count == (2 if k >= 24 else 1) * n, lab
    rng = np.random.default_rng(5)
    stride = S.stream_stride()
    for s in sorted(rng.choice(n, 64, replace=False)):
        s = int(s)
        one = body[s * stride:(s + 1) * stride].cpu().numpy()
        o = oracle.replay_body(one, 1, S.CAP, 0, labels, 33)
        assert len(o.events) == per
        got = ev[s * per * 32:(s + 1) * per * 32].cpu().numpy().view(O.EVENT_DTYPE)
        # (the oracle numbers the stream 0 and block / warp group come from
        # the header, so the records compare as they are)
        assert np.array_equal(got, o.events), s
    del body, ev
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("shape,switch", [(0, "WGPF_NO_TPS"), (1, "WGPF_NO_DEEP")])
def test_full_size_fast_kernel_equals_warp_kernel(ctx, monkeypatch, shape, switch):
    """Differential check at the full BASELINE sizes: the thread-per-stream
    kernel (k_tps on config 4, k_tpsd on config 5) and the independent
    warp-per-stream kernel (k_fast_emit: ballots, match.any, per-level
    tables), each pinned to the oracle on smaller bodies, give the same 531.8
    M / 436.2 M events bit for bit and the same statistics."""
    import torch
    from paper_2505_21661_b200 import trace as T
    n = S.MIXED_FULL_STREAMS if shape == 0 else S.NESTED_FULL_STREAMS
    body, ev, ne, w, labels, strategy = _device_replay(ctx, shape, 0, n, 0x2)
    want_st = ctx.stats()
    monkeypatch.setenv(switch, "1")
    wctx = T.Context(0)
    wctx.set_plan(plan_of(S.CAP, strategy, labels))
    ev2 = torch.empty_like(ev)
    ne2, w2 = wctx.replay_device(body.data_ptr(), body.numel(), n, 33, ev2.data_ptr(),
                                 n * 128, 0x2)
    assert ne2 == ne
    assert torch.equal(ev2[:ne * 32], ev[:ne * 32])
    assert (w2.dropped_heads, w2.truncated_tails, w2.flagged_preconditions,
            w2.malformed_groups) == (w.dropped_heads, w.truncated_tails,
                                     w.flagged_preconditions, w.malformed_groups)
    assert wctx.stats() == want_st
    del body, ev, ev2
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [4000, 40000])
def test_stats_only_equals_materialized(ctx, oracle, n):
    """WGPF_F_STATS_ONLY (no event materialisation) gives the same
    statistics as the full replay and as the oracle."""
    import torch
    ctx.set_plan(plan_of(S.CAP, 1, S.MIXED_LABELS))
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), 0, S.MIXED_FULL_LONG - n // 2, n, S.MIXED_FULL_LONG)
    ctx.replay_device(body.data_ptr(), body.numel(), n, 33, 0, 0, 0x1)
    only = ctx.stats()
    ev = torch.empty(n * 128 * 32, dtype=torch.uint8, device="cuda")
    ctx.replay_device(body.data_ptr(), body.numel(), n, 33, ev.data_ptr(), n * 128, 0)
    full = ctx.stats()
    o = oracle.replay_body(body.cpu().numpy(), n, S.CAP, 1, S.MIXED_LABELS, 33)
    want = {s.label: s for s in oracle.region_stats(o.events, S.MIXED_LABELS)}
    for k, s in want.items():
        for got in (only[k], full[k]):
            assert (got.count, got.sum, got.min, got.max, got.hist) == (
                s.count, s.sum, s.min, s.max, s.hist), k


def test_replay_image_pipelined_matches_device(ctx):
    """Images over 512 MB with host event output take the chunked pipeline
    (H2D / replay / D2H overlapped over 256 MB chunks): events, warnings and
    statistics (incl. first-event indices) equal one device-resident replay
    of the same body; a too-small event buffer reports the full count."""
    import torch
    t = T()
    n = 300000  # 619 MB of config-4 streams: three chunks
    plan = plan_of(S.CAP, 1, S.MIXED_LABELS)
    ctx.set_plan(plan)
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), 0, 0, n, n // 3)
    ne, _ = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, 0, 0, 0x1)
    dev_ev = torch.empty(ne * 32, dtype=torch.uint8, device="cuda")
    ne2, w = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, dev_ev.data_ptr(), ne, 0)
    assert ne2 == ne
    whole = ctx.stats()
    hdr = b"KPFT" + (2).to_bytes(2, "little") + b"\0\0" + n.to_bytes(8, "little")
    img = hdr + body.cpu().numpy().tobytes()
    c2 = t.Context(0)
    r = c2.replay_image_bytes(img, plan, 33, events_cap=7)  # E_BUFFER -> retry
    assert len(r.events) == ne
    assert r.events.tobytes() == dev_ev.cpu().numpy().tobytes()
    assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
            r.malformed_groups) == (w.dropped_heads, w.truncated_tails,
                                    w.flagged_preconditions, w.malformed_groups)
    assert c2.stats() == whole


def test_replay_image_pipelined_error_order(ctx, reference):
    """The reference decodes every stream before pairing any
    (pipeline.hpp:69-80 -> decode_image first), so a decode error in a late
    chunk of the pipelined path must win over a pair error (duration >= 2^32)
    in chunk 0, as in the reference on the same streams."""
    import torch
    t = T()
    n = 300000  # three chunks
    plan = plan_of(S.CAP, 1, S.MIXED_LABELS)
    ctx.set_plan(plan)
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), 0, 0, n, n // 3)
    b = body.cpu().numpy()
    st = S.stream_stride()
    # stream 5 (a consumer: S4 S5 S6 S7 E7 E6 ...): the gaps of records 1..7
    # grow by 2^31 + 1, so E6 closes S6 3 (2^31 + 1) > 2^32 cycles later ->
    # the reference's pair error
    w = b[5 * st:6 * st].view(np.uint32)
    clk = w[5:4 + 2 * 221:2].astype(np.int64)
    k = np.minimum(np.arange(len(clk)), 7)
    w[5:4 + 2 * 221:2] = ((clk + k * 0x80000001) & 0xFFFFFFFF).astype(np.uint32)
    # stream 290000 (chunk 2): a flush stream claiming more records than slots
    h = b[290000 * st:290000 * st + 16].view(np.uint32)
    h[2] = S.CAP + 1
    hdr = b"KPFT" + (2).to_bytes(2, "little") + b"\0\0" + n.to_bytes(8, "little")
    img = hdr + b.tobytes()
    with pytest.raises(t.Error) as e:
        t.Context(0).replay_image_bytes(img, plan, 33)
    # the reference on the streams that matter (v1 images of <= 65,535 streams)
    sub = np.concatenate([b[0:64 * st], b[290000 * st:290001 * st]])
    v1 = b"KPFT" + (1).to_bytes(2, "little") + (65).to_bytes(2, "little") + sub.tobytes()
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as er:
        reference.replay_kpft(v1, S.CAP, 1, S.MIXED_LABELS, 33)
    assert str(e.value) == str(er.value) == "flush stream claims more records than slots"
    # without the decode error the pair error is reported
    h[2] = 221
    with pytest.raises(t.Error) as e2:
        t.Context(0).replay_image_bytes(hdr + b.tobytes(), plan, 33)
    with pytest.raises(OracleError) as er2:
        reference.replay_kpft(b"KPFT" + (1).to_bytes(2, "little") + (64).to_bytes(2, "little")
                              + b[0:64 * st].tobytes(), S.CAP, 1, S.MIXED_LABELS, 33)
    assert str(e2.value) == str(er2.value)


def test_stats_merge_two_shards(ctx):
    """Multi-GPU shard-and-reduce on one device: two shards of a body, each
    replayed with its stream_base, stats exported, gathered and merged,
    equal the single-shot stats (integer fields and first-event keys)."""
    import torch
    t = T()
    n = 40000
    labels = S.MIXED_LABELS
    plan = plan_of(S.CAP, 1, labels)
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.set_plan(plan)
    ctx.synth_body(body.data_ptr(), 0, S.MIXED_FULL_LONG - n // 2, n, S.MIXED_FULL_LONG)
    ctx.replay_device(body.data_ptr(), body.numel(), n, 33, 0, 0, 0x1)
    whole = ctx.stats()
    parts = [t.Context(0), t.Context(0)]
    assert parts[0].stats_packed_bytes() == 0  # size needs the plan
    for c in parts:
        c.set_plan(plan)
    pb = parts[0].stats_packed_bytes()
    gathered = torch.zeros(2 * pb, dtype=torch.uint8, device="cuda")
    cut = 17003
    stride = S.stream_stride()
    for r, (a, b) in enumerate([(0, cut), (cut, n)]):
        c = parts[r]
        c.replay_device(body.data_ptr() + a * stride, (b - a) * stride, b - a, 33,
                        0, 0, 0x1, stream_base=a)
        c.stats_export(gathered.data_ptr() + r * pb)
    torch.cuda.synchronize()
    part_counts = [p.stats() for p in parts]
    for k in whole:
        assert whole[k].count == sum(pc[k].count for pc in part_counts if k in pc), k
    g = gathered.cpu().numpy().view(np.uint64)
    per = pb // 8
    for r in range(2):
        for i, k in enumerate(S.MIXED_LABELS):
            assert int(g[r * per + i * 70]) == part_counts[r][k].count, (r, k)
    merged_ctx = t.Context(0)
    merged_ctx.set_plan(plan)
    merged_ctx.stats_merge(gathered.data_ptr(), 2)
    merged = merged_ctx.stats()
    extra = {k: (v.count, v.sum) for k, v in merged.items() if k not in whole}
    assert list(merged) == list(whole), extra
    for k in whole:
        a, b = whole[k], merged[k]
        assert (a.count, a.sum, a.min, a.max, a.warp_group, a.kind, a.hist) == (
            b.count, b.sum, b.min, b.max, b.warp_group, b.kind, b.hist)


def test_cxx_shim_end_to_end(tmp_path):
    """The drop-in C++ shim (reference signatures) against libwgpf.so."""
    import subprocess
    from paper_2505_21661_b200 import _build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "shim_test")
    lib = _build.build()
    res = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                          os.path.join(root, "tests", "cxx", "shim_test.cpp"),
                          lib, f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", exe],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    from paper_2505_21661_b200 import trace as tr
    dp = tr.parse_device_program(open(os.path.join(GOLDEN, "fixtures",
                                                   "fa3_vanilla.dev")).read())
    edges = tmp_path / "edges.tsv"
    edges.write_text("".join(f"{a}\t{b}\n" for a, b in dp.barrier_edges))
    res = subprocess.run([exe, os.path.join(GOLDEN, "fixtures"), str(edges)],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "ALL PASS" in res.stdout


@pytest.mark.parametrize("name", FIXTURES)
def test_chrome_trace_export_byte_identical(ctx, name):
    """export_chrome_trace (trace.hpp:493-511) vs the reference's own JSON
    (fixtures regenerated byte-identically to proj/out/*.json)."""
    data, slots, strategy, labels, cost, _ = load_fixture(name)
    r = ctx.replay_image_bytes(data, plan_of(slots, strategy, labels), cost)
    got = ctx.export_chrome_trace(r.events, 1000.0)
    want = open(os.path.join(GOLDEN, "fixtures", name + ".json")).read()
    assert got == want


def test_chrome_trace_export_empty_and_escaping(ctx):
    t = T()
    ctx.set_plan(plan_of(4, 1, ['we"ird\\lab\tel']))
    assert ctx.export_chrome_trace(np.zeros(0, O.EVENT_DTYPE)) == \
        '{\n  "traceEvents": []\n}\n'
    ev = np.array([(0, 1000, 0 | O.EV_CORRECTED, 0, 1, 2)], O.EVENT_DTYPE)
    js = ctx.export_chrome_trace(ev)
    import json as J
    d = J.loads(js)["traceEvents"][0]
    assert d["name"] == 'we"ird\\lab\tel' and d["dur"] == 1.0 and d["pid"] == 1
    del t


def random_chrome_events(seed, n, n_labels):
    rng = np.random.default_rng(seed)
    start = rng.integers(0, 1 << 62, n, dtype=np.uint64) >> rng.integers(0, 62, n).astype(np.uint64)
    dur = rng.integers(0, 1 << 40, n, dtype=np.uint64) >> rng.integers(0, 40, n).astype(np.uint64)
    rid = rng.integers(0, n_labels + 40, n).astype(np.uint32)   # some out of table
    flags = rng.integers(0, 4, n).astype(np.uint32) << 30
    ev = np.zeros(n, O.EVENT_DTYPE)
    ev["start"], ev["end"] = start, start + dur
    ev["region"] = rid | flags
    ev["iteration"] = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32) >> \
        rng.integers(0, 32, n).astype(np.uint32)
    ev["block_index"] = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32) >> \
        rng.integers(0, 32, n).astype(np.uint32)
    ev["warp_group"] = rng.integers(0, 64, n).astype(np.uint32)
    return ev


@pytest.mark.parametrize("cpu", [1000.0, 1965.0, 1.0, 0.37])
def test_chrome_trace_gpu_formatter_vs_reference(ctx, reference, cpu):
    """The GPU formatter (events in HBM, k_chrome.cuh) and the host writer
    produce the reference's own export_chrome_trace text byte for byte on
    random events: 2^62-scale clocks, B200 cycles_per_us = 1965 (17-digit
    doubles where Grisu2 differs from the shortest representation), labels
    needing escapes, out-of-table region ids."""
    import torch
    labels = ["Load K", "GEMM0.c0", "we\"ird\\lab\tel", "Softmax.c1", "x" * 150, "é"]
    labels = labels[:5]
    ctx.set_plan(plan_of(8, 0, labels))
    ev = random_chrome_events(int(cpu * 7) + 1, 3000, len(labels))
    want = reference.export_chrome(ev, labels, cpu)
    d = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
    assert ctx.export_chrome_trace(None, cpu, on_device_ptr=d.data_ptr(),
                                   n_events=len(ev)) == want
    assert ctx.export_chrome_trace(ev, cpu) == want


def test_chrome_trace_gpu_formatter_attention_trace(ctx, reference):
    """A real device trace (the instrumented attention kernel, decoded on the
    GPU) exported on the GPU == the reference's export of the same events."""
    import torch
    from paper_2505_21661_b200 import p1
    BH, S = 2, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(BH, S, 128, generator=g, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    o = torch.empty_like(q)
    prof = torch.zeros(p1.attn_profile_bytes(BH, S), dtype=torch.uint8, device="cuda")
    p1.attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), BH, S,
                 instrument=True, profile_ptr=prof.data_ptr())
    ns = BH * S // 256 * p1.ATTN_WARPS
    t = T()
    ctx.set_plan(t.BufferPlan(p1.ATTN_SLOTS, t.BufferStrategy.Circular, p1.ATTN_LABELS))
    ev = torch.empty(ns * p1.ATTN_SLOTS * 32, dtype=torch.uint8, device="cuda")
    ne, _ = ctx.replay_device(prof.data_ptr(), prof.numel(), ns, 0, ev.data_ptr(),
                              ns * p1.ATTN_SLOTS)
    host = ev[: ne * 32].cpu().numpy().view(O.EVENT_DTYPE)
    want = reference.export_chrome(host, p1.ATTN_LABELS, 1965.0)
    assert ctx.export_chrome_trace(None, 1965.0, on_device_ptr=ev.data_ptr(),
                                   n_events=ne) == want


@pytest.mark.parametrize("shape", [0, 1])
def test_device_event_buffer_too_small(ctx, shape):
    """A device event buffer smaller than the trace: E_BUFFER with the full
    count, nothing written past the capacity (canary), and the events that
    fit are exactly the prefix of the full result (events sit at their final
    offsets) -- the thread-per-stream kernel's per-stream store limit, the
    warp kernel's per-store check."""
    import torch
    t = T()
    n = 4096
    plan = plan_of(S.CAP, 1 if shape == 0 else 0,
                   S.MIXED_LABELS if shape == 0 else S.NESTED_LABELS)
    ctx.set_plan(plan)
    body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
    ctx.synth_body(body.data_ptr(), shape, 0, n, n // 2)
    ne, _ = ctx.replay_device(body.data_ptr(), body.numel(), n, 33, 0, 0, 0x1)
    full = torch.empty(ne * 32, dtype=torch.uint8, device="cuda")
    assert ctx.replay_device(body.data_ptr(), body.numel(), n, 33, full.data_ptr(), ne)[0] == ne
    cap = ne // 3 + 5
    buf = torch.full(((cap + 64) * 32,), 0xAB, dtype=torch.uint8, device="cuda")
    with pytest.raises(t.BufferTooSmall) as ex:
        ctx.replay_device(body.data_ptr(), body.numel(), n, 33, buf.data_ptr(), cap)
    assert ex.value.needed == ne
    torch.cuda.synchronize()
    assert torch.all(buf[cap * 32:] == 0xAB)
    assert torch.equal(buf[: cap * 32], full[: cap * 32])


def test_chrome_trace_long_label_falls_back_to_host_writer(ctx, reference):
    """Labels longer than the GPU formatter's per-event budget take the host
    writer for device events: still the reference's bytes."""
    import torch
    labels = ["L" * 300, "short", 'q"uote']
    ctx.set_plan(plan_of(8, 0, labels))
    ev = random_chrome_events(5, 500, len(labels))
    want = reference.export_chrome(ev, labels, 1965.0)
    d = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
    assert ctx.export_chrome_trace(None, 1965.0, on_device_ptr=d.data_ptr(),
                                   n_events=len(ev)) == want


# ---------------------------------------------------------------------------
# record windows: TMA boxes (every stream of a warp's batch starts at slot 0)
# and cp.async chunks (wrapped circular streams, or WGPF_NO_TMA=1), with batch
# counts that are not multiples of 32 (the last box's rows past the body are
# zero-filled); consecutive and grouped (W streams per block) lane mappings
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("no_tma", [False, True])
def test_record_windows_tma_and_cp_async(oracle, monkeypatch, no_tma):
    t = T()
    if no_tma:
        monkeypatch.setenv("WGPF_NO_TMA", "1")
    else:
        monkeypatch.delenv("WGPF_NO_TMA", raising=False)
    c = t.Context(0)  # (the switch is read when the context is created)
    for seed in range(24):
        # (fuzz images have 4 streams per block: 160 and 256 streams take the
        # grouped lane mapping -- 40 blocks (a ragged second row of 32) and 64;
        # 100 streams = 25 blocks stay consecutive)
        n_streams = [32, 33, 95, 257, 160, 256, 100][seed % 7]
        data, cap, strategy, labels = fuzz.random_image(
            7000 + seed, n_streams=n_streams, cap=64 if seed % 2 else 32,
            mode="nested", big_gaps=(seed % 5 == 0))
        try:
            o, oerr = oracle.replay_kpft(data, cap, strategy, labels, 33), None
        except O.OracleError as e:
            o, oerr = None, (e.category, str(e))
        try:
            r = c.replay_image_bytes(data, plan_of(cap, strategy, labels), 33, flags=0x2)
            gerr = None
        except t.Error as e:
            r, gerr = None, (e.category(), str(e))
        assert oerr == gerr, (seed, oerr, gerr)
        if oerr:
            continue
        assert np.array_equal(r.events, o.events), seed
        assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups) == (o.dropped_heads, o.truncated_tails,
                                        o.flagged_preconditions, o.malformed_groups)
        want = oracle.region_stats(o.events, labels)
        got = c.stats()
        for s in want:
            g = got[s.label]
            assert (g.count, g.min, g.max, g.sum, g.mean, g.first_event,
                    g.hist) == (s.count, s.min, s.max, s.sum, s.mean,
                                s.first_event, s.hist), (seed, s.label)


@pytest.mark.parametrize("per_block", [1, 3, 5, 16, 33])
def test_grouped_lane_mapping_streams_per_block(ctx, oracle, per_block):
    """k_tps's grouped lane mapping for W = 1, 3, 5, 16, 33 streams per block
    (3-D TMA boxes of one warp index of 32 blocks; W not dividing 32; ragged
    last row of blocks; W that does not divide the stream count falls back to
    consecutive streams)."""
    t = T()
    for seed in range(6):
        n_blocks = [32, 40, 70, 33, 64, 31][seed]
        n = n_blocks * per_block + (1 if seed == 5 else 0)
        data, cap, strategy, labels = fuzz.random_image(
            9100 + 10 * per_block + seed, n_streams=n, cap=32, mode="nested",
            per_block=per_block)
        try:
            o, oerr = oracle.replay_kpft(data, cap, strategy, labels, 33), None
        except O.OracleError as e:
            o, oerr = None, (e.category, str(e))
        try:
            r = ctx.replay_image_bytes(data, plan_of(cap, strategy, labels), 33, flags=0x2)
            gerr = None
        except t.Error as e:
            r, gerr = None, (e.category(), str(e))
        assert oerr == gerr, (seed, oerr, gerr)
        if oerr:
            continue
        assert np.array_equal(r.events, o.events), seed
        assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups) == (o.dropped_heads, o.truncated_tails,
                                        o.flagged_preconditions, o.malformed_groups)
        want = oracle.region_stats(o.events, labels)
        got = ctx.stats()
        for s in want:
            g = got[s.label]
            assert (g.count, g.min, g.max, g.sum, g.mean, g.first_event,
                    g.hist) == (s.count, s.min, s.max, s.sum, s.mean,
                                s.first_event, s.hist), (seed, s.label)


@pytest.mark.parametrize("name", FIXTURES)
def test_reports_from_gpu_results_byte_identical(ctx, name):
    """The reference's replay / model reports rebuilt from the GPU path's
    statistics, critical path and warnings equal the golden files."""
    from paper_2505_21661_b200 import reports as R
    from test_reports import PARAMS, _golden
    from test_oracle import dev_barrier_edges
    data, slots, strategy, labels, cost, dev = load_fixture(name)
    plan = plan_of(slots, strategy, labels)
    r = ctx.replay_image_bytes(data, plan, cost)
    stats = T().region_stats(r.events, labels)  # (exact mean, the default context)
    cp = ctx.critical_path(r.events, dev_barrier_edges(dev))
    want = json.loads(_golden(name, "replay"))
    sim = R.SimTotals(want["total_cycles"], want["vanilla_cycles"], want["records_written"])
    assert R.dumps(R.replay_report(name, sim, stats, cp, r, cost)) == _golden(name, "replay")
    assert R.dumps(R.model_report(name, sim, stats, cp, cost, PARAMS.get(name))) == \
        _golden(name, "model")


# ---------------------------------------------------------------------------
# the deep thread-per-stream kernel (k_tpsd): nesting 9..64, circular wraps,
# TMA windows (one even start slot per batch) and cp.async windows (mixed or
# odd starts, windows across the wrap), clock wraps and >= 2^32 pairs (routed
# to the exact path), broken nesting, capacities at and past its 512 limit
# ---------------------------------------------------------------------------

DEEP_CASES = [
    dict(n_streams=96, cap=256, depth=64),                          # TMA, config-5-like
    dict(n_streams=96, cap=256, depth=20, same_start=False),        # cp.async
    dict(n_streams=64, cap=256, depth=33, odd=True),                # odd start
    dict(n_streams=70, cap=512, depth=64),                          # 9-bit positions
    dict(n_streams=64, cap=514, depth=12),                          # past the deep limit
    dict(n_streams=64, cap=128, depth=50, big_gaps=True),           # clock wraps
    dict(n_streams=64, cap=256, depth=30, violate=True),            # broken nesting
    dict(n_streams=33, cap=64, depth=10, same_start=False, big_gaps=True),
]


@pytest.mark.parametrize("case", range(len(DEEP_CASES)))
def test_deep_kernel_vs_oracle(ctx, oracle, case):
    t = T()
    for seed in range(3):
        data, cap, strategy, labels = fuzz.deep_image(31000 + 10 * case + seed,
                                                      **DEEP_CASES[case])
        try:
            o, oerr = oracle.replay_kpft(data, cap, strategy, labels, 33), None
        except O.OracleError as e:
            o, oerr = None, (e.category, str(e))
        try:
            r = ctx.replay_image_bytes(data, plan_of(cap, strategy, labels), 33, flags=0x2)
            gerr = None
        except t.Error as e:
            r, gerr = None, (e.category(), str(e))
        assert oerr == gerr, (case, seed, oerr, gerr)
        if oerr:
            continue
        assert len(r.events) == len(o.events) > 0
        assert np.array_equal(r.events, o.events), (case, seed)
        assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
                r.malformed_groups) == (o.dropped_heads, o.truncated_tails,
                                        o.flagged_preconditions, o.malformed_groups)
        want = oracle.region_stats(o.events, labels)
        got = ctx.stats()
        assert list(got) == [s.label for s in want]
        for s in want:
            g = got[s.label]
            assert (g.count, g.min, g.max, g.sum, g.mean, g.first_event, g.warp_group,
                    g.kind, g.hist) == (s.count, s.min, s.max, s.sum, s.mean,
                                        s.first_event, s.warp_group, s.kind,
                                        s.hist), (case, seed, s.label)


WIDE_CASES = [
    dict(n_streams=96, cap=256, depth=20),                          # TMA windows
    dict(n_streams=96, cap=256, depth=32, same_start=False),        # cp.async, full depth
    dict(n_streams=64, cap=256, depth=33),                          # past the wide depth
    dict(n_streams=64, cap=256, depth=12, n_labels=300),            # ids >= 256: general
    dict(n_streams=64, cap=128, depth=24, big_gaps=True),           # clock wraps
    dict(n_streams=64, cap=256, depth=16, violate=True),            # broken nesting
    dict(n_streams=40, cap=512, depth=8, n_labels=120),             # 9-bit positions
]


def _check_vs_oracle(ctx, oracle, data, cap, strategy, labels, tag):
    t = T()
    try:
        o, oerr = oracle.replay_kpft(data, cap, strategy, labels, 33), None
    except O.OracleError as e:
        o, oerr = None, (e.category, str(e))
    try:
        r = ctx.replay_image_bytes(data, plan_of(cap, strategy, labels), 33, flags=0x2)
        gerr = None
    except t.Error as e:
        r, gerr = None, (e.category(), str(e))
    assert oerr == gerr, (tag, oerr, gerr)
    if oerr:
        return None
    assert len(r.events) == len(o.events) > 0
    assert np.array_equal(r.events, o.events), tag
    assert (r.dropped_heads, r.truncated_tails, r.flagged_preconditions,
            r.malformed_groups) == (o.dropped_heads, o.truncated_tails,
                                    o.flagged_preconditions, o.malformed_groups)
    want = oracle.region_stats(o.events, labels)
    got = ctx.stats()
    assert list(got) == [s.label for s in want]
    for s in want:
        g = got[s.label]
        assert (g.count, g.min, g.max, g.sum, g.mean, g.first_event, g.warp_group,
                g.kind, g.hist) == (s.count, s.min, s.max, s.sum, s.mean,
                                    s.first_event, s.warp_group, s.kind,
                                    s.hist), (tag, s.label)
    return r


@pytest.mark.parametrize("case", range(len(WIDE_CASES)))
def test_wide_kernel_vs_oracle(ctx, oracle, case):
    """Plans with 120-300 labels: nesting up to 32 over region ids < 256 takes
    the wide thread-per-stream kernel (k_tpsd<kWide>), deeper streams the
    warp-per-stream kernel, ids >= 256 the general path -- all bit-exact with
    the oracle (events, warnings, every statistics field)."""
    for seed in range(3):
        data, cap, strategy, labels = fuzz.wide_image(41000 + 10 * case + seed,
                                                      **WIDE_CASES[case])
        _check_vs_oracle(ctx, oracle, data, cap, strategy, labels, (case, seed))


def test_wide_kernel_equals_warp_kernel(ctx, monkeypatch):
    """The wide thread-per-stream kernel and the warp-per-stream kernel
    (WGPF_NO_WIDE=1) give the same events and statistics on a larger body
    with 200 labels, 24-deep nesting."""
    import torch
    from paper_2505_21661_b200 import trace as Tm
    data, cap, strategy, labels = fuzz.wide_image(42000, n_streams=2048, depth=24)
    r = ctx.replay_image_bytes(data, plan_of(cap, strategy, labels), 33, flags=0x2)
    want_st = ctx.stats()
    monkeypatch.setenv("WGPF_NO_WIDE", "1")
    wctx = Tm.Context(0)
    r2 = wctx.replay_image_bytes(data, plan_of(cap, strategy, labels), 33, flags=0x2)
    assert np.array_equal(r.events, r2.events)
    assert wctx.stats() == want_st
    del torch


def test_exact_mean_recurrence_stress(ctx, oracle):
    """region_stats' bit-exact mean (pipeline.hpp:129) over long chains of
    random durations across the whole u32 range (the GPU division by the
    count runs a Markstein step with an exactness check, falling back to the
    IEEE division): equal to the CPU recurrence bit for bit."""
    t = T()
    rng = np.random.default_rng(11)
    n = 600_000
    ev = np.zeros(n, t.EVENT_DTYPE)
    ev["region"] = rng.integers(0, 3, n).astype(np.uint32)
    ev["start"] = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    scale = rng.choice([10, 1000, 1 << 20, (1 << 32) - 1], n)
    ev["end"] = ev["start"] + (rng.random(n) * scale).astype(np.uint64)
    labels = ["a", "b", "c"]
    got = t.region_stats(ev, labels)
    want = {s.label: s for s in oracle.region_stats(ev, labels)}
    for k, s in want.items():
        assert got[k].count == s.count and got[k].sum == s.sum
        assert got[k].mean == s.mean, (k, got[k].mean, s.mean)

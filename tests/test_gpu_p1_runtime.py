"""The P1 device runtime against the reference's vGPU on the same scope
programs.

A random scope program is lowered twice -- by the reference (lower.hpp:220,
from its text IR) and by wgpf_lower_scopes -- then simulated by the reference
(vgpu.hpp:424) and executed on the GPU by the scope-program interpreter
(csrc_p1/p1_selftest.cu k_program, one warp per warp group, the real
wgpf_dev::Recorder / Loop).  The device image (wgpf_collect) must carry the
vGPU image's stream headers and, slot for slot, its record tags (start bit,
region id, signature bits) -- only the clock payloads differ (hardware
cycles).  Covered: flush and circular strategies, power-of-two and odd
capacities (circular wrap, flush overflow), signature bits, iteration
signatures, and the reference's errors: pairing violations caught by the
debug-mode recorder (instrument.hpp:60-105 texts) and flush overflow
(vgpu.hpp:261-265 text).
"""
import random

import numpy as np
import pytest

from scopegen import dynamic_records, mutate, to_kir, valid_body

pytestmark = pytest.mark.gpu


def _hdr_and_tags(image: bytes):
    from paper_2505_21661_b200 import trace as T
    img = T.deserialize_image(image)
    out = []
    for s in img.streams:
        tags = [int(t) for t in s.slots["tag"]]
        out.append(((s.block_index, s.warp_group, s.record_count, s.slot_capacity), tags))
    return out


def _run_device(bodies, strategy, cap, sig_mode, validate, ctas=1, busy=2):
    import torch
    from paper_2505_21661_b200 import p1
    from paper_2505_21661_b200 import trace as T
    plan = p1.lower_scopes(bodies, strategy, 1 << 20, slots_total=cap * len(bodies),
                           iteration_signature=sig_mode == p1.SIG_ITER,
                           signature_bits=sig_mode == p1.SIG_HW)
    ops, offs = p1.program_encoding(bodies, plan, busy=busy)
    d_ops = torch.from_numpy(ops.astype(np.int32)).cuda()
    d_offs = torch.from_numpy(offs.astype(np.int32)).cuda()
    nb = len(bodies)
    prof = torch.zeros(ctas * nb * p1.stream_stride(cap), dtype=torch.uint8,
                       device="cuda")
    verr = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    p1.run_program(prof.data_ptr(), ctas, nb, cap, strategy == 1, validate, sig_mode,
                   d_ops.data_ptr(), d_offs.data_ptr(), verr.data_ptr() if validate else 0)
    torch.cuda.synchronize()
    ctx = T.Context(0)
    ctx.set_plan(T.BufferPlan(cap, T.BufferStrategy(strategy), plan.labels))
    return ctx.collect(prof.data_ptr(), ctas * nb, verr.data_ptr() if validate else 0), plan


def _ref_run(reference, bodies, strategy, cap, sig_mode):
    from paper_2505_21661_b200 import p1
    return reference.lower_kir(to_kir(bodies, 1 << 20), strategy,
                               slots_total=cap * len(bodies),
                               iteration_signature=sig_mode == p1.SIG_ITER,
                               signature_bits=sig_mode == p1.SIG_HW, simulate=True)


def _fits(bodies, cap, strategy):
    return strategy == 0 or all(dynamic_records(b) <= cap for b in bodies)


@pytest.mark.parametrize("seed", range(8))
def test_device_image_matches_vgpu_image(reference, seed):
    from paper_2505_21661_b200 import p1
    rng = random.Random(77 + seed)
    done = 0
    while done < 12:
        nwg = rng.randint(1, 6)
        bodies = [valid_body(rng, max_ops=10) for _ in range(nwg)]
        strategy = rng.randint(0, 1)
        if strategy == 1:
            cap = max(dynamic_records(b) for b in bodies) + rng.choice([0, 1, 3])
        else:
            cap = rng.choice([1, 2, 3, 4, 5, 7, 8, 13, 16, 64])
        sig = rng.choice([p1.SIG_NONE, p1.SIG_HW, p1.SIG_ITER])
        dev, plan = _run_device(bodies, strategy, cap, sig, validate=rng.random() < 0.5)
        ref = _ref_run(reference, bodies, strategy, cap, sig)
        assert plan.labels == ref["labels"]
        a, b = _hdr_and_tags(dev), _hdr_and_tags(ref["image"])
        assert len(a) == len(b) == nwg
        for k, ((ha, ta), (hb, tb)) in enumerate(zip(a, b)):
            assert ha == hb, (k, ha, hb)
            n = min(hb[2], hb[3])
            assert ta[:n] == tb[:n], (k, to_kir(bodies, 0), sig, cap)
            # the store log (vgpu.hpp:269-271): the tags in write order
            log = ref["store_log"][k]
            assert len(log) == hb[2]
            if strategy == 1:
                assert ta[:n] == log
            else:
                keep = log[-n:] if n else []
                start = hb[2] % hb[3] if hb[2] > hb[3] else 0
                ring = [ta[(start + i) % hb[3]] for i in range(n)]
                assert ring == keep
        done += 1


@pytest.mark.parametrize("seed", range(6))
def test_debug_mode_pairing_errors_match_reference(reference, seed):
    """Device-side validation (Recorder<..., kValidate>) reports the first
    violation of the lowest warp group with the reference's text."""
    from oracle.oracle import OracleError
    from paper_2505_21661_b200 import p1
    from paper_2505_21661_b200 import trace as T
    rng = random.Random(500 + seed)
    hits = 0
    while hits < 10:
        nwg = rng.randint(1, 4)
        bodies = [valid_body(rng, max_ops=10) for _ in range(nwg)]
        k = rng.randrange(nwg)
        bodies[k] = mutate(rng, bodies[k])
        try:
            reference.lower_kir(to_kir(bodies, 1 << 20), 0, slots_total=64 * nwg)
            continue  # the mutation kept the program valid
        except OracleError as e:
            want = (e.category, str(e))
        if want[0] != "instrument-error":
            continue
        # the device runs what the host would reject: lower ids by hand
        labels = []
        for b in bodies:
            for o in b:
                if o[0] in ("start", "end") and o[1] not in labels:
                    labels.append(o[1])
        ids = [[labels.index(o[1]) if o[0] in ("start", "end") else None for o in b]
               for b in bodies]
        plan = p1.ScopePlan(64, labels, ids, 0)
        import torch
        ops, offs = p1.program_encoding(bodies, plan, busy=1)
        d_ops = torch.from_numpy(ops.astype(np.int32)).cuda()
        d_offs = torch.from_numpy(offs.astype(np.int32)).cuda()
        prof = torch.zeros(nwg * p1.stream_stride(64), dtype=torch.uint8, device="cuda")
        verr = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        p1.run_program(prof.data_ptr(), 1, nwg, 64, False, True, p1.SIG_NONE,
                       d_ops.data_ptr(), d_offs.data_ptr(), verr.data_ptr())
        torch.cuda.synchronize()
        ctx = T.Context(0)
        ctx.set_plan(T.BufferPlan(64, T.BufferStrategy.Circular, labels))
        with pytest.raises(T.Error) as ei:
            ctx.collect(prof.data_ptr(), nwg, verr.data_ptr())
        got = (ei.value.category(), str(ei.value))
        assert got[0] == want[0]
        assert want[1].endswith(got[1]), (to_kir(bodies, 0), got, want)
        hits += 1


@pytest.mark.parametrize("cap", [3, 4, 8])
def test_flush_overflow_is_a_capacity_error(reference, cap):
    """A flush buffer that overflows keeps its first `cap` records and
    wgpf_collect raises the vGPU's capacity-error (vgpu.hpp:261-265)."""
    from oracle.oracle import OracleError
    from paper_2505_21661_b200 import p1
    from paper_2505_21661_b200 import trace as T
    small = [("start", "A"), ("end", "A")]
    big = [("loop", cap), ("start", "A"), ("end", "A"), ("endloop",)]
    bodies = [small, big, small]
    with pytest.raises(OracleError) as er:
        reference.lower_kir(to_kir(bodies, 1 << 20), 1, slots_total=cap * 3,
                            simulate=True)
    with pytest.raises(T.Error) as ed:
        _run_device(bodies, 1, cap, p1.SIG_NONE, validate=False)
    assert ed.value.category() == er.value.category == "capacity-error"
    assert str(er.value).endswith(str(ed.value)), (str(er.value), str(ed.value))


@pytest.mark.parametrize("cap,warps", [(3, 1), (3, 2), (5, 3), (1, 2), (7, 4)])
def test_odd_capacities_multi_cta(oracle, cap, warps):
    """Odd capacities give an 8-byte-aligned stream stride: the header and
    the flush use 8-byte stores; several CTAs' segments must land intact."""
    from paper_2505_21661_b200 import p1
    body = [("loop", 5), ("start", "A"), ("start", "B"), ("end", "B"), ("end", "A"),
            ("endloop",)]
    bodies = [body] * warps
    img, plan = _run_device(bodies, 0, cap, p1.SIG_NONE, validate=True, ctas=5)
    got = _hdr_and_tags(img)
    assert len(got) == 5 * warps
    writes = 20
    log = [0x80000000 | 0 << 12, 0x80000000 | 1 << 12, 1 << 12, 0 << 12] * 5
    start = writes % cap
    for s, (h, tags) in enumerate(got):
        assert h == (s // warps, s % warps, writes, cap)
        ring = [tags[(start + i) % cap] for i in range(cap)]
        assert ring == log[-cap:]


def test_loop_entry_cost_is_measured():
    """vgpu.hpp:366-369 charges loop_entry_cost (5 cycles) per dynamic entry
    of an instrumented loop.  The device recorder keeps its index in a
    register across loops -- no per-loop prologue -- so the measured extra
    cost of entering a loop that records, E(records) - E(plain), stays small
    next to the record pair itself."""
    from paper_2505_21661_b200 import p1
    r = p1.loop_entry_cost()
    print(r)
    assert r["record_pair_cycles_in_loop"] > 0
    assert abs(r["loop_entry_cost_cycles"]) < r["record_pair_cycles_in_loop"], r


def test_bulk_flush_equals_vector_flush():
    """wgpf_dev::flush_bulk (one cp.async.bulk shared -> global) leaves the
    same KPFT body segment in HBM as the vector-store flush, for the GEMM's
    3,168-B buffer and a 32-KB one; both costs are measured."""
    import bench_p1
    r = bench_p1.measure_flush()
    print(r)
    for nb, row in r.items():
        assert row["identical"], nb
        assert row["bulk"] > 0 and row["vector"] > 0

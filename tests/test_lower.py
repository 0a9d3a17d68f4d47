"""lower() of scope programs (C-ABI wgpf_lower_scopes, p1.lower_scopes) vs the
reference's own lower() (lower.hpp:220-301, compiled in oracle/_ref) on the
same programs rendered as its text IR: plans (slots per warp group, region
table in first-appearance order) and errors (kind and message of
validate ir.hpp:347-390, validate_record_pairing instrument.hpp:60-105 and the
configuration / capacity checks lower.hpp:223-279).  Host code: CPU tests.
"""
import random

import pytest

from scopegen import mutate, to_kir, valid_body

from paper_2505_21661_b200 import p1
from paper_2505_21661_b200.trace import Error


def _ours(bodies, strategy, smem, **kw):
    try:
        pl = p1.lower_scopes(bodies, strategy, smem, **kw)
        return ("ok", pl.slots_per_stream, pl.labels)
    except Error as e:
        return ("err", e.category(), str(e))


def _ref(reference, bodies, strategy, smem, **kw):
    from oracle.oracle import OracleError
    try:
        r = reference.lower_kir(to_kir(bodies, smem), strategy, **kw)
        return ("ok", r["slots"], r["labels"])
    except OracleError as e:
        return ("err", e.category, str(e))


def _norm(x):
    if x[0] == "err":
        return (x[0], x[1], x[2].split(": ", 1)[-1] if x[2].startswith(x[1]) else x[2])
    return x


def _cmp(reference, bodies, strategy, smem, **kw):
    a = _ours(bodies, strategy, smem, **kw)
    kw_ref = dict(kw)
    b = _ref(reference, bodies, strategy, smem, **kw_ref)
    assert _norm(a) == _norm(b), (to_kir(bodies, smem), kw, a, b)
    return a


def test_error_kind_messages_known_cases(reference):
    S = [("start", "A"), ("end", "B")]
    assert _cmp(reference, [S], 1, 4096)[0] == "err"
    cross = [("start", "A"), ("loop", 2), ("end", "A"), ("endloop",)]
    r = _cmp(reference, [[("start", "X"), ("end", "X")], cross], 1, 4096)
    assert r[0] == "err" and "wg1" in r[2] and "crosses a loop boundary" in r[2]
    open_ = [("loop", 3), ("start", "A"), ("endloop",)]
    r = _cmp(reference, [open_], 0, 4096)
    assert "record start \"A\" crosses a loop boundary" in r[2]
    r = _cmp(reference, [[("start", "A")]], 0, 4096)
    assert "is never closed" in r[2]
    ok = [("loop", 4), ("start", "A"), ("end", "A"), ("endloop",)]
    # explicit slots not divisible by the warp-group count
    r = _cmp(reference, [ok, ok], 1, 4096, slots_total=7)
    assert r[1] == "lower-error" and "not divisible" in r[2]
    # iteration signature needs the signature bits free
    r = _cmp(reference, [ok], 1, 4096, signature_bits=True, iteration_signature=True)
    assert r[1] == "lower-error"
    # shared-memory budget
    r = _cmp(reference, [ok], 1, 32, slots_total=8)
    assert r[1] == "capacity-error" and "needs 64 bytes" in r[2]
    # circular sizing with too little shared memory
    r = _cmp(reference, [ok, ok, ok], 0, 16)
    assert r[1] == "capacity-error"
    # a global buffer skips the smem check
    assert _cmp(reference, [ok], 1, 32, slots_total=8, global_buffer=True)[:2] == ("ok", 8)
    # zero-trip loop (validate)
    r = _cmp(reference, [[("loop", 0), ("start", "A"), ("end", "A"), ("endloop",)]], 1, 64)
    assert r[1] == "validate-error"


@pytest.mark.parametrize("seed", range(6))
def test_random_programs_match_reference_lowering(reference, seed):
    rng = random.Random(1000 + seed)
    for _ in range(60):
        nwg = rng.randint(1, 4)
        bodies = [valid_body(rng) for _ in range(nwg)]
        if rng.random() < 0.5:
            k = rng.randrange(nwg)
            bodies[k] = mutate(rng, bodies[k])
        strategy = rng.randint(0, 1)
        smem = rng.choice([64, 1024, 4096, 1 << 16])
        kw = {}
        if rng.random() < 0.3:
            kw["slots_total"] = rng.choice([nwg * 4, nwg * 32, nwg * 4 + 1])
        if rng.random() < 0.3:
            kw["iteration_signature"] = True
        if rng.random() < 0.2:
            kw["signature_bits"] = True
        _cmp(reference, bodies, strategy, smem, **kw)


def test_region_ids_first_appearance_order():
    b0 = [("start", "B"), ("start", "A"), ("end", "A"), ("end", "B")]
    b1 = [("start", "C"), ("end", "C"), ("start", "B"), ("end", "B")]
    pl = p1.lower_scopes([b0, b1], 1, 1 << 16)
    assert pl.labels == ["B", "A", "C"]
    assert pl.region_ids == [[0, 1, 1, 0], [2, 2, 0, 0]]
    assert pl.slots_per_stream == 4
    assert pl.smem_bytes_per_cta == 2 * (16 + 8 * 4)

"""Analytic models (paper_2505_21661_b200/models.py) against the reference's
own known answers (tests/test_perfmodel.cpp) and the live reference
(oracle/_ref, perfmodel.hpp) on random inputs -- CPU only."""
import itertools
import os

import numpy as np
import pytest

from conftest import FIXTURES, load_fixture
from paper_2505_21661_b200 import models as M
from paper_2505_21661_b200.trace import Error, ErrorKind


# ---- known answers (test_perfmodel.cpp) --------------------------------------

def test_swp_known_answers():
    r = M.swp_latency(M.SwpInput(1, 2, 10, [M.SwpStage("s0", 200, 100),
                                           M.SwpStage("s1", 80, 50)]))
    assert (r.delta, r.latency) == (0, 1500)
    r = M.swp_latency(M.SwpInput(1, 2, 10, [M.SwpStage("s0", 400, 100),
                                           M.SwpStage("s1", 80, 50)]))
    assert (r.delta, r.latency) == (-200, 2500)
    r = M.swp_latency(M.SwpInput(1, 1, 7, [M.SwpStage("s0", 0, 130)]))
    assert (r.delta, r.latency) == (0, 910)
    r = M.swp_latency(M.SwpInput(1, 3, 11, [M.SwpStage("a", 240, 60),
                                           M.SwpStage("b", 10, 40)]))
    assert (r.delta, r.latency) == (0, 1100) and (300 * 11 + 2) // 3 == 1100
    with pytest.raises(Error, match="inputs must be positive") as e:
        M.swp_latency(M.SwpInput(1, 1, 1, []))
    assert e.value.kind == ErrorKind.Validate


def test_swp_monotone_in_stage_times():
    rng = np.random.default_rng(0x5A)
    for _ in range(300):
        n = int(rng.integers(1, 5))
        inp = M.SwpInput(1, int(rng.integers(1, 5)), int(rng.integers(1, 65)),
                         [M.SwpStage(f"s{s}", int(rng.integers(0, 1000)),
                                     int(rng.integers(0, 1000))) for s in range(n)])
        base = M.swp_latency(inp).latency
        k = int(rng.integers(0, n))
        bump = int(rng.integers(1, 101))
        if rng.integers(0, 2):
            inp.stages[k].t_comp += bump
        else:
            inp.stages[k].t_load += bump
        assert M.swp_latency(inp).latency >= base


def test_ws_known_answers():
    N = M.WsNode
    r = M.ws_latency(M.WsInput([N("a", 300), N("b", 200), N("c", 100)], [(0, 1), (1, 2)]))
    assert (r.latency, r.critical_path) == (600, ["a", "b", "c"])
    r = M.ws_latency(M.WsInput([N("src", 100), N("left", 400), N("right", 350),
                                N("sink", 50)], [(0, 1), (0, 2), (1, 3), (2, 3)]))
    assert (r.latency, r.critical_path) == (550, ["src", "left", "sink"])
    r = M.ws_latency(M.WsInput())
    assert (r.latency, r.critical_path) == (0, [])
    with pytest.raises(Error, match="cycle"):
        M.ws_latency(M.WsInput([N("a", 1), N("b", 1)], [(0, 1), (1, 0)]))
    r = M.ws_latency(M.WsInput([N("start", 10), N("zeta", 20), N("alpha", 20)],
                               [(0, 1), (0, 2)]))
    assert (r.latency, r.critical_path) == (30, ["start", "alpha"])
    with pytest.raises(Error, match="edge index out of range"):
        M.ws_latency(M.WsInput([N("a", 1)], [(0, 1)]))


def _brute_force_ws(inp):
    succ = [[] for _ in inp.nodes]
    for a, b in inp.edges:
        succ[a].append(b)
    best = 0

    def dfs(v, acc):
        nonlocal best
        acc += inp.nodes[v].duration
        best = max(best, acc)
        for s in succ[v]:
            dfs(s, acc)

    for v in range(len(inp.nodes)):
        dfs(v, 0)
    return best


def test_ws_matches_brute_force():
    rng = np.random.default_rng(0x37)
    for _ in range(300):
        n = int(rng.integers(1, 13))
        nodes = [M.WsNode(f"n{v}", int(rng.integers(0, 1000))) for v in range(n)]
        edges = [(a, b) for a in range(n) for b in range(a + 1, n)
                 if rng.integers(0, 3) == 0]
        inp = M.WsInput(nodes, edges)
        assert M.ws_latency(inp).latency == _brute_force_ws(inp)


def test_roofline_and_overhead_known_answers():
    assert M.roofline(M.RooflineInput(1000, 500, 0, 0, 1)).compute_cycles == 2
    assert M.roofline(M.RooflineInput(0, 1, 100, 4096, 64)).memory_cycles == 164
    assert M.roofline(M.RooflineInput(0, 7, 0, 0, 3)).compute_cycles == 0
    assert M.overhead_model(M.OverheadInput(1000, 10, 33)) == 1330
    assert M.overhead_model(M.OverheadInput(777, 0, 33)) == 777
    assert M.overhead_model(M.OverheadInput(199381, 800, 32)) == 224981
    with pytest.raises(Error, match="rates must be positive"):
        M.roofline(M.RooflineInput(1, 0, 0, 0, 1))


def test_stage_table_known_answers():
    st = M.load_stage_table("# stage t_load t_comp\nqk 200 100\npv 80 50\n\n")
    assert [(s.name, s.t_load, s.t_comp) for s in st] == [("qk", 200, 100), ("pv", 80, 50)]
    with pytest.raises(Error, match="stage table line 1") as e:
        M.load_stage_table("qk 200\n")
    assert e.value.kind == ErrorKind.Parse


# ---- against the live reference ------------------------------------------------

def _ref_raw(reference, text):
    import ctypes as C
    L = reference.lib
    L.ref_models.restype = C.c_void_p
    L.ref_models.argtypes = [C.c_char_p]
    p = L.ref_models(text.encode())
    out = C.string_at(p).decode()
    L.ref_free_text(C.c_void_p(p))
    return out


def _enc(label):
    return "".join(c if " " < c < "\x7f" and c != "%" else
                   "".join(f"%{b:02X}" for b in c.encode()) for c in label)


def _ours(fn):
    try:
        return "ok " + " ".join(str(x) for x in fn())
    except Error as e:
        return f"err {int(e.kind)} {e}"


_QUERIES = []  # every protocol query the reference comparisons below sent


def _ref(reference, text):
    _QUERIES.append(text)
    return _ref_raw(reference, text)


def test_swp_vs_reference(reference):
    rng = np.random.default_rng(11)
    big = [0, 1, 2, 7, 1000, (1 << 32) - 1, (1 << 40), (1 << 63) - 5, (1 << 64) - 1]
    for _ in range(400):
        n = int(rng.integers(0, 5))
        pick = (lambda: big[int(rng.integers(len(big)))]) if rng.integers(0, 4) == 0 else \
               (lambda: int(rng.integers(0, 2000)))
        nwg, npipe = int(rng.integers(0, 4)), int(rng.integers(0, 5))
        nloop = pick()
        stages = [M.SwpStage(f"s{i}", pick(), pick()) for i in range(n)]
        text = f"swp {nwg} {npipe} {nloop}\n" + "".join(
            f"stage {s.name} {s.t_load} {s.t_comp}\n" for s in stages)
        inp = M.SwpInput(nwg, npipe, nloop, stages)
        got = _ours(lambda: (lambda r: (r.delta, r.latency))(M.swp_latency(inp)))
        assert got == _ref(reference, text), text


def test_ws_vs_reference(reference):
    rng = np.random.default_rng(12)
    for it in range(500):
        n = int(rng.integers(0, 9))
        # few distinct durations and labels: ties everywhere
        nodes = [M.WsNode(str(rng.choice(["a", "b", "c", "dd", "a0", "Load A", "a b"])) + str(int(rng.integers(0, 3))),
                          int(rng.integers(0, 4)) * 10) for _ in range(n)]
        edges = []
        for _ in range(int(rng.integers(0, 2 * n + 1))):
            a, b = int(rng.integers(0, n + 1)), int(rng.integers(0, n + 1))
            if it % 7 and (a >= n or b >= n or a >= b):
                continue  # mostly DAGs; every 7th graph may be bad
            edges.append((a, b))
        text = "wsempty\n" + "".join(f"node {_enc(x.label)} {x.duration}\n" for x in nodes) + \
            "".join(f"edge {a} {b}\n" for a, b in edges)
        inp = M.WsInput(nodes, edges)
        got = _ours(lambda: (lambda r: [r.latency] + [_enc(l) for l in r.critical_path])(
            M.ws_latency(inp)))
        assert got == _ref(reference, text), text


def test_roofline_overhead_vs_reference(reference):
    rng = np.random.default_rng(13)
    vals = [0, 1, 3, 64, 1000, (1 << 32) + 1, (1 << 63), (1 << 64) - 1]
    for f, t, r, b, w in itertools.islice(
            ((vals[int(rng.integers(len(vals)))] for _ in range(5)) for _ in itertools.count()), 300):
        got = _ours(lambda: (lambda x: (x.compute_cycles, x.memory_cycles))(
            M.roofline(M.RooflineInput(f, t, r, b, w))))
        assert got == _ref(reference, f"roofline {f} {t} {r} {b} {w}")
        got = "ok " + str(M.overhead_model(M.OverheadInput(f, t, r)))
        assert got == _ref(reference, f"overhead {f} {t} {r}")


def test_stage_table_vs_reference(reference):
    lines = ["qk 200 100", "  pv\t80 50  # tail", "# only a comment", "", "   ",
             "x 1", "y a b", "z -5 7", "w +3 4", "v 12abc 4", "u 3 4 extra",
             "t 18446744073709551615 0", "s 18446744073709551616 0", "r 0x10 2",
             "q 1\r", "p 2 3\r", "#", "o 1 2 # 3 4", "n -0 -0"]
    rng = np.random.default_rng(14)
    for _ in range(300):
        k = int(rng.integers(0, 6))
        text = "\n".join(str(rng.choice(lines)) for _ in range(k))
        if rng.integers(0, 2):
            text += "\n"
        got = _ours(lambda: [x for s in M.load_stage_table(text)
                             for x in (s.name, s.t_load, s.t_comp)])
        assert got.rstrip() == _ref(reference, "table\n" + text).rstrip(), repr(text)


@pytest.mark.parametrize("name", FIXTURES)
def test_stage_graph_from_critical_path_vs_reference(oracle, reference, name):
    """ws_latency input built from a critical-path result equals the
    reference's CriticalPathAnalysis.graph (the CPU oracle's critical path
    is the GPU's, tests/test_gpu_overlap.py)."""
    data, slots, strategy, labels, cost, dev = load_fixture(name)
    ref = reference.critical_path_kpft(data, dev, cost)
    r = oracle.replay_kpft(data, slots, strategy, labels, cost)
    cp = oracle.critical_path(r.events, labels, ref["barrier_edges"])
    g = M.ws_input_from_critical_path(cp)
    assert [x.label for x in g.nodes] == ref["nodes"]
    assert [x.duration for x in g.nodes] == ref["durations"]
    assert [tuple(e) for e in g.edges] == [tuple(e) for e in ref["edges"]]
    text = "wsempty\n" + "".join(f"node {_enc(x.label)} {x.duration}\n" for x in g.nodes) + \
        "".join(f"edge {a} {b}\n" for a, b in g.edges)
    got = _ours(lambda: (lambda w: [w.latency] + [_enc(l) for l in w.critical_path])(
        M.ws_latency(g)))
    assert got == _ref(reference, text)


def test_cxx_dropin_models_vs_reference(reference, tmp_path):
    """The C++ drop-in's models (include/wgprof_b200.hpp) answer every query
    of the comparisons above exactly like the reference (host code: built
    and run here, no GPU)."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    exe = str(tmp_path / "models_cli")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(here, "..", "include"),
                    "-o", exe, os.path.join(here, "cxx", "models_cli.cpp")], check=True)
    if len(_QUERIES) < 1000:  # (run on its own: replay the comparisons)
        test_swp_vs_reference(reference)
        test_ws_vs_reference(reference)
        test_roofline_overhead_vs_reference(reference)
        test_stage_table_vs_reference(reference)
    queries = list(_QUERIES)
    res = subprocess.run([exe], input="\0".join(queries) + "\0", capture_output=True,
                         text=True, check=True)
    got = res.stdout.split("\n")[:len(queries)]
    for q, g in zip(queries, got):
        assert g.rstrip() == _ref_raw(reference, q).rstrip(), q


# ---- buffer planning and stream signatures (P1 host helpers) -------------------

def test_plan_slots_known_answers():
    from paper_2505_21661_b200 import p1
    from paper_2505_21661_b200.trace import BufferStrategy
    assert p1.plan_slots(4, [512], 2, BufferStrategy.Flush, 1 << 20).slots_per_warp_group * 2 == 4096
    with pytest.raises(Error) as e:
        p1.plan_slots(4, [512], 2, BufferStrategy.Flush, 16384)
    assert e.value.kind == ErrorKind.Capacity
    assert p1.plan_slots(1, [], 1, BufferStrategy.Circular, 1024).slots_per_warp_group == 128
    assert p1.plan_slots(1, [], 1, BufferStrategy.Circular, 1000).slots_per_warp_group == 64


def test_plan_slots_and_signature_vs_reference(reference):
    from paper_2505_21661_b200 import p1
    rng = np.random.default_rng(15)
    for _ in range(400):
        regions, nwg = int(rng.integers(0, 20)), int(rng.integers(0, 9))
        strat = int(rng.integers(0, 2))
        cap = int(rng.choice([0, 7, 8, 1000, 1024, 4096, 1 << 16, 1 << 20]))
        trips = [int(rng.integers(0, 600)) for _ in range(int(rng.integers(0, 3)))]
        text = f"plan {regions} {nwg} {strat} {cap} {len(trips)} " + " ".join(map(str, trips))
        got = _ours(lambda: [p1.plan_slots(regions, trips, nwg, strat, cap).slots_per_warp_group])
        assert got == _ref(reference, text), text
    for wg in list(range(0, 2048, 7)) + [4095, 4096, 65535, (1 << 32) - 1]:
        assert "ok " + str(p1.signature_for(wg)) == _ref(reference, f"sig {wg}")

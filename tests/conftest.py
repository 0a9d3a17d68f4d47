import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
FIXTURES = ["simple", "gemm_swp", "fa3_vanilla", "fa3_improved"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    return O.Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return O.Reference()


@pytest.fixture(scope="session")
def ctx():
    from paper_2505_21661_b200 import trace as T
    return T.Context(0)


def parse_dev_header(dev: str):
    first = dev.splitlines()[0]
    kv = dict(tok.split("=", 1) for tok in first.split() if "=" in tok)
    labels = []
    for line in dev.splitlines()[1:]:
        t = line.strip()
        if t.startswith("region "):
            labels.append(json.loads(t[t.index('"'):]))
    strategy = 0 if kv["strategy"] == "circular" else 1
    return int(kv["slots_per_wg"]), strategy, labels


def load_fixture(name):
    """(kpft bytes, slots, strategy, labels, record_cost, dev text)."""
    base = os.path.join(GOLDEN, "fixtures", name)
    data = open(base + ".kpft", "rb").read()
    dev = open(base + ".dev").read()
    slots, strategy, labels = parse_dev_header(dev)
    cost = int(open(base + ".cost").read().split()[0])
    return data, slots, strategy, labels, cost, dev


def load_random_set(name):
    z = np.load(os.path.join(GOLDEN, f"random_{name}.npz"), allow_pickle=True)
    blob = z["blob"].tobytes()
    offs = z["offsets"]
    out = []
    for i in range(len(offs) - 1):
        img = blob[int(offs[i]):int(offs[i + 1])]
        dev = str(z["devs"][i])
        slots, strategy, labels = parse_dev_header(dev)
        out.append((img, slots, strategy, labels, z["results"][i]))
    return out


def load_synth(name):
    return dict(np.load(os.path.join(GOLDEN, f"synth_{name}.npz"), allow_pickle=True))


def canon_golden(res, space):
    """Golden reference replay result -> canonical event array."""
    from oracle import oracle as O
    return O.canon_from_ref(res["events"], list(res["labels"]), space)

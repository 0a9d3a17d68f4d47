import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2505_21661_b200 import trace as T
rng = np.random.default_rng(1)
n = 20_000_000
ev = np.zeros(n, T.EVENT_DTYPE)
ev["region"] = rng.integers(0, 8, n).astype(np.uint32)
ev["end"] = rng.integers(0, 5000, n).astype(np.uint64)
st = T.region_stats(ev, [f"L{i}" for i in range(8)])
print(len(st))

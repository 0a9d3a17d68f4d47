"""Raw pinned host<->device copy bandwidth (the ceiling of the e2e path)."""
import json
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        fn()
    e1.record(); torch.cuda.synchronize()
    res[name] = 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(s1):
    for _ in range(4):
        d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(4):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
res["duplex_total"] = 8 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
print(json.dumps({k: round(v, 1) for k, v in res.items()}))

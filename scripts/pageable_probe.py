"""Host-memory options for pageable caller buffers on this box: cost of
cudaHostRegister / Unregister, pinned H2D / D2H, pageable H2D / D2H, and a
multi-threaded host memcpy (the bounce-buffer alternative)."""
import ctypes as C
import json
import os
import threading
import time

import numpy as np
import torch

cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if cudart is None:
    cudart = C.CDLL("libcudart.so")
cudart.cudaHostRegister.argtypes = [C.c_void_p, C.c_size_t, C.c_uint]
cudart.cudaHostUnregister.argtypes = [C.c_void_p]
GB = 1 << 30
out = {"nproc": os.cpu_count()}
for size_gb in (1, 8):
    a = np.ones(size_gb * GB, np.uint8)  # pageable, touched
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(C.c_void_p(a.ctypes.data), a.nbytes, 0)
    t_reg = time.perf_counter() - t
    t = time.perf_counter()
    cudart.cudaHostUnregister(C.c_void_p(a.ctypes.data))
    t_unreg = time.perf_counter() - t
    d = torch.empty(a.nbytes, dtype=torch.uint8, device="cuda")
    ta = torch.from_numpy(a)
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(ta)
    torch.cuda.synchronize()
    t_h2d_pageable = time.perf_counter() - t
    t = time.perf_counter()
    ta.copy_(d)
    torch.cuda.synchronize()
    t_d2h_pageable = time.perf_counter() - t
    out[f"{size_gb}GB"] = {"register_rc": rc, "register_gbs": size_gb / t_reg,
                          "unregister_gbs": size_gb / t_unreg,
                          "h2d_pageable_gbs": size_gb / t_h2d_pageable,
                          "d2h_pageable_gbs": size_gb / t_d2h_pageable}
    del d
    torch.cuda.empty_cache()
# multi-threaded host memcpy
src = np.ones(8 * GB, np.uint8)
dst = np.empty_like(src)
for nt in (1, 4, 8, 16):
    parts = np.array_split(np.arange(8 * GB // (1 << 20)), nt)

    def work(p):
        dst[p[0] << 20:(p[-1] + 1) << 20] = src[p[0] << 20:(p[-1] + 1) << 20]
    t = time.perf_counter()
    th = [threading.Thread(target=work, args=(p,)) for p in parts]
    for x in th:
        x.start()
    for x in th:
        x.join()
    out[f"memcpy_{nt}t_gbs"] = 8 / (time.perf_counter() - t)
print(json.dumps(out))

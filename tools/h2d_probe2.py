"""Is slow pinned H2D a property of the buffer or a warm-up effect?"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def h2d(h, d, reps=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    return reps * h.numel() * 8 / (time.perf_counter() - t0) / 1e9


def main():
    from paper_2408_09662_b200 import _native
    L = _native.lib()
    n = (8 << 20) // 8
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    bufs = []
    for k in range(4):
        h = torch.empty(n, dtype=torch.float64).pin_memory()
        h.fill_(1.0)
        bufs.append(("torch_pin", h))
    for k in range(3):
        ptr = ctypes.c_void_p()
        L.vsb_host_alloc(ctypes.byref(ptr), n * 8)
        arr = np.frombuffer((ctypes.c_char * (n * 8)).from_address(ptr.value), dtype=np.float64)
        arr[:] = 1.0
        bufs.append(("vsb_host_alloc", torch.from_numpy(arr)))
    res = []
    for rnd in range(2):
        for name, h in bufs:
            res.append({"round": rnd, "buf": name, "h2d_gbs": round(h2d(h, d), 1)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()

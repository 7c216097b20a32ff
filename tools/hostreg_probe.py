"""cudaHostRegister cost on fresh / touched numpy arrays (development helper)."""
import time

import numpy as np
import torch

cr = torch.cuda.cudart()
dev = torch.device("cuda", 0)
d = torch.empty(101 * 2 ** 20 // 16, dtype=torch.complex128, device=dev)


def reg(arr):
    rc = cr.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    assert int(rc) == 0, rc


def unreg(arr):
    cr.cudaHostUnregister(arr.ctypes.data)


for label, make in (("fresh 101 MB", lambda: np.empty(d.numel(), np.complex128)),
                    ("touched 101 MB", lambda: np.ones(d.numel(), np.complex128))):
    for _ in range(3):
        arr = make()
        t0 = time.perf_counter()
        reg(arr)
        t1 = time.perf_counter()
        torch.from_numpy(arr).copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        unreg(arr)
        t3 = time.perf_counter()
        print(f"{label}: register {1e3 * (t1 - t0):.2f} ms, D2H {1e3 * (t2 - t1):.2f} ms, unregister {1e3 * (t3 - t2):.2f} ms",
              flush=True)
x = np.ones((1, 1025 ** 2), np.complex128)
for _ in range(3):
    t0 = time.perf_counter()
    reg(x)
    t1 = time.perf_counter()
    y = torch.from_numpy(x).to(dev, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    unreg(x)
    t3 = time.perf_counter()
    print(f"upload 16.8 MB: register {1e3 * (t1 - t0):.2f}, H2D {1e3 * (t2 - t1):.2f}, unregister {1e3 * (t3 - t2):.2f} ms")

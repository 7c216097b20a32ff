"""Host memory copy strategies for the staging path (development helper)."""
import concurrent.futures as cf
import time

import numpy as np
import torch

n = 16 << 20
src = np.random.default_rng(0).standard_normal(n // 8)
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pin_np = pin.numpy()
src_u8 = src.view(np.uint8)
pool = cf.ThreadPoolExecutor(8)


def t(label, fn, reps=10):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - t0) / reps
    print(f"{label:50s} {dt * 1e3:7.3f} ms  {n / dt / 1e9:6.1f} GB/s", flush=True)


t("torch copy_ uint8 pageable->pinned", lambda: pin.copy_(torch.from_numpy(src_u8)))
t("torch copy_ float64 pageable->pinned", lambda: pin.view(torch.float64).copy_(torch.from_numpy(src)))
t("np.copyto single thread", lambda: np.copyto(pin_np, src_u8))


def par(k):
    step = n // k

    def one(i):
        np.copyto(pin_np[i * step:(i + 1) * step], src_u8[i * step:(i + 1) * step])

    list(pool.map(one, range(k)))


for k in (2, 4, 8):
    t(f"np.copyto x{k} threads", lambda k=k: par(k))
print("torch threads", torch.get_num_threads())

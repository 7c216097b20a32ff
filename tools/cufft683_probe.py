"""cuFFT probe (development helper): batched length-683 (and 43) DFTs, contiguous and strided."""
import torch
dev = torch.device("cuda", 0)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for P, R, rings in ((683, 12, 4098), (43, 12, 16 * 258)):
    x = torch.randn(rings * 3 * R, P, dtype=torch.complex128, device=dev)
    ms = t(lambda: torch.fft.fft(x, dim=-1))
    gb = x.numel() * 16 * 2 / 1e9
    print(f"P={P}: batch {x.shape[0]} contiguous {ms:.3f} ms ({gb / ms:.0f} GB/ms = TB/s x1e0)")
    # strided: residue-major view of a ring field (rings, n, 3): x[ring, r + R q, c]
    f = torch.randn(rings, R * P, 3, dtype=torch.complex128, device=dev)
    v = f.view(rings, P, R, 3)  # element (ring, q, r, c) = f[ring, q R + r, c]: DFT over q
    ms2 = t(lambda: torch.fft.fft(v, dim=1))
    print(f"P={P}: strided over q (torch may copy) {ms2:.3f} ms")

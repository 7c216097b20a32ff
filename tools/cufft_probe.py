"""cuFFT probe (development helper): C4 / C2 ring lengths, contiguous vs strided layouts."""
import torch
dev = torch.device("cuda", 0)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for (nr, n) in ((4098, 8196), (16 * 258, 516), (4 * 1026, 2052)):
    x = torch.randn(nr, n, 3, dtype=torch.complex128, device=dev)
    xc = x.permute(2, 0, 1).contiguous()
    gb = x.numel() * 16 * 2 / 1e9
    ms_c = t(lambda: torch.fft.fft(xc, dim=-1))
    ms_s = t(lambda: torch.fft.fft(x, dim=1))
    ms_tr = t(lambda: x.permute(2, 0, 1).contiguous())
    print(f"rings {nr} x3 n={n}: contiguous {ms_c:.3f} ms ({gb/ms_c:.0f} GB/s)  strided(dim=1) {ms_s:.3f} ms  transpose {ms_tr:.3f} ms")

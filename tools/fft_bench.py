"""cuFFT Z2Z throughput at the ring lengths of C2/C3/C4 (development helper)."""
import torch, time
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for (L, B) in ((256, 16), (1024, 4), (4096, 1)):
    nth, nph = L + 2, 2 * L + 4
    x = torch.randn(B, nth * nph, 3, dtype=torch.complex128, device="cuda")
    xc = x.permute(2, 0, 1).contiguous().view(3 * B * nth, nph)
    gb = x.numel() * 16 / 1e9
    ms_c = t(lambda: torch.fft.fft(xc, dim=-1))
    xs = x.view(B * nth, nph, 3)
    ms_s = t(lambda: torch.fft.fft(xs, dim=1))
    ms_tr = t(lambda: x.permute(2, 0, 1).contiguous())
    print(f"L={L} B={B}: contiguous fft {ms_c:.3f} ms ({2*gb/ms_c:.0f} GB/s eff), strided {ms_s:.3f} ms, transpose copy {ms_tr:.3f} ms; data {gb*1e3:.0f} MB")

"""Host link probe (development helper): pinned H2D / D2H bandwidth alone and concurrent."""
import torch, time
dev = torch.device("cuda", 0)
n = 404_227_584 // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True); h_in.fill_(1.0)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device=dev); d_b = torch.empty(n, dtype=torch.float64, device=dev)
s1 = torch.cuda.Stream(dev); s2 = torch.cuda.Stream(dev)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
gb = n * 8 / 1e9
t = timeit(lambda: d_a.copy_(h_in, non_blocking=True)); print(f"H2D alone {gb/t:.1f} GB/s")
t = timeit(lambda: h_out.copy_(d_b, non_blocking=True)); print(f"D2H alone {gb/t:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
t = timeit(both); print(f"concurrent H2D+D2H {gb/t:.1f} GB/s each way")
for parts in (4, 16, 64):
    k = n // parts
    def chunked():
        for i in range(parts):
            with torch.cuda.stream(s1): d_a[i*k:(i+1)*k].copy_(h_in[i*k:(i+1)*k], non_blocking=True)
            with torch.cuda.stream(s2): h_out[i*k:(i+1)*k].copy_(d_b[i*k:(i+1)*k], non_blocking=True)
    t = timeit(chunked); print(f"concurrent chunked x{parts} {gb/t:.1f} GB/s each way")
# copy-engine-free alternative: a kernel reading mapped host memory (zero-copy) for H2D
hv = h_in
def zc():
    d_a.copy_(hv, non_blocking=True)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:2000])
import os; print("cpus", os.cpu_count())
print(open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0])

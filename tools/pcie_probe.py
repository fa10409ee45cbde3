"""PCIe copy rates with pinned host memory: H2D alone, D2H alone, both at once."""
import torch, time
n = 1 << 31  # 8 GiB of f32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t
GB = n * 4 / 1e9
for _ in range(2):
    t1 = timeit(lambda: d_a.copy_(h_in, non_blocking=True))
    t2 = timeit(lambda: h_out.copy_(d_b, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    t3 = timeit(both)
    print(f"H2D {GB/t1:.1f} GB/s  D2H {GB/t2:.1f} GB/s  both {2*GB/t3:.1f} GB/s total ({t3*1e3:.0f} ms for {GB:.1f}+{GB:.1f} GB)")

import torch, time
n = 3_200_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    th = t(lambda: d.copy_(h, non_blocking=True))
    tdh = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    tb = t(both)
print(f"H2D {n/th/1e9:.1f} GB/s  D2H {n/tdh/1e9:.1f} GB/s  both concurrently {2*n/tb/1e9:.1f} GB/s total ({tb*1e3:.1f} ms for 2x3.2 GB)")

import torch, time
n = 1 << 29  # 4 GiB of int64
h1 = torch.empty(n, dtype=torch.int64, pin_memory=True); h2 = torch.empty(n, dtype=torch.int64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.int64, device="cuda"); d2 = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
b = n * 8
print("H2D GB/s", b / t(lambda: d1.copy_(h1, non_blocking=True)) / 1e9)
print("D2H GB/s", b / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("both (each dir) GB/s", b / t(both) / 1e9)

import torch, time
n = 512 * 1024 * 1024 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device='cuda'); d2 = torch.empty(n, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bo = t(both)
GB = n * 8 / 1e9
print(f"H2D {GB/h2d:.1f} GB/s  D2H {GB/d2h:.1f} GB/s  concurrent {2*GB/bo:.1f} GB/s total ({GB/bo:.1f} each)")

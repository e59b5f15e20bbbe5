import torch, time
n = 512*1024*1024
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(both):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        if both:
            with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    return n / dt / 1e9
print("H2D alone GB/s", run(False))
print("H2D with concurrent D2H, each direction GB/s", run(True))
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize(); print("D2H alone GB/s", n/((time.perf_counter()-t)/5)/1e9)

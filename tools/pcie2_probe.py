import time, torch
n = 283115520
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def one():
    d.copy_(h, non_blocking=True)
def two(k):
    chunk = n // 4 // k
    ss = [torch.cuda.Stream() for _ in range(k)]
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
for f, name in ((one, "1 stream"), (lambda: two(2), "2 streams"), (lambda: two(4), "4 streams"), (lambda: two(8), "8 streams")):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t) / 5
    print(f"{name}: {n / el / 1e9:.1f} GB/s")

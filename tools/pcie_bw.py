import torch, time
x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for name, f in [("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(name, round(ms, 3), "ms for 64 MiB", round(64 * 1.048576 / ms, 1), "GB/s")
# bidirectional concurrently
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
x2 = torch.empty(64 << 20, dtype=torch.uint8).pin_memory(); d2 = torch.empty_like(d)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): x2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print("both", round((time.perf_counter() - t) / 10 * 1e3, 3), "ms")

import torch, time
n = 24_696_000 // 8
a = torch.empty(n, dtype=torch.float64).pin_memory(); b = torch.empty(4*n, dtype=torch.float64).pin_memory()
d = torch.empty(5*n, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, k=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/k
def one(): d[:n].copy_(a, non_blocking=True)
def two():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d[:n//2].copy_(a[:n//2], non_blocking=True)
    with torch.cuda.stream(s2): d[n//2:n].copy_(a[n//2:], non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
def big(): d[n:].copy_(b, non_blocking=True)
for name, f, by in [("pos 1 stream", one, 8*n), ("pos 2 streams", two, 8*n), ("moments", big, 32*n)]:
    ms = t(f); print(name, ms, "ms", by/ms/1e6, "GB/s")

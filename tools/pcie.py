"""Pinned host<->device copy bandwidth (the e2e ceiling): H2D alone, D2H alone, both concurrently."""
import torch
n = 768 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e[0].record()
    for _ in range(reps): fn()
    e[1].record(); torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / reps
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bt = t(both)
print(f"H2D {n/h2d/1e6:.1f} GB/s  D2H {h2.numel()/d2h/1e6:.1f} GB/s  both: {bt:.2f} ms for {n>>20} MB up + {h2.numel()>>20} MB down")

#!/usr/bin/env python3
"""Dev probe: pinned H2D / D2H / concurrent copy bandwidth on cuda:0."""
import torch
m = 256 << 20
h = torch.empty(m, dtype=torch.uint8).pin_memory(); h2 = torch.empty(m, dtype=torch.uint8).pin_memory()
d = torch.empty(m, dtype=torch.uint8, device="cuda"); d2 = torch.empty(m, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    f(); torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1e-3
h2d = t(lambda: d.copy_(h, non_blocking=True)); d2h = t(lambda: h.copy_(d, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bt = t(both)
print(f"H2D {m/h2d/1e9:.1f} GB/s  D2H {m/d2h/1e9:.1f} GB/s  concurrent H2D+D2H {2*m/bt/1e9:.1f} GB/s total")

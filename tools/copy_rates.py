"""Pinned host <-> device copy rates on this box (the e2e bound of bench.py)."""
import torch

def rate(nbytes, d2h, both=False):
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    h2 = torch.empty_like(h).pin_memory() if both else None
    d2 = torch.empty_like(d) if both else None
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        (h.copy_(d, non_blocking=True) if d2h else d.copy_(h, non_blocking=True))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    with torch.cuda.stream(s1):
        for _ in range(5):
            (h.copy_(d, non_blocking=True) if d2h else d.copy_(h, non_blocking=True))
    if both:
        with torch.cuda.stream(s2):
            for _ in range(5):
                d2.copy_(h2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return 5 * nbytes / (a.elapsed_time(b) / 1e3) / 1e9

print(f"H2D {rate(1_200_000_000, False):.1f} GB/s")
print(f"D2H {rate(1_600_000_000, True):.1f} GB/s")
print(f"D2H with concurrent H2D: {rate(1_600_000_000, True, both=True):.1f} GB/s (D2H bytes only)")

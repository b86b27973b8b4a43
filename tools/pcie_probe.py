"""PCIe probe: pinned H2D / D2H / both at once, 160 MB and 94 MB (the c2b batch's copies)."""
import torch

h_in = torch.empty(160_000_000, dtype=torch.uint8).pin_memory()
h_out = torch.empty(94_000_000, dtype=torch.uint8).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty_like(h_out, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
bo = t(both)
print(f"H2D 160 MB {h2d:.3f} ms ({160 / h2d:.1f} GB/s); D2H 94 MB {d2h:.3f} ms ({94 / d2h:.1f} GB/s); "
      f"both {bo:.3f} ms")

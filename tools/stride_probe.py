"""DRAM probe (experiment tool): achieved read bandwidth of one 8-byte word per S bytes over a
134 MB array (the remap's phys-page gather at 64 KiB granularity is S = 128), against a
contiguous read of the same array.  Prints GB/s of USEFUL bytes and of sector bytes."""
import torch

n = 16 * 1048576                       # 16 Mi u64 = 134 MB (64 GiB of 4 KiB pages)
x = torch.arange(n, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for stride in (1, 2, 4, 8, 16, 64, 512):
    v = x[::stride]
    ms = t(lambda: v.sum())
    useful = v.numel() * 8
    sector = max(useful, v.numel() * 32) if stride >= 4 else n * 8
    print(f"stride {stride * 8:5d} B: {ms * 1e3:7.1f} us  useful {useful / ms / 1e6:7.0f} GB/s  "
          f"sectors {sector / ms / 1e6:7.0f} GB/s", flush=True)

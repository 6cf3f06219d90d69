"""Store-bandwidth micro: time torch fill_ over buffers the size of the Eq. 3 table (config 3:
32 units x 32 groups x 8192 x 8 B = 64 MiB; config 4: 16 MiB) to bound k_table's store stream.
Measurement only (no part of the product path)."""
import torch

def t(fn, reps=50):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for mb in (16, 64, 256):
    x = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    us = t(lambda: x.fill_(1))
    print(f"fill {mb} MiB: {us:.1f} us  {(mb << 20) / us / 1e3:.0f} GB/s")

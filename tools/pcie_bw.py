"""Pinned host<->device copy bandwidth vs copy size (for the e2e floor in bench.py)."""
import torch

total = 116 << 20
hb = torch.empty(total, dtype=torch.uint8).pin_memory()
hb.fill_(1)
db = torch.empty(total, dtype=torch.uint8, device="cuda")
for chunk in (1 << 20, 2 << 20, 8 << 20, 16 << 20, 32 << 20, total):
    for name, dst, src in (("h2d", db, hb), ("d2h", hb, db)):
        def go():
            for o in range(0, total, chunk):
                dst[o:o + chunk].copy_(src[o:o + chunk], non_blocking=True)
        go(); go()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            go()
        z.record()
        torch.cuda.synchronize()
        print(f"{name} chunk {chunk >> 20:4d} MiB: {5 * total / (a.elapsed_time(z) / 1e3) / 1e9:6.1f} GB/s")

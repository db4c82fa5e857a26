"""Pure-read HBM bandwidth reference points on this GPU (diagnostics): torch
reductions over a 2 GiB bf16 buffer and a strided 'many streams' read."""
import torch

a = torch.empty(2 ** 30, dtype=torch.bfloat16, device="cuda").normal_()
for name, fn in (("sum", lambda: a.sum(dtype=torch.float32)), ("amax", lambda: a.amax())):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name}: {a.numel() * 2 / ms / 1e6:.0f} GB/s")

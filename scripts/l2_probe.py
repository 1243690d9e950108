"""L2-resident vs HBM streaming read bandwidth (torch sum over a buffer)."""
import torch
for mb in (16, 32, 64, 96, 128, 256, 1024, 4096):
    n = mb * 1024 * 1024 // 8
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        x.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        x.sum()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{mb:5d} MB: {ms*1e3:8.1f} us  {n*8/ms/1e6:8.1f} GB/s", flush=True)

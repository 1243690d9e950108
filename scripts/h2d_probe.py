"""H2D bandwidth from pinned host memory: one stream vs the same bytes split
over 2 / 4 streams (copy engines), 283.6 MB like the e2e upload."""
import torch

n = 283_639_816 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4, 1, 2, 4):
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        chunk = (n + ns - 1) // ns
        evs = []
        for i in range(ns):
            s = streams[i]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
        for ev in evs:
            cur.wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"streams {ns}: {ms:.3f} ms  {n * 8 / ms / 1e6:.1f} GB/s", flush=True)

"""Pinned host -> device copy bandwidth (the e2e leg's ceiling)."""
import json, time, torch
n = 200_000_000  # 1.6 GB
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for chunk in (1 << 20, 1 << 22, n):
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for b in range(0, n, chunk):
        d[b:b + chunk].copy_(h[b:b + chunk], non_blocking=True)
    ev1.record(); torch.cuda.synchronize()
    print(json.dumps({"chunk_doubles": chunk, "GBps": 8 * n / (ev0.elapsed_time(ev1) * 1e-3) / 1e9}))

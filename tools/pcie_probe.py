"""Pinned host <-> device copy bandwidth on the box (the e2e leg's transfers)."""
import json, torch
out = {}
for mb in (1.6, 4.7, 64):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        out[f"{name}_{mb}MB"] = {"us": round(ms * 1e3, 1), "GBps": round(n / ms / 1e6, 1)}
print(json.dumps(out))

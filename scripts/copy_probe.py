"""Pinned host <-> HBM copy bandwidth on this box for 1, 2 and 4 concurrent
streams (the e2e sweep's downloads are the exposed tail).

    python scripts/copy_probe.py
"""
import json
import time

import torch

nbytes = 64 << 20
dev = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
host = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
for direction in ("h2d", "d2h"):
    for ns in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        chunks_d = dev.chunk(ns)
        chunks_h = host.chunk(ns)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                for st, d, h in zip(streams, chunks_d, chunks_h):
                    with torch.cuda.stream(st):
                        if direction == "h2d":
                            d.copy_(h, non_blocking=True)
                        else:
                            h.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 5
        print(json.dumps({"dir": direction, "streams": ns, "GB_s": nbytes / dt / 1e9}), flush=True)

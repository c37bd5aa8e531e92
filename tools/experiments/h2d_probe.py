"""Pinned host -> device copy bandwidth with 1 / 2 / 4 concurrent streams and
several chunk sizes (is one upload stream the end-to-end path's ceiling?)."""
import time

import torch

dev = torch.device("cuda", 0)
total = 1 << 30
h = torch.empty(total, dtype=torch.uint8).pin_memory()
d = torch.empty(total, dtype=torch.uint8, device=dev)
for chunk_mb in (4, 12, 64):
    chunk = chunk_mb << 20
    n = total // chunk
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream(dev) for _ in range(ns)]
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(n):
                with torch.cuda.stream(streams[i % ns]):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"chunk {chunk_mb:3d} MB  streams {ns}: {n * chunk / dt / 1e9:6.1f} GB/s", flush=True)

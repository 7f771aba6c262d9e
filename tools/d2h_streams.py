"""Pinned D2H bandwidth vs copy size and number of streams (PCIe check).

    python tools/d2h_streams.py
"""
import torch, time
for mb in (100, 201, 400):
    n = mb * 1024 * 1024 // 4
    src = torch.empty(n, device="cuda")
    dst = torch.empty(n).pin_memory()
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        chunks_s = src.chunk(ns); chunks_d = dst.chunk(ns)
        for _ in range(2):
            for s, a, b in zip(streams, chunks_s, chunks_d):
                with torch.cuda.stream(s): b.copy_(a, non_blocking=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            for s, a, b in zip(streams, chunks_s, chunks_d):
                with torch.cuda.stream(s): b.copy_(a, non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"{mb} MB, {ns} streams: {mb * 1.048576e6 / dt / 1e9:.1f} GB/s")

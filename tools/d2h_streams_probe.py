"""D2H bandwidth of one 2.08 GB transfer (config 2's unique columns) into
page-locked host memory split over S concurrent CUDA streams (chunks of
C MB dealt round-robin): does a second copy engine raise the PCIe rate?
python tools/d2h_streams_probe.py"""
import time

import torch

n = 2_080_800_000 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda").fill_(1.0)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(4)]


def run(S, chunk_mb):
    c = chunk_mb * (1 << 20) // 8
    i = 0
    for k, off in enumerate(range(0, n, c)):
        s = streams[k % S]
        with torch.cuda.stream(s):
            h[off:off + c].copy_(d[off:off + c], non_blocking=True)
        i += 1
    torch.cuda.synchronize()


for S in (1, 2, 4):
    for chunk in (6, 32):
        run(S, chunk)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            run(S, chunk)
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[2]
        print(f"streams={S} chunk={chunk} MB: {t * 1e3:.1f} ms = {n * 8 / t / 1e9:.1f} GB/s",
              flush=True)

import torch, time
n = 2_080_800_000 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda").fill_(1.0)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for _ in range(2): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
t = sorted(ts)[2]
print(f"D2H pinned {n*8/1e9:.2f} GB: {t*1e3:.1f} ms = {n*8/t/1e9:.1f} GB/s")
h2 = torch.empty_like(h)
for _ in range(2): h2.copy_(h)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); h2.copy_(h); ts.append(time.perf_counter() - t0)
t = sorted(ts)[2]
print(f"host copy (torch, {torch.get_num_threads()} threads) {n*8/1e9:.2f} GB: {t*1e3:.1f} ms = {n*8/t/1e9:.1f} GB/s")

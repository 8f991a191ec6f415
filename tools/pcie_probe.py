import torch, time, json
n = 99532800 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory(); d = torch.empty(n, device="cuda")
o = torch.empty(33177600 // 4, device="cuda"); ho = torch.empty(33177600 // 4).pin_memory()
for _ in range(3): d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); up = 10 * 99532800 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(10): ho.copy_(o, non_blocking=True)
torch.cuda.synchronize(); down = 10 * 33177600 / (time.perf_counter() - t) / 1e9
s2 = torch.cuda.Stream()
t = time.perf_counter()
for _ in range(10):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(o, non_blocking=True)
torch.cuda.synchronize(); both = 10 * 99532800 / (time.perf_counter() - t) / 1e9
print(json.dumps({"h2d_GBs": up, "d2h_GBs": down, "h2d_GBs_with_concurrent_d2h": both,
                  "frame_bound_ms": 99532800 / up / 1e6, "frame_bound_mpix_s": 8294400 / (99532800 / up) / 1e6 * 1e3 / 1e3}))

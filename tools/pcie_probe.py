import torch, time
for nbytes in (147456, 786432, 1572864, 3145728):
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    for direction in ("d2h", "h2d"):
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if direction == "d2h": h.copy_(d, non_blocking=True)
            else: d.copy_(h, non_blocking=True)
            e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(direction, nbytes, "median us", round(ts[10], 2), "GB/s", round(nbytes / ts[10] / 1e3, 2))
# host wake latency: tiny kernel + sync
x = torch.zeros(1, device="cuda")
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); x.add_(1); torch.cuda.current_stream().synchronize(); ts.append((time.perf_counter() - t0) * 1e6)
ts.sort(); print("launch+sync round trip us", round(ts[25], 2))

"""Host-to-device copy bandwidth of a c3 record (276 MB, pinned) on one and two copy streams
(the e2e path's input transfer)."""
import torch, time
n = 360000 * 192
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(4)]
for ns in (1, 2, 4):
    st = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for j in range(8):
            with torch.cuda.stream(st[j % ns]):
                d[j % 4].copy_(h[j % 4], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{ns} stream(s): {8 * n * 4 / dt / 1e9:.1f} GB/s")

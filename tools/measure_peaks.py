"""Measure the roofline denominators MEASURED_PEAKS.json lacks: FP64 (cuBLAS DGEMM),
TF32 and INT8 GEMM rates on this B200, plus host facts for the CPU baseline.
Writes gpurun_out/peaks_extra.json. Library GEMMs here are only a yardstick."""
import json, os, time, platform
import torch

def bench(fn, iters=10):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

def sustained(fn, flops, secs=4.0):
    torch.cuda.synchronize(); t0 = time.time(); n = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < secs:
        fn(); n += 1
        if n % 4 == 0: torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    return flops * n / (s.elapsed_time(e) / 1e3)

out = {}
dev = torch.device("cuda")
n = 8192
a = torch.randn(n, n, device=dev, dtype=torch.float64); b = torch.randn(n, n, device=dev, dtype=torch.float64)
c = torch.empty_like(a)
f = lambda: torch.matmul(a, b, out=c)
f(); t = bench(f, 5)
out["fp64_dgemm_tflops_burst"] = 2 * n**3 / t / 1e12
out["fp64_dgemm_tflops_sustained"] = sustained(f, 2 * n**3, 4.0) / 1e12
del a, b, c
torch.backends.cuda.matmul.allow_tf32 = True
a = torch.randn(n, n, device=dev); b = torch.randn(n, n, device=dev); c = torch.empty_like(a)
f = lambda: torch.matmul(a, b, out=c)
f(); t = bench(f)
out["tf32_tflops_burst"] = 2 * n**3 / t / 1e12
del a, b, c
try:
    a = torch.randint(-127, 127, (n, n), device=dev, dtype=torch.int8)
    b = torch.randint(-127, 127, (n, n), device=dev, dtype=torch.int8).t()
    f = lambda: torch._int_mm(a, b)
    f(); t = bench(f)
    out["int8_tops_burst"] = 2 * n**3 / t / 1e12
except Exception as ex:
    out["int8_err"] = str(ex)[:200]
# HBM copy for cross-check
x = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev); y = torch.empty_like(x)
f = lambda: y.copy_(x)
f(); t = bench(f)
out["hbm_copy_gbs"] = 2 * x.numel() * 2 / t / 1e9
out["host_cores"] = len(os.sched_getaffinity(0))
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    out["cpu_model"] = platform.processor()
out["gpu"] = torch.cuda.get_device_name(0)
out["sm_count"] = torch.cuda.get_device_properties(0).multi_processor_count
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/peaks_extra.json", "w"), indent=1)
print(json.dumps(out))

"""Measure the FP64 DGEMM peak on the box (MEASURED_PEAKS.json has no FP64 entry).

torch.matmul float64 8192^3 (2*N^3 flops): best of 10 (burst) and back to back
for 4 s (sustained), CUDA events on the current stream — mirrors how the driver
measured bf16. Also records host core count / CPU model for the cpu_baseline.
"""
import json, os, platform, subprocess, time
import torch

def main():
    dev = torch.device("cuda:0")
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b, out=c); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    flops = 2.0 * n ** 3
    # sustained
    t0 = time.time(); cnt = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c); cnt += 1
        if cnt % 8 == 0:
            torch.cuda.synchronize()
    e.record(); e.synchronize()
    sus = cnt * flops / (s.elapsed_time(e) / 1e3)
    # HBM copy for reference
    x = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev); y = torch.empty_like(x)
    bw = 0.0
    for _ in range(10):
        s.record(); y.copy_(x); e.record(); e.synchronize()
        bw = max(bw, 2 * x.numel() * 2 / (s.elapsed_time(e) / 1e3))
    try:
        cpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = [l.split(":", 1)[1].strip() for l in cpu.splitlines() if l.startswith("Model name")]
    except Exception:
        model = []
    out = {"fp64_tflops": flops / best / 1e12, "fp64_tflops_sustained": sus / 1e12,
           "hbm_gbs_copy": bw / 1e9, "nproc": os.cpu_count(),
           "cpu_model": model[0] if model else platform.processor(),
           "gpu": torch.cuda.get_device_name(0),
           "how": "torch.matmul float64 8192^3, best of 10 / 4 s back-to-back; bf16 1Gi copy best of 10"}
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/fp64_peak.json", "w") as f:
        json.dump(out, f, indent=1)

if __name__ == "__main__":
    main()

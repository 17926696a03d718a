"""Measure the FP64 roofline denominators on the GPU box: cuBLAS DGEMM (torch.matmul
float64), burst and sustained, plus the HBM copy bandwidth. Prints one JSON line."""
import json, time, torch

def dgemm(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n ** 3 / (best * 1e-3) / 1e12
    # sustained: back to back for ~4 s
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    it = 0; e0.record(); t0 = time.time()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c); it += 1
        if it % 4 == 0: torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sustained = 2 * n ** 3 * it / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return burst, sustained

def copy_bw(nbytes=4 << 30):
    a = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda"); a.fill_(1.0)
    b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    torch.cuda.synchronize(); best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * nbytes / (best * 1e-3) / 1e9

if __name__ == "__main__":
    burst, sust = dgemm()
    print(json.dumps({"dgemm_tflops_burst": round(burst, 3), "dgemm_tflops_sustained": round(sust, 3),
                      "hbm_copy_gbs": round(copy_bw(), 1), "gpu": torch.cuda.get_device_name()}))

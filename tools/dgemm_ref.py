"""cuBLAS DGEMM throughput (library reference point for the FP64 roofline)."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5 if n < 16384 else 2
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"probe": "cublas_dgemm", "n": n, "tflops": round(2 * n**3 / ms / 1e9, 2), "ms": round(ms, 3)}))

"""cuBLAS DGEMM at the trailing-update shape (C -= A B^T, K = tile)."""
import json, torch
for (m, k) in [(16384, 256), (32768, 256), (16384, 512), (32768, 512), (8192, 8192)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    c = torch.randn(m, m, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c.addmm_(a, a.T, alpha=-1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        c.addmm_(a, a.T, alpha=-1.0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"probe": "cublas_addmm_NT", "m": m, "k": k, "tflops": round(2 * m * m * k / ms / 1e9, 2)}))

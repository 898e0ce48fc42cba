"""A few tile POTRF launches (for ncu)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_4886_b200 import spawn
b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cl = spawn(1, tile=b)
B = np.random.default_rng(0).standard_normal((b, b))
A = B @ B.T + b * np.eye(b)
t0 = torch.from_numpy(np.tril(A).T.copy()).to(cl.device)
w = torch.empty_like(t0)
info = ctypes.c_int64()
for _ in range(3):
    w.copy_(t0)
    cl.lib.bgp_tile_potrf(cl._ctx, ctypes.c_void_p(w.data_ptr()), b, 0, ctypes.byref(info), cl.stream)
L = np.tril(w.cpu().numpy().T)
print("info", info.value, "err", np.abs(L @ L.T - A).max() / np.abs(A).max())
cl.shutdown()

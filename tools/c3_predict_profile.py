"""C3 kriging: time predict(se_fit=True) at fresh thetas (tile from argv)."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from oracle.blockgp_oracle import c3_pred_coords, config_inputs
from paper_1305_4886_b200 import spawn
from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
tile = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cl = spawn(1, tile=tile)
kern, X, theta, extra, z = config_inputs(3)
Xp = c3_pred_coords(64)
spec = builtin_spec(kern, X, Xp, **extra)
y = np.random.default_rng(0).standard_normal(len(X))
prob = KrigeProblem(cl, "c3", spec, y, theta, m=len(Xp))
prob.log_density()
th = np.array(theta, dtype=float); th[1] += 1e-12
prob.log_density(th)
for k in range(3):  # fresh theta each time: log_density + predict, predict timed alone
    th = np.array(theta, dtype=float); th[1] += (k + 2) * 1e-12
    prob.log_density(th)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    prob.predict(se_fit=True)
    torch.cuda.synchronize(); print("predict_s", round(time.perf_counter() - t0, 4))
cl.shutdown()

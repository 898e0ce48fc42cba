"""Time one FULL reference-algorithm evaluation at C4 on this host.

Run on a GPU box (its host cores are the CPU baseline's):
    python tools/cpu_full_eval.py > profiles/r02_cpu_full_eval.json
Warm-up: one evaluation at another theta on n = 8,192 (BLAS thread pool,
page faults), then the timed C4 evaluation (oracle/full_eval.py, BLAS on all
host threads).  Records nproc, the lscpu model and the parity of the ll
against the survey's golden.  bench.py reports the committed record beside
the sampler's extrapolation.
"""

import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import full_eval  # noqa: E402
from oracle.cpu_baseline import host_cores  # noqa: E402


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    except OSError:
        return None
    info = {}
    for line in out.splitlines():
        k, _, v = line.partition(":")
        if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
            info[k.strip()] = v.strip()
    return info


def main():
    d = np.load(os.path.join(ROOT, "tests", "golden", "c4_inputs.npz"))
    with open(os.path.join(ROOT, "tests", "golden", "c4_scalars.json")) as f:
        sc = json.load(f)
    X, y = d["X"], d["y"]
    log = lambda m: print(m, file=sys.stderr, flush=True)  # noqa: E731
    t0 = time.perf_counter()
    full_eval.log_density(X[:8192], y[:8192], np.array([1.0, 0.1, 0.02]))
    warm = time.perf_counter() - t0
    log(f"warm-up {warm:.1f} s")
    r = full_eval.log_density(X, y, np.array([1.0, 0.08, 0.02]), log=log)
    ref = sc["survey"]["ll"]
    rec = {"what": "one full C4 evaluation of the reference algorithm (P=1 block sweep, "
                   "oracle/full_eval.py), construct single-threaded numpy, BLAS on all threads",
           "n": len(y), "nproc": os.cpu_count(), "cores_used": host_cores(),
           "lscpu": lscpu_model(), "warmup_s": warm, **r,
           "evals_per_s": 1.0 / r["eval_s"], "ll_ref": ref,
           "ll_rel_err": abs(r["ll"] - ref) / abs(ref)}
    print(json.dumps(rec))


if __name__ == "__main__":
    main()

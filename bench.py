"""Benchmark: GP log-likelihood evaluations at n = 67,275 (BASELINE config 4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--tile 256]

A step is one `KrigeProblem.log_density(theta)` at a fresh theta (range
rho_k = 0.08 + k*1e-12, so every step rebuilds): covariance construction,
tiled Cholesky, forward solve, log-determinant and sum of squares on the
GPU.  Inputs are BASELINE.json config 4 (SURVEY.md 8d recipe, frozen in
tests/golden/c4_inputs.npz): 67,275 points in [0,1]^2 with 10 % jittered
duplicates, exponential covariance theta = (1, 0.08, 0.02).  The 18.1 GB
covariance is rebuilt every step, so every timed step streams a working set
far larger than the 126 MB L2.

Prints ONE JSON line (rank 0).  `value` is evaluations/s over the whole job
with inputs resident on the device; `e2e` repeats the measurement through the
public API from host arrays (coords + y uploaded, scalars read back, every
step).  `roofline` is the trailing-update DMMA kernel (the dominant one)
against the measured FP64 DMMA peak; `cpu_baseline` / `--impl reference` time
the reference algorithm on the host cores (oracle/cpu_baseline.py).

With --gpus N > 1 the evaluation is sharded over N GPUs of the box: one
process per GPU (started here under torch.distributed.run when the caller
did not launch the ranks itself), the covariance tiles spread 2-D
block-cyclically (paper_1305_4886_b200/parallel.py), one launch per sweep
step with the panel solve + NVLink push inside it; `value` is evaluations/s
of the whole job (strong scaling: the problem size is fixed).  N larger than
the visible GPU count is refused.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Cholesky FP64 TFLOP/s and log-lik evals/sec at n=67,275, 1/2/4/8 B200"
THETA = np.array([1.0, 0.08, 0.02])
# measured FP64 peaks (profiles/r01_fp64_peaks.jsonl): DMMA.8x8x4 in-register
# loop 37.1 TFLOP/s; cuBLAS DGEMM 16384^3 35.8 TFLOP/s.  MEASURED_PEAKS.json
# carries no FP64 entry, so the roofline uses the DMMA probe.
FP64_DMMA_PEAK = 37.1
CUBLAS_DGEMM = 35.8
REF_SUB_BLOCKS = 20  # reference sampler: sub-evaluation of 20 reference blocks (19,800 points)


# the committed ncu --set full capture of one C4 trailing-update launch
# (k = 111 tiles of 512) that the roofline's `traffic` comes from
GEMM_NCU_CAPTURE = "profiles/r02final5_ncu_gemm_full.txt"


def hbm_kernels():
    """The HBM-bound kernels of a C4 step from the committed ncu captures
    (same pass as GEMM_NCU_CAPTURE): achieved GB/s of algorithmic bytes
    against the measured HBM copy bandwidth (MEASURED_PEAKS.json)."""
    import re
    peak = None
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6549.1  # the pool's measured copy bandwidth (round-2 MEASURED_PEAKS.json)
    out = {}
    for name, suffix in (("cov_tri_kernel (K1, covariance build)", "ncu_cov_full.txt"),
                         ("trsv_fwd_persistent_kernel (K3a, forward solve)", "ncu_trsv_full.txt")):
        path = os.path.join(ROOT, GEMM_NCU_CAPTURE.replace("ncu_gemm_full.txt", suffix))
        if not os.path.exists(path):
            continue
        m = re.search(r"achieved ([0-9.]+) GB/s", open(path).read())
        if m:
            gbs = float(m.group(1))
            out[name] = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "source": os.path.relpath(path, ROOT)}
    return out


def gemm_traffic():
    """DRAM bytes (read + write) of one trailing-update launch from the
    committed ncu --set full capture (GEMM_NCU_CAPTURE), with the algorithmic
    bytes of the same launch (C tiles read + written once, panel tiles read
    once) as the summary states them; None when no capture is committed."""
    import re
    path = os.path.join(ROOT, GEMM_NCU_CAPTURE)
    if not os.path.exists(path):
        return None, None
    txt = open(path).read()
    m = re.search(r"traffic \(read\+write\)\s+([0-9.e+]+) B", txt)
    a = re.search(r"algorithmic bytes\s+([0-9.e+]+) B", txt)
    head = txt.splitlines()[0].lstrip("# ").strip()
    if not m:
        return None, None
    return float(m.group(1)), {"file": os.path.relpath(path, ROOT), "launch": head,
                               "algorithmic_bytes": float(a.group(1)) if a else None}


def load_c4():
    d = np.load(os.path.join(ROOT, "tests", "golden", "c4_inputs.npz"))
    with open(os.path.join(ROOT, "tests", "golden", "c4_scalars.json")) as f:
        sc = json.load(f)
    return d["X"], d["y"], sc


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, power, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_setup(impl, share_gpu=False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if impl == "reference" or share_gpu:
            dist.init_process_group("gloo")
        else:
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def full_eval_record():
    """Timed FULL reference-algorithm evaluations at C4 on a GPU box's host
    (tools/cpu_full_eval.py, committed under profiles/), reported beside the
    sampler's extrapolation; None if none is committed."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_cpu_full_eval.json")))
    if not files:
        return None
    runs = []
    for f in files:
        with open(f) as fh:
            rec = json.load(fh)
        runs.append({"file": os.path.relpath(f, ROOT), "eval_s": rec["eval_s"],
                     "construct_s": rec["construct_s"], "cholesky_s": rec["cholesky_s"],
                     "ll_rel_err": rec["ll_rel_err"]})
    mean = statistics.mean(r["eval_s"] for r in runs)
    return {"what": rec["what"], "n": rec["n"], "cores_used": rec["cores_used"], "lscpu": rec["lscpu"],
            "runs": runs, "eval_s_mean": mean, "evals_per_s": 1.0 / mean}


def cpu_reference(samples, X):
    """Sampled reference evaluation time: the median over `samples`
    sub-evaluations of each one's extrapolated evaluation time."""
    from oracle.cpu_baseline import SubEvalSampler, host_cores
    s = SubEvalSampler(X, THETA, blocks=REF_SUB_BLOCKS)
    evals, chols, walls = [], [], []
    for _ in range(samples):
        t, wall = s.sample()
        walls.append(wall)
        total, chol = s.extrapolate(t)
        evals.append(total)
        chols.append(chol)
    total, chol = statistics.median(evals), statistics.median(chols)
    n = s.n
    return {"evals_per_s": 1.0 / total, "eval_s": total, "chol_s": chol,
            "eval_s_range": [min(evals), max(evals)],
            "chol_tflops": n ** 3 / 3 / chol / 1e12, "cores": host_cores(),
            "sample": s.describe() + f"; median over {samples} sub-evaluation(s); "
                      f"{sum(walls):.1f} s of sampling", "walls": walls}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on the host cores."""
    X, _, _ = load_c4()
    if rank != 0:
        return
    from oracle.cpu_baseline import SubEvalSampler, host_cores
    s = SubEvalSampler(X, THETA, blocks=REF_SUB_BLOCKS)
    per_step, per_step_chol = [], []
    for _ in range(args.warmup):
        s.sample()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        # one step = one sub-evaluation (~20-30 s of host work), extrapolated
        # to the full evaluation by exact operation counts
        t, _ = s.sample()
        a, c = s.extrapolate(t)
        per_step.append(a)
        per_step_chol.append(c)
    wall = time.perf_counter() - t0
    total, chol = statistics.median(per_step), statistics.median(per_step_chol)
    value = 1.0 / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": None,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config 4 recipe)",
        "config": {"workload": "C4: n=67,275 exponential GP log-likelihood (reference "
                               "P=1 block sweep, block 990)", "n": 67275},
        "cholesky_tflops": 67275 ** 3 / 3 / chol / 1e12,
        "extrapolated_eval_s": total,
        "per_step_eval_s": per_step,
        "measured_full_eval": full_eval_record(),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": host_cores(),
                         "kind": "port", "sample": s.describe() +
                         "; each step = one sub-evaluation, line value = median over steps",
                         "extrapolated_eval_s": total, "measured_full_eval": full_eval_record()},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, world, rank):
    import ctypes

    import torch

    from paper_1305_4886_b200 import spawn
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec

    X, y, sc = load_c4()
    n = len(y)
    local = 0 if args.debug_share_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    cl = spawn(world, tile=args.tile, device=local)
    dev = cl.device
    spec = builtin_spec("matern-nugget", X, nu=0.5)
    prob = KrigeProblem(cl, "c4", spec, y, THETA)

    def theta_k(k):
        return np.array([THETA[0], THETA[1] + k * 1e-12, THETA[2]])

    # warm-up (untimed); the first evaluation at the exact theta is the parity check
    step = 0
    ll0 = prob.log_density(THETA)
    ref_ll = sc["survey"]["ll"]
    parity = {"ll": ll0, "ref_ll": ref_ll, "rel_err": abs(ll0 - ref_ll) / abs(ref_ll),
              "tol": 1e-10}
    for _ in range(max(0, args.warmup - 1)):
        step += 1
        prob.log_density(theta_k(step))

    lib, ctx = cl.lib, cl._ctx
    lib.bgp_set_profiling(ctx, 1)
    prof = (ctypes.c_double * 10)()  # BGP_PROFILE_SLOTS
    lib.bgp_profile_read(ctx, prof)  # clear
    clocks = ClockSampler(dev.index)
    launches0 = cl.launches()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(dev)
    clocks.start()
    e0.record(stream)
    for _ in range(args.steps):
        step += 1
        prob.log_density(theta_k(step))
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier(world)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = cl.launches() - launches0
    lib.bgp_profile_read(ctx, prof)
    lib.bgp_set_profiling(ctx, 0)
    ms_max = max_over_ranks(ms, world)
    value = args.steps / (ms_max / 1e3)

    potrf_ms, trsm_ms, gemm_ms = prof[0], prof[1], prof[2]
    gemm_launches, gemm_flops, facts = prof[3], prof[4], max(prof[7], 1)
    chol_ms = prof[8] / facts  # first to last launch of each factorization (POTRF overlaps)
    if prof[7] == 0:  # sharded path: host-synchronised time of the last factorization
        chol_ms = max_over_ranks(cl.last_cholesky_ms or 0.0, world)
    # the update launches carry the whole factorization (the look-ahead POTRF,
    # inverse and panel TRSM run inside them), so the algorithmic work of
    # their summed event time is the unpadded n^3/3; the
    # padded-tile flops they execute are reported beside it
    executed_flops = gemm_flops / facts
    gemm_flops = n ** 3 / 3 * facts
    gemm_tflops = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    peak = FP64_DMMA_PEAK
    roof_kernel = "gemm_dmma_kernel (trailing SYRK/GEMM with the in-launch POTRF/TRSM)"
    if world > 1:  # aggregate: the whole factorization against N x the per-GPU peak
        gemm_tflops = n ** 3 / 3 / (chol_ms / 1e3) / 1e12 if chol_ms else 0.0
        gemm_flops, facts = n ** 3 / 3, 1
        peak = FP64_DMMA_PEAK * world
        roof_kernel = f"distributed Cholesky, aggregate over {world} GPUs (n^3/3 per factorization)"
    phases = {"cholesky_ms_per_eval": chol_ms, "potrf_ms_per_eval": potrf_ms / facts,
              "potrf_exposed_ms_per_eval": prof[9] / facts,
              "trsm_ms_per_eval": trsm_ms / facts, "gemm_ms_per_eval": gemm_ms / facts,
              "eval_ms": ms / args.steps,
              "other_ms_per_eval": ms / args.steps - chol_ms,
              "gemm_share_of_step": (gemm_ms / facts) / (ms / args.steps)}

    # G > 1: one more (untimed) evaluation with CUDA-event spans around the
    # panel broadcasts and the trailing updates -> exposed communication
    comm = None
    if world > 1:
        cl.comm_timeline = True
        step += 1
        prob.log_density(theta_k(step))
        cl.comm_timeline = False
        c = cl.last_comm or {}
        comm = {"comm_ms": max_over_ranks(c.get("comm_ms", 0.0), world),
                "exposed_comm_ms": max_over_ranks(c.get("exposed_comm_ms", 0.0), world),
                "collectives_per_rank": c.get("collectives", 0),
                "rank0_step_launch_ms": c.get("step_launch_ms"),
                "rank0_comm_span_ms": c.get("comm_span_ms"),
                "panel_exchange": ("fused TRSM + NVLink peer stores (bgp_panel_trsm_push)"
                                   if cl.__dict__.get("_panel_xchg", {}).get("x") is not None
                                   and cl._panel_xchg["x"].ok else "NCCL broadcasts"),
                "how": "CUDA events around each step barrier (push exchange) or panel broadcast "
                       "(fallback) and each step launch of one untimed evaluation (one stream: every "
                       "barrier wait is exposed, including waiting for the slowest rank); "
                       "max over ranks"}

    # end to end through the public API from host buffers (pinned), every step
    # uploads coords + y and reads back the scalars
    Xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory().numpy()
    yh = torch.from_numpy(np.ascontiguousarray(y)).pin_memory().numpy()
    e2e_steps = max(1, args.e2e_steps if args.e2e_steps is not None else args.steps)
    barrier(world)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        step += 1
        p = KrigeProblem(cl, f"e2e{k % 2}", builtin_spec("matern-nugget", Xh, nu=0.5), yh,
                         theta_k(step))
        p.log_density()
        for suffix in ("C", "L", "u", "mu", "resid", "y"):
            cl.remote_rm(f"e2e{k % 2}.{suffix}")
    torch.cuda.synchronize(dev)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    barrier(world)
    e2e = {"value": e2e_steps / e2e_s, "unit": "evals/s",
           "h2d_bytes_per_step": int(Xh.nbytes + yh.nbytes),
           "d2h_bytes_per_step": 5 * 8, "steps": e2e_steps,
           "path": "KrigeProblem(cluster, spec(host coords), host y, theta).log_density()"}

    traffic, traffic_src = gemm_traffic()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(args.cpu_samples, X)
        cpu = {"value": r["evals_per_s"], "unit": "evals/s", "cores": r["cores"],
               "kind": "port", "sample": r["sample"],
               "cholesky_tflops": r["chol_tflops"], "extrapolated_eval_s": r["eval_s"],
               "extrapolated_eval_s_range": r["eval_s_range"],
               "measured_full_eval": full_eval_record()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else None,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config 4 recipe, frozen inputs)",
            "config": {"workload": "C4: n=67,275 exponential GP log-likelihood "
                                   "(build + Cholesky + forward solve + logdet + ssq)",
                       "n": n, "tile": args.tile, "theta": THETA.tolist(),
                       "parallelism": (f"2-D block-cyclic tiles over {world} GPUs "
                                       f"(grid {cl.grid.shape[0]}x{cl.grid.shape[1]}), panel exchange: "
                                       f"{(comm or {}).get('panel_exchange', 'n/a')}")
                                      if world > 1 else "single GPU",
                       "l2": "no flush needed: each step rebuilds and streams the 18.1 GB "
                             "covariance (>> 126 MB L2)"},
            "cholesky_tflops": n ** 3 / 3 / (chol_ms / 1e3) / 1e12 if chol_ms else None,
            "phases": phases,
            "roofline": {"bound": "tensor", "kernel": roof_kernel,
                         "achieved": gemm_tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": gemm_tflops / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": "measured DMMA.8x8x4 loop (profiles/r01_fp64_peaks.jsonl); "
                                        "MEASURED_PEAKS.json has no FP64 figure",
                         "algorithmic_flops_per_eval": gemm_flops / facts,
                         "executed_flops_per_eval": executed_flops if world == 1 else None,
                         "launches_per_eval": gemm_launches / facts,
                         "cublas_dgemm_tflops": CUBLAS_DGEMM,
                         "hbm_kernels": hbm_kernels()},
            "parity": parity,
            "clocks": clk,
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if comm is not None:
            line["communication"] = comm
        print(json.dumps(line), flush=True)
    cl.shutdown()


C5_LOGDET_1GPU = -287708.10703490116  # profiles/r01l_configs_tile{256,512}.jsonl (same at both tiles)


def run_b200_c5(args, world, rank):
    """--workload c5 (opt-in): BASELINE config 5, one squared-exponential +
    nugget factorization of n = 131,072 per step (68.7 GB packed), spread
    over the job's GPUs; value = aggregate Cholesky TFLOP/s (strong scaling),
    with the exposed exchange time at N > 1.  The CPU reference cannot hold
    this matrix (68.7 GB > host RAM), so parity is the log-determinant
    against this library's own 1-GPU result."""
    import torch

    from paper_1305_4886_b200 import distla, spawn
    from paper_1305_4886_b200.gp import CovarianceSpec

    n = 131072
    X = np.random.default_rng(0).uniform(0, 1, (n, 2))  # SURVEY.md 8d C5 recipe
    theta = np.array([1.0, 0.02, 0.1])
    local = 0 if args.debug_share_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    cl = spawn(world, tile=args.tile, device=local)
    dev = cl.device
    spec = CovarianceSpec(cov_fn="gen.sqexp-nugget.cov", cross_cov_fn="gen.sqexp-nugget.cross",
                          pred_cov_fn="gen.sqexp-nugget.pred", inputs={"coords": X}, n_params=3)
    lay = distla.make_layout(n, cl.grid)
    cl.push("c5.inputs", {"coords": X})

    def step():
        distla.construct_distributed(cl, "c5.C", "triangular", spec.cov_fn, theta,
                                     inputs_name="c5.inputs", row_layout=lay)
        L, _ = distla.distributed_cholesky(cl, distla.DistTriangular("c5.C", lay), "c5.L")
        return L

    for _ in range(args.warmup):
        step()
        cl.remote_rm("c5.L")
    clocks = ClockSampler(dev.index)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = cl.launches()
    barrier(world)
    torch.cuda.synchronize(dev)
    clocks.start()
    e0.record(stream)
    for k in range(args.steps):
        L = step()
        if k + 1 < args.steps:
            cl.remote_rm("c5.L")
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier(world)
    clk = clocks.stop()
    ms_max = max_over_ranks(e0.elapsed_time(e1), world)
    launches = cl.launches() - launches0
    ld = distla.log_det_from_chol(cl, L)
    cl.remote_rm("c5.L")
    tflops = args.steps * n ** 3 / 3 / (ms_max / 1e3) / 1e12
    # independent check: the same kernel and recipe at n = 16,384 against the
    # REFERENCE's logdet (tests/golden/full_configs.json, make_full_configs.py)
    with open(os.path.join(ROOT, "tests", "golden", "full_configs.json")) as f:
        ref_small = json.load(f)["c5s"]
    ns = ref_small["n"]
    Xs = np.random.default_rng(0).uniform(0, 1, (ns, 2))  # the C5 recipe's first ns points
    lays = distla.make_layout(ns, cl.grid)
    cl.push("c5s.inputs", {"coords": Xs})
    distla.construct_distributed(cl, "c5s.C", "triangular", spec.cov_fn, theta,
                                 inputs_name="c5s.inputs", row_layout=lays)
    Ls, _ = distla.distributed_cholesky(cl, distla.DistTriangular("c5s.C", lays), "c5s.L")
    ld_small = distla.log_det_from_chol(cl, Ls)
    cl.remote_rm("c5s.L")
    comm = None
    if world > 1:
        cl.comm_timeline = True
        step()
        cl.comm_timeline = False
        c = cl.last_comm or {}
        comm = {"comm_ms": max_over_ranks(c.get("comm_ms", 0.0), world),
                "exposed_comm_ms": max_over_ranks(c.get("exposed_comm_ms", 0.0), world)}
        cl.remote_rm("c5.L")
    # end to end: host coords pushed, covariance built, factored, logdet read back
    barrier(world)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    cl.push("c5.inputs", {"coords": X})
    Le = step()
    distla.log_det_from_chol(cl, Le)
    torch.cuda.synchronize(dev)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    cl.remote_rm("c5.L")
    if rank == 0:
        line = {
            "metric": "C5 Cholesky FP64 TFLOP/s at n=131,072 (sqexp + nugget)", "value": tflops,
            "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else None, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config 5 recipe, seed 0)",
            "config": {"workload": "C5: n=131,072 squared-exponential (length 0.02) + nugget 0.1, "
                                   "covariance build + Cholesky per step",
                       "n": n, "tile": args.tile,
                       "parallelism": (f"2-D block-cyclic tiles over {world} GPUs "
                                       f"(grid {cl.grid.shape[0]}x{cl.grid.shape[1]})")
                                      if world > 1 else "single GPU",
                       "l2": "no flush needed: 68.7 GB matrix per step"},
            "roofline": {"bound": "tensor", "kernel": "whole factorization (n^3/3 per step)",
                         "achieved": tflops, "peak": FP64_DMMA_PEAK * world, "unit": "TFLOP/s",
                         "frac": tflops / (FP64_DMMA_PEAK * world), "traffic": None},
            "parity": {"logdet": ld, "ref_logdet_1gpu": C5_LOGDET_1GPU,
                       "rel_err": abs(ld - C5_LOGDET_1GPU) / abs(C5_LOGDET_1GPU), "tol": 1e-10,
                       "reference_n16384": {"logdet": ld_small, "ref_logdet": ref_small["logdet"],
                                            "rel_err": abs(ld_small - ref_small["logdet"])
                                            / abs(ref_small["logdet"]), "tol": 1e-12},
                       "note": "the CPU reference cannot hold C5; reference = this library on 1 GPU"},
            "clocks": clk, "gpu_launches": launches,
            "e2e": {"value": n ** 3 / 3 / e2e_s / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": int(X.nbytes), "d2h_bytes_per_step": 8 * world},
            "cpu_baseline": None,
        }
        if comm is not None:
            line["communication"] = comm
        print(json.dumps(line), flush=True)
    cl.shutdown()


def launch_ranks(args):
    """--gpus N without a launcher: start N ranks (one process per GPU) under
    torch.distributed.run and exit with their status; rank 0 prints the line."""
    import socket

    import torch
    ndev = torch.cuda.device_count()
    if args.gpus > ndev and not args.debug_share_gpu:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {ndev} GPU(s) are visible; "
                 "refusing to time fewer GPUs than requested")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--tile", type=int, default=None,
                    help="device tile size (default: 512 on one GPU; 256 on several, where the "
                         "one-CTA POTRF + inverse chain of each step -- 4x shorter at 256 -- is "
                         "exposed once a rank's share of the step's update gets small)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-samples", type=int, default=1)  # sub-evaluations (~20-30 s of host work)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c4", choices=["c4", "c5"],
                    help="c4: the BASELINE metric (default); c5: config 5 Cholesky scaling")
    ap.add_argument("--debug-share-gpu", action="store_true",
                    help="test only: every rank on cuda:0 over gloo, to exercise the N > 1 path "
                         "on a one-GPU box (the numbers mean nothing)")
    args = ap.parse_args()
    env_world = int(os.environ.get("WORLD_SIZE", "1"))
    if env_world > 1 and env_world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
    if env_world == 1 and args.gpus > 1 and args.impl == "b200":
        launch_ranks(args)  # does not return
    world, rank = dist_setup(args.impl, args.debug_share_gpu)
    if args.tile is None:
        args.tile = 512 if world == 1 else 256
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.workload == "c5":
        run_b200_c5(args, world, rank)
    else:
        run_b200(args, world, rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

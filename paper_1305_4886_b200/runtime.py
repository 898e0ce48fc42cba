"""The b200 runtime: the `Cluster` contract on one GPU per process.

Replaces the reference's worker runtime (bg/transport/base.py:126-276 with
the in-process / socket backends) by a device object store driven from the
calling process.  `run(op_id, **kwargs)` keeps the reference contract
(bg/transport/base.py:229-234): it looks the op up in the registry, runs it
on this process's GPU and returns the per-rank results as a list.  Errors
keep the reference's selection rules (base.py:213-227): package errors pass
through, anything else becomes WorkerFailure(rank, cause) with
rank = GPU index + 1.

Everything numeric is a libbgp call on the current torch CUDA stream;
PyTorch only allocates device buffers.
"""

import ctypes
import os
import time

import numpy as np

from . import _lib, registry
from .errors import (BackendUnavailable, BlockGPError, ClusterDown, NoSuchObject,
                     WorkerFailure)
from .grid import DeviceGrid

RUNTIME_OBJECT = ".runtime"
DEFAULT_TILE = 256


def _torch():
    import torch
    return torch


class B200Cluster:
    """Master-side handle of the GPU backend (single process, one GPU)."""

    backend = "b200"

    def __init__(self, G=1, seed=0, tile=DEFAULT_TILE, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise BackendUnavailable("backend 'b200' needs a CUDA device (no CPU fallback)")
        if tile % 128 or not 128 <= tile <= 512:
            raise BackendUnavailable(f"tile must be 128, 256, 384 or 512, got {tile}")
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0")) if G > 1 else torch.cuda.current_device()
        self.lib = _lib.load()
        self.device_index = int(device)
        self.device = torch.device("cuda", self.device_index)
        torch.cuda.set_device(self.device)
        self._ctx = ctypes.c_void_p()
        rc = self.lib.bgp_init(self.device_index, ctypes.byref(self._ctx))
        if rc != 0:
            raise BackendUnavailable(f"bgp_init failed on device {self.device_index}")
        self.grid = DeviceGrid(G)
        self.rank = 1
        self.comm = None
        if G > 1:
            # one process per GPU: triangular objects are spread 2-D
            # block-cyclically and the panel broadcasts run over NCCL
            import torch.distributed as tdist
            if not tdist.is_initialized():
                tdist.init_process_group("nccl", device_id=self.device)
            if tdist.get_world_size() != G:
                raise BackendUnavailable(f"process group has {tdist.get_world_size()} ranks, P={G}")
            from .parallel import TorchComm
            self.rank = tdist.get_rank() + 1
            self.comm = TorchComm()
        self.seed = seed
        self.tile = int(tile)
        self.state = "running"
        self.epoch = 0
        self.stats = {"collectives": 0}
        self.store = {RUNTIME_OBJECT: {"rank": self.rank, "device": self.device_index,
                                       "G": G, "tile": self.tile, "seed": seed}}
        self._dev_inputs = {}
        self.last_cholesky_ms = None
        self.comm_timeline = False  # G > 1: record comm / compute spans of the factorization
        self.last_comm = None       # their summary (parallel.Timeline.summary)
        self.stream_pos = 0  # draws consumed from this rank's normal stream
        self.events = []
        self.events_enabled = False

    # -- reference-compatible attributes --------------------------------------
    @property
    def P(self):
        return self.grid.P

    @property
    def G(self):
        return self.grid.G

    @property
    def coord(self):
        return self.grid.rank_to_coord(self.rank)

    # -- device helpers used by the ops ----------------------------------------
    @property
    def stream(self):
        return _torch().cuda.current_stream(self.device).cuda_stream

    @property
    def num_sms(self):
        return _torch().cuda.get_device_properties(self.device).multi_processor_count

    def call(self, name, *args):
        """Invoke a libbgp entry point; non-zero status -> WorkerFailure."""
        rc = getattr(self.lib, name)(self._ctx, *args)
        if rc != 0:
            msg = self.lib.bgp_last_error(self._ctx).decode(errors="replace")
            raise WorkerFailure(self.rank, RuntimeError(f"{name} returned {rc}: {msg}"))
        return rc

    def empty(self, shape):
        return _torch().empty(shape, dtype=_torch().float64, device=self.device)

    def zeros(self, shape):
        return _torch().zeros(shape, dtype=_torch().float64, device=self.device)

    def upload(self, array):
        """Host array -> contiguous FP64 device tensor (pinned staging)."""
        torch = _torch()
        a = np.ascontiguousarray(np.asarray(array, dtype=np.float64))
        host = torch.from_numpy(a)
        if a.size * 8 >= (1 << 16):
            host = host.pin_memory()
        return host.to(self.device, non_blocking=True)

    def upload_int32(self, array):
        torch = _torch()
        a = np.ascontiguousarray(np.asarray(array, dtype=np.int32).ravel())
        return torch.from_numpy(a).to(self.device)

    def device_input(self, inputs_name, key):
        """Device copy of a pushed coordinate array, (n, dim) row-major."""
        inputs = self.fetch(inputs_name)
        arr = inputs[key]
        cache_key = (inputs_name, key)
        hit = self._dev_inputs.get(cache_key)
        if hit is not None and hit[0] is arr:
            return hit[1]
        pts = np.asarray(arr, dtype=np.float64)
        if pts.ndim == 1:
            pts = pts[:, None]
        dev = self.upload(pts)
        self._dev_inputs[cache_key] = (arr, dev)
        return dev

    def input_span(self, inputs_name, keys):
        """Upper bound on the distance between any two points of the pushed
        coordinate arrays `keys` (their joint bounding-box diagonal), cached
        with the arrays; lets the covariance kernel drop its underflow test."""
        inputs = self.fetch(inputs_name)
        arrs = tuple(inputs[k] for k in keys)
        cache = self.__dict__.setdefault("_spans", {})
        hit = cache.get((inputs_name, keys))
        if hit is not None and all(a is b for a, b in zip(hit[0], arrs)):
            return hit[1]
        pts = [np.asarray(a, dtype=np.float64).reshape(len(a), -1) for a in arrs]
        lo = np.min([p.min(axis=0) for p in pts], axis=0)
        hi = np.max([p.max(axis=0) for p in pts], axis=0)
        span = float(np.sqrt(np.sum((hi - lo) ** 2))) * (1.0 + 1e-12)
        cache[(inputs_name, keys)] = (arrs, span)
        return span

    def launches(self):
        total = int(self.lib.bgp_launch_count(self._ctx))
        for c, _ in self.__dict__.get("_lanes", []):
            total += int(self.lib.bgp_launch_count(c))
        return total

    def lanes(self, k):
        """k (library context, CUDA stream) pairs for pipelined work: each
        lane has its own scratch, status and counters, so factorizations on
        different lanes can be in flight at once (distla.loglik_many)."""
        torch = _torch()
        lanes = self.__dict__.setdefault("_lanes", [])
        while len(lanes) < k:
            c = ctypes.c_void_p()
            if self.lib.bgp_init(self.device_index, ctypes.byref(c)) != 0:
                raise WorkerFailure(self.rank, RuntimeError("bgp_init failed for a lane"))
            lanes.append((c, torch.cuda.Stream(device=self.device)))
        return lanes[:k]

    def call_on(self, ctx, name, *args):
        """A libbgp entry point on another context of this device (a lane)."""
        rc = getattr(self.lib, name)(ctx, *args)
        if rc != 0:
            msg = self.lib.bgp_last_error(ctx).decode(errors="replace")
            raise WorkerFailure(self.rank, RuntimeError(f"{name} returned {rc}: {msg}"))
        return rc

    def fetch(self, name):
        try:
            return self.store[name]
        except KeyError:
            raise NoSuchObject(name, self.rank) from None

    def log_event(self, op, I=0, J=0):
        if self.events_enabled:
            self.events.append((time.monotonic_ns(), self.rank, op, I, J))

    # -- Cluster contract (bg/transport/base.py:229-276) -----------------------
    def _check_up(self):
        if self.state != "running":
            raise ClusterDown("cluster has been shut down")

    def run_local(self, fn_id, **kwargs):
        """Run a registered operation on this rank; returns its own result."""
        self._check_up()
        self.epoch += 1
        self.stats["collectives"] += 1
        fn = registry.lookup(fn_id)
        try:
            return fn(self, **kwargs)
        except BlockGPError:
            raise
        except Exception as exc:  # device / driver failures carry rank attribution
            raise WorkerFailure(self.rank, exc) from exc

    def run(self, fn_id, **kwargs):
        """Run a registered operation; returns the per-rank results in rank
        order, one per GPU (bg/transport/base.py:229-234).  With G > 1 (one
        process per GPU) every rank runs the op and the results of the ops
        that return per-rank values (stats, partial sums) are all-gathered,
        so every process sees the same P-length list."""
        result = self.run_local(fn_id, **kwargs)
        if self.G == 1:
            return [result]
        return per_rank_results(self.comm, fn_id, result, self.G)

    def push(self, name, value, targets=None):
        self._check_up()
        self.store[name] = _copy_value(value)
        self._dev_inputs = {k: v for k, v in self._dev_inputs.items() if k[0] != name}

    def scatter(self, name, per_rank_values):
        self._check_up()
        if self.rank in per_rank_values:
            self.push(name, per_rank_values[self.rank])

    def pull(self, name, source=1):
        self._check_up()
        value = self.fetch(name)
        from .distla.objects import DevObj
        if isinstance(value, DevObj):
            from .distla import ops
            return ops.dense_of(self, value)
        return _copy_value(value)

    def remote_ls(self, rank=1):
        self._check_up()
        return sorted(self.store)

    def remote_rm(self, name, targets=None):
        self._check_up()
        self.store.pop(name, None)

    def remote_apply(self, fn_id, input_names, output_name):
        if isinstance(input_names, str):
            input_names = [input_names]
        self.run("core.apply", op_id=fn_id, input_names=list(input_names),
                 output_name=output_name)

    def set_events(self, enabled):
        self._check_up()
        self.events_enabled = bool(enabled)

    def drain_events(self):
        self._check_up()
        out, self.events = sorted(self.events), []
        return out

    def collect_dense(self, name, diagonal=False):
        """Unpadded host copy of a device object (distla.collect /
        collect_diagonal); collective when the object is distributed."""
        self._check_up()
        from .distla import ops
        from .distla.objects import DevObj
        from .errors import DimensionMismatch
        obj = self.fetch(name)
        if not isinstance(obj, DevObj):
            raise DimensionMismatch(f"{name!r} is not a distributed object")
        return ops.diagonal_of(self, obj) if diagonal else ops.dense_of(self, obj)

    def synchronize(self):
        _torch().cuda.synchronize(self.device)

    def shutdown(self):
        if self.state == "running":
            self.state = "shutting-down"
            self.store.clear()
            self._dev_inputs.clear()
            try:
                x = self.__dict__.get("_panel_xchg", {}).get("x")
                if x is not None:  # peer panel mappings (collective)
                    x.close()
                _torch().cuda.synchronize(self.device)
            finally:
                for c, _ in self.__dict__.pop("_lanes", []):
                    self.lib.bgp_finalize(c)
                self.lib.bgp_finalize(self._ctx)
                self._ctx = ctypes.c_void_p()
                self.state = "shutdown"

    def __del__(self):
        try:
            self.shutdown()
        except Exception:
            pass


# ops whose per-rank results are gathered for run(); the others return None
# everywhere ("distla.collect": rank 1 returns the whole object, the other
# ranks nothing, so the reference's merge of per-rank pieces still works)
GATHERED_OPS = ("distla.cholesky", "distla.logdet", "distla.sumsq")


def per_rank_results(comm, fn_id, result, G):
    if fn_id in GATHERED_OPS:
        return comm.all_gather_object(result)
    if fn_id == "distla.collect":
        return [result] + [{} for _ in range(G - 1)]
    return [result] * G


def _copy_value(value):
    if isinstance(value, np.ndarray):
        return value.copy()
    if isinstance(value, dict):
        return {k: _copy_value(v) for k, v in value.items()}
    if isinstance(value, list):
        return [_copy_value(v) for v in value]
    return value

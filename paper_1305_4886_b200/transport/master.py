"""`spawn(P)` from a plain Python process: a master driving P GPU workers.

The reference's `spawn(P)` returns a master-side `Cluster` whose workers
(threads or socket subprocesses) run every operation SPMD and return their
per-rank results to the master (bg/transport/base.py:183-276, the command /
result protocol of inprocess.py:1-68 and socketbackend.py:1-120).  Here the
workers are one process per GPU: each runs the SPMD `B200Cluster` of its
device (runtime.py) inside one torch.distributed group -- NCCL when every
worker has its own GPU, gloo when several share one (a debugging setup in
which no kernel waits on another process) -- and the master forwards each
call over a pipe and assembles the P results in rank order.

Error selection follows bg/transport/base.py:213-227: the lowest rank's
error is raised; package errors pass through, anything else arrives as
WorkerFailure(rank, cause).  A worker that dies, or ranks that stop
answering after another rank failed, shut the cluster down.
"""

import os
import pickle
import socket
import time

from ..errors import BackendUnavailable, BlockGPError, ClusterDown, WorkerFailure
from ..grid import DeviceGrid

# a rank still silent this long after another rank reported an error is
# taken to be stuck in a collective the failed rank never joined
STRAGGLER_TIMEOUT_S = 60.0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _picklable(exc, rank):
    try:
        pickle.dumps(exc)
        return exc
    except Exception:
        return WorkerFailure(rank, RuntimeError(repr(exc)))


def _worker_main(rank, world, port, device, backend, seed, tile, conn):
    """Worker loop: one GPU, one SPMD B200Cluster, commands from the pipe."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(device))
    cl = None
    try:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(device)
        kw = {"device_id": torch.device("cuda", device)} if backend == "nccl" else {}
        dist.init_process_group(backend, rank=rank, world_size=world, **kw)
        from ..runtime import B200Cluster
        cl = B200Cluster(G=world, seed=seed, tile=tile, device=device)
        conn.send(("ok", None))
    except BaseException as exc:  # noqa: BLE001  (reported to the master)
        conn.send(("err", _picklable(BackendUnavailable(f"worker {rank + 1}: {exc!r}"), rank + 1)))
        return
    try:
        while True:
            method, args, kwargs = conn.recv()
            if method == "shutdown":
                cl.shutdown()
                conn.send(("ok", None))
                break
            try:
                conn.send(("ok", getattr(cl, method)(*args, **kwargs)))
            except BaseException as exc:  # noqa: BLE001
                conn.send(("err", _picklable(exc, rank + 1)))
    finally:
        try:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()
        except Exception:
            pass


class MasterCluster:
    """Master-side handle of P GPU workers (the reference's `Cluster`)."""

    backend = "b200"

    def __init__(self, G, seed=0, tile=None, devices=None):
        import torch
        import torch.multiprocessing as mp
        if not torch.cuda.is_available():
            raise BackendUnavailable("backend 'b200' needs a CUDA device (no CPU fallback)")
        from ..runtime import DEFAULT_TILE
        ndev = torch.cuda.device_count()
        devices = list(devices) if devices is not None else [r % ndev for r in range(G)]
        if len(devices) != G or any(not 0 <= d < ndev for d in devices):
            raise BackendUnavailable(f"need {G} device ids in [0, {ndev}), got {devices}")
        # NCCL needs one GPU per rank; ranks sharing a GPU talk over gloo
        self.comm_backend = "nccl" if len(set(devices)) == G else "gloo"
        self.grid = DeviceGrid(G)
        self.seed = seed
        self.tile = int(tile or DEFAULT_TILE)
        self.devices = devices
        self.stats = {"collectives": 0}
        self.state = "running"
        self.epoch = 0
        ctx = mp.get_context("spawn")
        port = _free_port()
        self._conns, self._procs = [], []
        for r in range(G):
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_worker_main, daemon=True,
                            args=(r, G, port, devices[r], self.comm_backend, seed, self.tile, child))
            p.start()
            child.close()
            self._conns.append(parent)
            self._procs.append(p)
        try:
            self._collect(range(G), timeout=600.0)
        except BaseException:
            self._kill()
            raise

    # -- reference-compatible attributes --------------------------------------
    @property
    def P(self):
        return self.grid.P

    @property
    def G(self):
        return self.grid.G

    # -- command protocol ------------------------------------------------------
    def _check_up(self):
        if self.state != "running":
            raise ClusterDown("cluster has been shut down")

    def _kill(self):
        self.state = "shutdown"
        for p in self._procs:
            if p.is_alive():
                p.kill()
        for p in self._procs:
            p.join(timeout=10)

    def _collect(self, ranks, timeout=None):
        """Replies of `ranks` (0-based) in rank order; raises the lowest
        rank's error (bg/transport/base.py:213-227)."""
        from multiprocessing.connection import wait
        pending = {r: self._conns[r] for r in ranks}
        replies, first_err_t = {}, None
        t0 = time.monotonic()
        while pending:
            sentinels = {self._procs[r].sentinel: r for r in pending}
            ready = wait(list(pending.values()) + list(sentinels), timeout=1.0)
            for obj in ready:
                if obj in sentinels:
                    r = sentinels[obj]
                    if r in pending and not pending[r].poll():
                        replies[r] = ("err", WorkerFailure(r + 1, RuntimeError(
                            f"worker process exited ({self._procs[r].exitcode})")))
                        pending.pop(r)
                    continue
                r = next(k for k, c in pending.items() if c is obj)
                try:
                    replies[r] = pending.pop(r).recv()
                except EOFError:
                    replies[r] = ("err", WorkerFailure(r + 1, RuntimeError("worker pipe closed")))
                if replies[r][0] == "err" and first_err_t is None:
                    first_err_t = time.monotonic()
            now = time.monotonic()
            if pending and ((first_err_t is not None and now - first_err_t > STRAGGLER_TIMEOUT_S)
                            or (timeout is not None and now - t0 > timeout)):
                for r in pending:
                    replies[r] = ("err", WorkerFailure(r + 1, RuntimeError("no reply (stuck collective)")))
                self._kill()
                pending = {}
        errs = sorted((r, v) for r, (tag, v) in replies.items() if tag == "err")
        if errs:
            if any(not p.is_alive() for p in self._procs) and self.state == "running":
                self._kill()
            r, exc = errs[0]
            if isinstance(exc, BlockGPError):
                raise exc
            raise WorkerFailure(r + 1, exc)
        return [replies[r][1] for r in sorted(replies)]

    def _all(self, method, *args, **kwargs):
        self._check_up()
        for c in self._conns:
            c.send((method, args, kwargs))
        return self._collect(range(self.G))

    # -- Cluster contract (bg/transport/base.py:229-276) -----------------------
    def run(self, fn_id, **kwargs):
        """Run a registered operation on every GPU; per-rank results in rank
        order (the collectives and the result gather run in the workers)."""
        self.epoch += 1
        self.stats["collectives"] += 1
        return self._all("run", fn_id, **kwargs)[0]

    def push(self, name, value, targets=None):
        self._all("push", name, value)

    def scatter(self, name, per_rank_values):
        self._check_up()
        for r, c in enumerate(self._conns):
            c.send(("scatter", (name, {r + 1: per_rank_values[r + 1]} if r + 1 in per_rank_values else {}), {}))
        self._collect(range(self.G))

    def pull(self, name, source=1):
        return self._all("pull", name)[source - 1]

    def remote_ls(self, rank=1):
        return self._all("remote_ls")[rank - 1]

    def remote_rm(self, name, targets=None):
        self._all("remote_rm", name)

    def remote_apply(self, fn_id, input_names, output_name):
        if isinstance(input_names, str):
            input_names = [input_names]
        self.run("core.apply", op_id=fn_id, input_names=list(input_names), output_name=output_name)

    def collect_dense(self, name, diagonal=False):
        return self._all("collect_dense", name, diagonal)[0]

    def set_events(self, enabled):
        self._all("set_events", enabled)

    def drain_events(self):
        return sorted(e for part in self._all("drain_events") for e in part)

    def launches(self):
        return sum(self._all("launches"))

    def synchronize(self):
        self._all("synchronize")

    def shutdown(self):
        if self.state != "running":
            return
        self.state = "shutting-down"
        try:
            for c in self._conns:
                c.send(("shutdown", (), {}))
            self._collect(range(self.G), timeout=120.0)
        except Exception:
            pass
        finally:
            for p in self._procs:
                p.join(timeout=30)
            self._kill()

    def __del__(self):
        try:
            self.shutdown()
        except Exception:
            pass

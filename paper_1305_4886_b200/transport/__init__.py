"""`spawn` for the b200 backend (drop-in for bg/transport/__init__.py:10-25).

The reference starts P = D(D+1)/2 CPU workers ("in-process" threads or
"multi-process-socket" subprocesses) behind a master-side Cluster.  Here the
workers are GPUs, one process per GPU:

  * P = 1: the calling process drives one GPU (runtime.B200Cluster);
  * P > 1 from a plain process: the caller is the master and P worker
    processes are started, one per GPU (transport.master.MasterCluster);
    `run` returns the P per-rank results, as in the reference;
  * P > 1 under torchrun (WORLD_SIZE = P): every process is a rank of the
    job (SPMD); `run` all-gathers the per-rank results, so each process sees
    the same P-length list.

There is no CPU backend and no fallback.
"""

import os

from ..errors import BackendUnavailable

BACKENDS = ("b200",)


def spawn(P=1, backend="b200", seed=0, blas_threads=None, tile=None, device=None, devices=None):
    """Start the GPU runtime and return its Cluster handle.

    `tile` is the device tile size b (128, 256, 384 or 512; default 256).
    `devices` (master mode) lists the GPU of each worker (default: rank mod
    the visible GPU count; workers sharing a GPU use gloo instead of NCCL).
    `blas_threads` is accepted for signature compatibility and ignored.
    """
    if backend != "b200":
        raise BackendUnavailable(f"unknown backend {backend!r}; this package provides "
                                 f"{BACKENDS} only (no CPU fallback)")
    if P < 1:
        raise BackendUnavailable(f"P must be >= 1, got {P}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    from ..runtime import DEFAULT_TILE, B200Cluster
    if P == 1 or (world == P and world > 1):
        return B200Cluster(G=P, seed=seed, tile=tile or DEFAULT_TILE, device=device)
    if world > 1:
        raise BackendUnavailable(
            f"P={P} GPUs requested inside a job of WORLD_SIZE={world}; use P=WORLD_SIZE "
            "(one process per GPU) or call spawn(P) from a plain process")
    from .master import MasterCluster
    return MasterCluster(P, seed=seed, tile=tile or DEFAULT_TILE, devices=devices)


__all__ = ["spawn", "BACKENDS"]

"""`spawn` for the b200 backend (drop-in for bg/transport/__init__.py:10-25).

The reference starts P = D(D+1)/2 CPU workers ("in-process" threads or
"multi-process-socket" subprocesses).  Here the workers are GPUs: P is the
GPU count G of this job (1 in a plain process; WORLD_SIZE under torchrun,
one process per GPU).  There is no CPU backend and no fallback.
"""

import os

from ..errors import BackendUnavailable

BACKENDS = ("b200",)


def spawn(P=1, backend="b200", seed=0, blas_threads=None, tile=None, device=None):
    """Start the GPU runtime and return its Cluster handle.

    `tile` is the device tile size b (128, 256, 384 or 512; default 256).
    `blas_threads` is accepted for signature compatibility and ignored.
    """
    if backend != "b200":
        raise BackendUnavailable(f"unknown backend {backend!r}; this package provides "
                                 f"{BACKENDS} only (no CPU fallback)")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if P != 1 and P != world:
        raise BackendUnavailable(
            f"P={P} GPUs requested but this job has WORLD_SIZE={world}; launch one "
            "process per GPU (torchrun --nproc-per-node P)")
    from ..runtime import DEFAULT_TILE, B200Cluster
    return B200Cluster(G=P, seed=seed, tile=tile or DEFAULT_TILE, device=device)


__all__ = ["spawn", "BACKENDS"]

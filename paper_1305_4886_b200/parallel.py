"""Multi-GPU likelihood path: 2-D block-cyclic lower tiles, one process per GPU.

Replaces the reference's triangular D(D+1)/2 process fold
(bg/grid.py:116-139) and its tag-matched point-to-point messages
(bg/distla/kernels.py:139-250) with the SURVEY.md 8e plan:

  * tiles (I, J), I >= J, live on rank (I mod Pr) + Pr*(J mod Pc) of a
    Pr x Pc grid (1x1, 1x2, 2x2, 2x4); a rank stores its tiles packed by
    tile column, so each owned part of a panel is contiguous;
  * construct: every rank generates only its own tiles (no communication);
  * Cholesky step J: the owner of (J, J) factors it and broadcasts L_JJ; the
    ranks of process column J mod Pc solve their panel tiles; every process
    row's panel chunk is broadcast to all ranks; each rank applies the
    DMMA trailing update to its own tiles (bgp_tile_update, tile-list mode);
  * forward / back solve: per block, the partial products of the owners of
    row (column) J are reduced to the diagonal owner, which solves and
    broadcasts x_J (2 x b doubles of traffic per step);
  * logdet: per-rank partials gathered and summed in rank order, as the
    reference's master does (bg/distla/__init__.py:154-157).

The schedule below is written against two small interfaces so the same code
runs on the GPUs (`LibTileOps` over libbgp + NCCL) and in the CPU tests
(a numpy tile backend + gloo, world size 2).
"""

from dataclasses import dataclass, field

import numpy as np

from .grid import DeviceGrid


@dataclass
class TileDist:
    """Ownership map of the lower tiles of an n x n matrix for one rank."""

    n: int
    b: int
    grid: DeviceGrid
    rank: int  # 0-based
    T: int = field(init=False)
    tiles: np.ndarray = field(init=False)      # (k, 2) int32 (I, J), column-major
    local: dict = field(init=False)            # (I, J) -> local tile index
    col_start: np.ndarray = field(init=False)  # first local index of column J
    col_count: np.ndarray = field(init=False)

    def __post_init__(self):
        self.T = -(-self.n // self.b)
        T = self.T
        pr, pc = self.grid.shape
        r_row, r_col = self.rank % pr, self.rank // pr
        tl = [(I, J) for J in range(T) if J % pc == r_col
              for I in range(J, T) if I % pr == r_row]
        self.tiles = np.array(tl, dtype=np.int32).reshape(-1, 2)
        self.local = {(int(I), int(J)): k for k, (I, J) in enumerate(tl)}
        self.col_start = np.zeros(T + 1, dtype=np.int64)
        self.col_count = np.zeros(T, dtype=np.int64)
        for I, J in tl:
            self.col_count[J] += 1
        self.col_start[1:] = np.cumsum(self.col_count)

    @property
    def count(self):
        return len(self.tiles)

    def owner(self, I, J):
        return self.grid.owner(I, J)

    def panel_rows(self, J, pr_row):
        """Rows I > J of panel J held by process row pr_row (ascending)."""
        pr, _ = self.grid.shape
        start = J + 1 + ((pr_row - (J + 1)) % pr)
        return list(range(start, self.T, pr))

    def panel_layout(self, J):
        """Panel buffer layout for step J: per process row, (root rank,
        first panel slot, tile count); and slot of each panel row I."""
        pr, pc = self.grid.shape
        chunks, slot = [], np.full(self.T, -1, dtype=np.int64)
        off = 0
        for p in range(pr):
            rows = self.panel_rows(J, p)
            root = p + pr * (J % pc)
            chunks.append((root, off, len(rows)))
            for k, I in enumerate(rows):
                slot[I] = off + k
            off += len(rows)
        return chunks, slot, off

    def my_panel(self, J):
        """(first local index, count) of my tiles (I > J, J) in column J."""
        s = int(self.col_start[J])
        c = int(self.col_count[J])
        if c and self.tiles[s][0] == J:
            return s + 1, c - 1
        return s, c

    def update_items(self, J, slot):
        """(C local, A slot, B slot, lower) for my tiles (R, C), J < C <= R."""
        first = int(self.col_start[J + 1]) if J + 1 <= self.T - 1 else self.count
        t = self.tiles[first:]
        if len(t) == 0:
            return np.zeros((0, 4), dtype=np.int32)
        R, C = t[:, 0].astype(np.int64), t[:, 1].astype(np.int64)
        items = np.stack([np.arange(first, first + len(t)), slot[R], slot[C], (R == C)], axis=1)
        return items.astype(np.int32)

    def diag_items(self):
        """(local index, J) of my diagonal tiles."""
        d = [(k, int(I)) for k, (I, J) in enumerate(self.tiles) if I == J]
        return np.array(d, dtype=np.int32).reshape(-1, 2)

    def column_items(self, J, below=True):
        """(local index, I) of my tiles (I > J, J) -- forward-solve partials."""
        s, c = self.my_panel(J)
        I = self.tiles[s:s + c, 0]
        return np.stack([np.arange(s, s + c), I], axis=1).astype(np.int32)

    def row_items(self, J):
        """(local index, K) of my tiles (J, K), K < J -- back-solve partials."""
        sel = [(k, int(Jc)) for k, (I, Jc) in enumerate(self.tiles) if I == J and Jc < J]
        return np.array(sel, dtype=np.int32).reshape(-1, 2)


def dist_cholesky(dist, local, ops, comm):
    """Right-looking tiled Cholesky of a distributed matrix, in place, with a
    one-panel look-ahead.

    `local` is this rank's (count, b, b) tile stack.  Returns the first
    failing pivot row (1-based, LAPACK info) agreed by all ranks, or 0.

    Step J: every rank first updates its tiles of column J+1 with panel J.
    Then, on the side stream (ops.side()), the owner of (J+1, J+1) factors
    and inverts it, the inverse is broadcast, process column (J+1) mod Pc
    solves its panel tiles (A <- A Linv^T on the DMMA GEMM) and the panel
    reaches every rank -- stored by that same TRSM kernel into every rank's
    panel buffer over NVLink (PanelExchange), or, as the fallback, broadcast
    row chunk by row chunk over NCCL -- while the rest of the trailing update
    (columns >= J+2, panel J) runs on the compute stream on all SMs but a few
    (ops.update(..., reserve=True)), which the collectives and the small
    panel kernels use.  ops.join_side() then orders step J+1 after panel J+1.
    The update items of every step are built and uploaded once, and a failing
    pivot stays in the device status until the end, so the host never waits
    on the GPU inside the loop.
    """
    b, T, me = dist.b, dist.T, dist.rank
    inv_buf = ops.empty((b, b))
    ops.begin()
    info = [0]
    panels = [None, None]
    layouts = [dist.panel_layout(J) for J in range(T - 1)]
    col_items, rest_items = [], []
    for J in range(T - 1):
        it = np.asarray(dist.update_items(J, layouts[J][1])).reshape(-1, 4)
        cols = dist.tiles[it[:, 0], 1] if len(it) else np.zeros(0, dtype=np.int32)
        col_items.append(it[cols == J + 1])
        rest_items.append(it[cols != J + 1])
    dev_col = ops.prepare_items(col_items)
    dev_rest = ops.prepare_items(rest_items)
    # fused panel exchange (TRSM epilogue stores into every rank's panel
    # buffer over NVLink), or None: TRSM then NCCL broadcasts
    xchg = ops.panel_exchange(comm, T) if hasattr(ops, "panel_exchange") else None

    def factor_panel(K):
        d = dist.owner(K, K)
        if xchg is not None and K + 1 < T:
            # every rank is done with buffer K % 2 (its last reader, step K-2's
            # update, precedes this point on every rank's streams)
            comm.barrier_stream()
        if me == d:
            info[0] = info[0] or ops.potrf_factor(local, dist.local[(K, K)], K * b,
                                                  inv_buf if K + 1 < T else None)
        if K + 1 >= T:
            return
        comm.broadcast(inv_buf, d)
        s, c = dist.my_panel(K)
        chunks, _, ntot = layouts[K]
        if xchg is not None:
            if c:
                off = next(o for root, o, cnt in chunks if root == me and cnt)
                xchg.push(inv_buf, local, s, c, K % 2, off)
            comm.barrier_stream()  # panel K is in every rank's buffer
            panels[K % 2] = xchg.bufs[K % 2]
            return
        if c:
            ops.trsm_inv(inv_buf, local, s, c)
        if panels[K % 2] is None or panels[K % 2].shape[0] < ntot:
            panels[K % 2] = ops.empty((max(ntot, 1), b, b))
        panel = panels[K % 2]
        for root, off, cnt in chunks:
            if cnt == 0:
                continue
            view = panel[off:off + cnt]
            if me == root:
                ps, pcount = dist.my_panel(K)
                assert pcount == cnt
                ops.copy_tiles(view, local, ps, cnt)
            comm.broadcast(view, root)

    factor_panel(0)
    for J in range(T - 1):
        ops.update(local, panels[J % 2], dev_col[J])
        with ops.side():
            factor_panel(J + 1)
        ops.update(local, panels[J % 2], dev_rest[J], reserve=True)
        ops.join_side()
    return comm.min_nonzero(ops.end(info[0]))


def dist_trsv(dist, local, y, ops, comm, forward=True):
    """Solve L x = y (forward) or L^T x = y (back) with y replicated.

    Returns (x replicated on every rank, info)."""
    b, T, me = dist.b, dist.T, dist.rank
    acc = ops.zeros((T * b,))
    x = ops.zeros((T * b,))
    ops.begin()
    info = 0
    order = list(range(T)) if forward else list(range(T - 1, -1, -1))
    per_step = [dist.column_items(J) if forward else dist.row_items(J) for J in order]
    dev_items = ops.prepare_gemv_items(per_step)
    for J, items in zip(order, dev_items):
        d = dist.owner(J, J)
        blk = acc[J * b:(J + 1) * b]
        comm.reduce_sum(blk, d)
        xJ = x[J * b:(J + 1) * b]
        if me == d:
            ops.sub_into(xJ, y[J * b:(J + 1) * b], blk)
            info = info or ops.tile_trsv(local, dist.local[(J, J)], J * b, xJ, 0 if forward else 1)
        comm.broadcast(xJ, d)
        ops.gemv(local, items, xJ, acc, 0 if forward else 1)
    info = ops.end(info)
    return x, comm.min_nonzero(info)


def col_shards(T, world):
    """Contiguous split of T tile rows over `world` ranks: [(r0, r1)] per
    rank, the first T mod world ranks one row longer.  The kriging RHS
    columns (tile rows of the transposed rectangular object) are sharded
    this way: every column is solved independently."""
    base, extra = divmod(T, world)
    out, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def gather_col_shards(comm, part, shards, fill):
    """All-gather per-rank column shards into the full object.

    `part` is this rank's (lead, r1 - r0, ...) slice, padded by the caller
    to the widest shard along dim 1; `fill(r0, r1, piece)` stores rank r's
    piece (already cut to its width).  Every rank ends with the full object.
    """
    parts = comm.all_gather(part)
    for (r0, r1), piece in zip(shards, parts):
        if r1 > r0:
            fill(r0, r1, piece[:, :r1 - r0])


def dist_logdet(dist, local, ops, comm):
    """2 sum log diag(L): per-rank partials summed in rank order."""
    part, info = ops.logdet_partial(local, dist.diag_items())
    parts = comm.all_gather_float(part)
    return float(sum(parts)), comm.min_nonzero(info)


def exposed_time(comm, compute):
    """Total length of the `comm` intervals not covered by the union of the
    `compute` intervals (lists of (start, end)): the communication time the
    schedule failed to hide (SURVEY.md 8d, C5 "exposed NVLink time")."""
    cover = []
    for a, b in sorted(compute):
        if cover and a <= cover[-1][1]:
            cover[-1][1] = max(cover[-1][1], b)
        else:
            cover.append([a, b])
    total = 0.0
    for a, b in comm:
        hidden = sum(max(0.0, min(b, y) - max(a, x)) for x, y in cover)
        total += (b - a) - hidden
    return total


class Timeline:
    """CUDA-event spans of a distributed factorization: "comm" around each
    collective (recorded on the stream that issues it) and "compute" around
    each trailing update.  summary() syncs and reports milliseconds."""

    def __init__(self, device):
        self.device = device
        self.spans = []
        self._origin = None

    def span(self, kind):
        import contextlib

        import torch

        @contextlib.contextmanager
        def rec():
            if self._origin is None:
                self._origin = torch.cuda.Event(enable_timing=True)
                self._origin.record(torch.cuda.current_stream(self.device))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(self.device))
            yield
            e1.record(torch.cuda.current_stream(self.device))
            self.spans.append((kind, e0, e1))
        return rec()

    def summary(self):
        import torch
        torch.cuda.synchronize(self.device)
        iv = {"comm": [], "compute": []}
        for kind, e0, e1 in self.spans:
            iv[kind].append((self._origin.elapsed_time(e0), self._origin.elapsed_time(e1)))
        comm = sum(b - a for a, b in iv["comm"])
        return {"comm_ms": comm, "collectives": len(iv["comm"]),
                "exposed_comm_ms": exposed_time(iv["comm"], iv["compute"])}


class TorchComm:
    """Collectives over a torch.distributed process group (NCCL on GPUs,
    gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.timeline = None  # Timeline: spans around the panel broadcasts

    def broadcast(self, tensor, src):
        if self.world > 1:
            if self.timeline is not None:
                with self.timeline.span("comm"):
                    self.dist.broadcast(tensor, src, group=self.group)
            else:
                self.dist.broadcast(tensor, src, group=self.group)

    def reduce_sum(self, tensor, dst):
        # all-reduce (not reduce): 2 KB per step, and it is supported by every
        # backend for CUDA tensors; only `dst` uses the result
        if self.world > 1:
            self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)

    def all_reduce_sum(self, tensor):
        if self.world > 1:
            self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)

    def all_gather(self, tensor):
        """Equal-shaped tensors of every rank, in rank order.  NCCL gathers
        into one buffer; gloo (the CPU tests, and ranks sharing one GPU)
        stages device tensors through host memory."""
        if self.world == 1:
            return [tensor]
        import torch
        t = tensor.contiguous()
        if t.is_cuda and self.dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return list(out.unbind(0))
        host = t.cpu()
        outs = [torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(outs, host, group=self.group)
        return [o.to(t.device) for o in outs]

    def barrier_stream(self):
        """A barrier ordered on the current stream (a 1-element all-reduce):
        later work on this stream runs after every rank's earlier work."""
        if self.world > 1:
            import torch
            nccl = self.dist.get_backend(self.group) == "nccl"
            if getattr(self, "_one", None) is None:
                dev = torch.cuda.current_device() if nccl else "cpu"
                self._one = torch.ones(1, dtype=torch.int32, device=dev)
            if not nccl and torch.cuda.is_available():
                # host-side collective: finish this rank's queued GPU work first
                torch.cuda.current_stream().synchronize()
            op = self.dist.ReduceOp.MAX  # the value stays 1
            if self.timeline is not None:
                with self.timeline.span("comm"):
                    self.dist.all_reduce(self._one, op=op, group=self.group)
            else:
                self.dist.all_reduce(self._one, op=op, group=self.group)

    def all_gather_bytes(self, value):
        if self.world == 1:
            return [value]
        out = [None] * self.world
        self.dist.all_gather_object(out, bytes(value), group=self.group)
        return out

    def all_gather_float(self, value):
        if self.world == 1:
            return [value]
        out = [None] * self.world
        self.dist.all_gather_object(out, float(value), group=self.group)
        return out

    def min_nonzero(self, info):
        if self.world == 1:
            return int(info)
        vals = [None] * self.world
        self.dist.all_gather_object(vals, int(info), group=self.group)
        nz = [v for v in vals if v]
        return min(nz) if nz else 0


class _DevMem:
    """Zero-copy torch view of a raw device allocation."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3}


class PanelExchange:
    """Two panel buffers per rank in IPC-exported device memory, opened by
    every peer: the panel TRSM stores each solved tile straight into all
    ranks' buffers (bgp_panel_trsm_push), so the solve and the panel
    exchange are one kernel over NVLink peer memory instead of a TRSM
    followed by NCCL broadcasts.  Built collectively; `ok` is False (and the
    schedule falls back to NCCL broadcasts) when the peer mappings or a
    one-tile self-check fail on any rank."""

    def __init__(self, cluster, comm, tiles):
        # Every rank runs the same sequence of collectives whatever fails
        # locally (a rank that stops early would leave the others waiting).
        import ctypes
        import warnings

        import torch
        self.cl, self.comm = cluster, comm
        b = cluster.tile
        self.tiles = max(tiles, comm.world)
        nbytes = self.tiles * b * b * 8
        me = comm_rank(comm)
        self.own, self.peers = [], []
        self.bufs, self.dst = [], []
        ok, why = True, None
        for _ in range(2):
            ptr, h = ctypes.c_void_p(), ctypes.create_string_buffer(64)
            if ok:
                try:
                    cluster.call("bgp_ipc_alloc", nbytes, ctypes.byref(ptr), h)
                    self.own.append(ptr.value)
                except Exception as exc:
                    ok, why = False, exc
            handles = comm.all_gather_bytes(h.raw if ok else b"")
            if ok and any(len(hr) != 64 for hr in handles):
                ok, why = False, "a peer could not export its buffer"
            if not ok:
                continue
            try:
                ptrs = []
                for r, hr in enumerate(handles):
                    if r == me:
                        ptrs.append(ptr.value)
                        continue
                    q = ctypes.c_void_p()
                    cluster.call("bgp_ipc_open", hr, ctypes.byref(q))
                    self.peers.append(q.value)
                    ptrs.append(q.value)
                self.dst.append((ctypes.c_void_p * len(ptrs))(*ptrs))
                self.bufs.append(torch.as_tensor(_DevMem(ptr.value, self.tiles * b * b),
                                                 device=cluster.device).view(self.tiles, b, b))
            except Exception as exc:
                ok, why = False, exc
        if not self._agree(ok):  # no P2P mapping somewhere: NCCL broadcasts
            if why is not None:
                warnings.warn(f"panel push unavailable ({why}); using NCCL panel broadcasts")
            self.ok = False
            return
        self.ok = self._agree(self._self_check())

    def _agree(self, ok):
        vals = self.comm.all_gather_bytes(b"\x01" if ok else b"\x00")
        return all(v == b"\x01" for v in vals)

    def _self_check(self):
        """Every rank pushes a tile (identity inverse: the tile itself) into
        slot `rank` of buffer 0 everywhere; each rank then checks its slots.
        The two barriers run on every rank even if the push raises."""
        import warnings

        import torch
        b, me, G = self.cl.tile, comm_rank(self.comm), self.comm.world
        err = None
        self.comm.barrier_stream()
        try:
            eye = torch.eye(b, dtype=torch.float64, device=self.cl.device)
            t = torch.full((1, b, b), float(me + 1), dtype=torch.float64, device=self.cl.device)
            self.push(eye, t, 0, 1, 0, me)
        except Exception as exc:
            err = exc
        self.comm.barrier_stream()
        if err is None:
            try:
                torch.cuda.synchronize(self.cl.device)
                got = self.bufs[0][:G, 0, 0].cpu().tolist()
                if got != [float(r + 1) for r in range(G)]:
                    err = f"received {got}"
            except Exception as exc:
                err = exc
        if err is not None:
            warnings.warn(f"panel push self-check failed ({err}); using NCCL panel broadcasts")
            return False
        return True

    def push(self, inv, local, start, count, which, slot0):
        import ctypes
        self.cl.call("bgp_panel_trsm_push", ctypes.c_void_p(inv.data_ptr()),
                     ctypes.c_void_p(local[start].data_ptr()), count, self.cl.tile,
                     self.dst[which], len(self.dst[which]), slot0, self.tiles, self.cl.stream)

    def close(self):
        for q in self.peers:
            self.cl.lib.bgp_ipc_close(self.cl._ctx, q)
        self.peers = []
        try:
            self.comm.barrier_stream()
            import torch
            torch.cuda.synchronize(self.cl.device)
        except Exception:
            pass
        for q in self.own:
            self.cl.lib.bgp_ipc_free(self.cl._ctx, q)
        self.own, self.bufs = [], []


def comm_rank(comm):
    return comm.dist.get_rank(comm.group) if comm.world > 1 else 0


class LibTileOps:
    """Tile operations of the distributed schedule on this rank's GPU (libbgp)."""

    def __init__(self, cluster, n, timeline=None):
        self.cl = cluster
        self.b = cluster.tile
        self.n = n
        self.timeline = timeline  # Timeline: spans around the trailing updates

    # buffers ---------------------------------------------------------------
    def empty(self, shape):
        return self.cl.empty(shape)

    def zeros(self, shape):
        return self.cl.zeros(shape)

    def _items(self, arr):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32).ravel())
        return t.to(self.cl.device, non_blocking=False)

    @staticmethod
    def _p(t):
        import ctypes
        return ctypes.c_void_p(t.data_ptr())

    # tile kernels ------------------------------------------------------------
    def begin(self):
        self.cl.call("bgp_info_reset", self.cl.stream)

    def end(self, info):
        import ctypes
        dev = ctypes.c_int64(0)
        self.cl.call("bgp_info_read", ctypes.byref(dev), self.cl.stream)
        return int(info or dev.value)

    def potrf_factor(self, local, k, row0, inv):
        """Factor tile k in place and (inv not None) write its inverse; the
        status stays on the device until end()."""
        self.cl.call("bgp_tile_potrf_async", self._p(local[k]), self.b, row0,
                     self._p(inv) if inv is not None else None, self.cl.stream)
        return 0

    def potrf(self, local, k, row0):
        import ctypes
        info = ctypes.c_int64(0)
        self.cl.call("bgp_tile_potrf", self._p(local[k]), self.b, row0, ctypes.byref(info),
                     self.cl.stream)
        return int(info.value)

    def copy_tile(self, dst, local, k):
        dst.copy_(local[k])

    def copy_tiles(self, dst, local, start, count):
        dst.copy_(local[start:start + count])

    def trsm_inv(self, inv, local, start, count):
        self.cl.call("bgp_panel_trsm_inv", self._p(inv), self._p(local[start]), count, self.b,
                     self.cl.stream)

    def trsm(self, diag, local, start, count):
        self.cl.call("bgp_panel_trsm", self._p(diag), self._p(local[start]), count, self.b,
                     self.cl.stream)

    def prepare_items(self, per_step):
        """Upload the update items of every step at once; returns per-step
        (device view, count)."""
        flat = [np.asarray(a, dtype=np.int32).reshape(-1, 4) for a in per_step]
        total = np.concatenate(flat) if flat and sum(len(a) for a in flat) else np.zeros((1, 4), np.int32)
        dev = self._items(total)
        out, off = [], 0
        for a in flat:
            out.append((dev[4 * off:4 * (off + len(a))], len(a)))
            off += len(a)
        return out

    def panel_exchange(self, comm, T):
        """The cluster's PanelExchange for T panel tiles (built collectively
        on first use), or None for NCCL broadcasts (BGP_PANEL_XFER=nccl, one
        rank, or a failed self-check)."""
        import os
        if comm.world == 1 or os.environ.get("BGP_PANEL_XFER", "push") != "push":
            return None
        cache = self.cl.__dict__.setdefault("_panel_xchg", {})
        x = cache.get("x")
        if x is None or x.tiles < T:
            if x is not None:
                x.close()
            x = PanelExchange(self.cl, comm, T)
            cache["x"] = x
        return x if x.ok else None

    # SMs left free during a reserved update for the side stream's NCCL
    # collectives, POTRF and panel solve
    RESERVE_SMS = 8

    def side(self):
        """Context: run on the side stream, after the work enqueued so far."""
        import torch
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.cl.device)
        self._side.wait_stream(torch.cuda.current_stream(self.cl.device))
        return torch.cuda.stream(self._side)

    def join_side(self):
        import torch
        if getattr(self, "_side", None) is not None:
            torch.cuda.current_stream(self.cl.device).wait_stream(self._side)

    def update(self, local, panel, items, reserve=False):
        if isinstance(items, tuple):
            dev, count = items
        else:
            dev, count = self._items(items), len(items)
        if count == 0:
            return
        if self.timeline is not None:
            with self.timeline.span("compute"):
                self._update(local, panel, dev, count, reserve)
        else:
            self._update(local, panel, dev, count, reserve)

    def _update(self, local, panel, dev, count, reserve):
        if reserve:
            self.cl.call("bgp_tile_update_limited", self._p(local), self._p(panel), self._p(panel),
                         self._p(dev), count, self.b, self.cl.num_sms - self.RESERVE_SMS, self.cl.stream)
        else:
            self.cl.call("bgp_tile_update", self._p(local), self._p(panel), self._p(panel),
                         self._p(dev), count, self.b, self.cl.stream)

    def sub_into(self, out, a, b):
        self.cl.call("bgp_sub", self._p(a), self._p(b), self._p(out), out.numel(), self.cl.stream)

    def tile_trsv(self, local, k, row0, x, trans):
        """Stream-ordered: a zero pivot stays in the device status (end())."""
        self.cl.call("bgp_tile_trsv", self._p(local[k]), self.b, row0, self.n, self._p(x), trans, None,
                     self.cl.stream)
        return 0

    def prepare_gemv_items(self, per_step):
        flat = [np.asarray(a, dtype=np.int32).reshape(-1, 2) for a in per_step]
        total = np.concatenate(flat) if flat and sum(len(a) for a in flat) else np.zeros((1, 2), np.int32)
        dev = self._items(total)
        out, off = [], 0
        for a in flat:
            out.append((dev[2 * off:2 * (off + len(a))], len(a)))
            off += len(a)
        return out

    def gemv(self, local, items, xJ, acc, trans):
        if isinstance(items, tuple):
            dev, count = items
        else:
            dev, count = self._items(items), len(items)
        if count == 0:
            return
        self.cl.call("bgp_tile_gemv", self._p(local), self._p(dev), count, self.b,
                     self._p(xJ), self._p(acc), trans, self.cl.stream)

    def logdet_partial(self, local, diag):
        import ctypes
        out, info = ctypes.c_double(0.0), ctypes.c_int64(0)
        if len(diag) == 0:
            return 0.0, 0
        dev = self._items(diag)
        self.cl.call("bgp_tile_logdet", self._p(local), self._p(dev), len(diag), self.b,
                     self.n, ctypes.byref(out), ctypes.byref(info), self.cl.stream)
        return out.value, int(info.value)

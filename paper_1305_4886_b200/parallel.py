"""Multi-GPU likelihood path: 2-D block-cyclic lower tiles, one process per GPU.

Replaces the reference's triangular D(D+1)/2 process fold
(bg/grid.py:116-139) and its tag-matched point-to-point messages
(bg/distla/kernels.py:139-250) with the SURVEY.md 8e plan:

  * tiles (I, J), I >= J, live on rank (I mod Pr) + Pr*(J mod Pc) of a
    Pr x Pc grid (1x1, 1x2, 2x2, 2x4); a rank stores its tiles packed by
    tile column, so each owned part of a panel is contiguous;
  * construct: every rank generates only its own tiles (no communication);
  * Cholesky step J: ONE launch per rank (bgp_dist_step) updates the rank's
    tiles with panel J; on process column (J+1) mod Pc the same launch
    factors (J+1, J+1) (the owner's tile or a shadow copy), solves the
    rank's panel-(J+1) tiles and stores them into every rank's panel buffer
    over NVLink; a stream-ordered barrier separates the steps (dist_cholesky);
  * forward / back solve: per block, the partial products of the owners of
    row (column) J are reduced to the diagonal owner, which solves and
    broadcasts x_J (2 x b doubles of traffic per step);
  * logdet: per-rank partials gathered and summed in rank order, as the
    reference's master does (bg/distla/__init__.py:154-157).

The schedule below is written against two small interfaces so the same code
runs on the GPUs (`LibTileOps` over libbgp + NCCL) and in the CPU tests
(a numpy tile backend + gloo, world sizes 2, 4 and 8).
"""

from dataclasses import dataclass, field

import numpy as np

from .grid import DeviceGrid


@dataclass
class StepPlan:
    """What one rank does in step J of the sweep (one launch, bgp_dist_step).

    items: (C local, A slot, B slot, flags) int32, column J+1 first
      (col_items of them); flags bit 0 = diagonal tile, bits 8.. = gate + 1.
    diag: local index of the tile (J+1, J+1) this rank factors in the launch
      (its own, or its shadow copy), or -1.
    trsm: (first local index, count) of its panel-(J+1) tiles, solved in the
      launch once their gates and the inverse are in.
    """

    items: np.ndarray
    col_items: int
    diag: int
    diag_row0: int
    trsm: tuple


@dataclass
class TileDist:
    """Ownership map of the lower tiles of an n x n matrix for one rank.

    Besides the tiles it owns, a rank keeps SHADOW copies of the diagonal
    tiles (K, K) of its process column owned by the other process row, for
    every K whose panel has tiles on this rank.  A shadow receives the same
    updates as the owner's tile (every panel is on every rank), so each rank
    of process column K mod Pc factors and inverts (K, K) itself inside its
    step launch and no rank ever waits on another inside a kernel.  Storage:
    owned tiles packed by tile column at [0, count), shadows at
    [count, count + len(shadows)).
    """

    n: int
    b: int
    grid: DeviceGrid
    rank: int  # 0-based
    T: int = field(init=False)
    tiles: np.ndarray = field(init=False)      # (k, 2) int32 (I, J), column-major
    local: dict = field(init=False)            # (I, J) -> local tile index
    col_start: np.ndarray = field(init=False)  # first local index of column J
    col_count: np.ndarray = field(init=False)
    shadows: list = field(init=False)          # K of the shadow diagonal tiles
    shadow_local: dict = field(init=False)     # K -> local index of the shadow

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
        self.shadows = [K for K in range(T) if K % pc == r_col and K % pr != r_row
                        and self.my_panel(K)[1] > 0]
        self.shadow_local = {K: len(tl) + i for i, K in enumerate(self.shadows)}

    @property
    def count(self):
        return len(self.tiles)

    @property
    def storage_count(self):
        """Local tiles including the shadow diagonal tiles."""
        return len(self.tiles) + len(self.shadows)

    @property
    def storage_tiles(self):
        """(I, J) of every local tile, shadows last (what construct builds)."""
        sh = np.array([(K, K) for K in self.shadows], dtype=np.int32).reshape(-1, 2)
        return np.concatenate([self.tiles, sh]).astype(np.int32)

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

    def factor_tile(self, K):
        """Local index of the (K, K) copy this rank factors, or -1: the owner
        always factors its tile; another rank of process column K mod Pc
        factors its shadow when it holds panel-K tiles to solve."""
        k = self.local.get((K, K))
        if k is not None:
            return k
        return self.shadow_local.get(K, -1)

    def update_items(self, J, slot):
        """(C local, A slot, B slot, lower) for my tiles (R, C), J < C <= R,
        and my shadows (K, K), K > J."""
        first = int(self.col_start[J + 1]) if J + 1 <= self.T - 1 else self.count
        t = self.tiles[first:]
        rows = []
        if len(t):
            R, C = t[:, 0].astype(np.int64), t[:, 1].astype(np.int64)
            # L2 super-columns (as the single-GPU update, gemm.cu
            # trail_order): ~16 MB of B-operand panel tiles per group of
            # local columns, swept row by row, so each A-operand panel tile
            # is read from HBM once per group instead of once per column
            sw = max(8, min(64, (16 << 20) // (self.b * self.b * 8)))
            order = np.lexsort((C, R, (C // self.grid.shape[1]) // sw))
            rows.append(np.stack([np.arange(first, first + len(t)), slot[R], slot[C], (R == C)], axis=1)[order])
        sh = [(self.shadow_local[K], slot[K], slot[K], 1) for K in self.shadows if K > J]
        if sh:
            rows.append(np.array(sh, dtype=np.int64))
        if not rows:
            return np.zeros((0, 4), dtype=np.int32)
        return np.concatenate(rows).astype(np.int32)

    def step_plan(self, J, slot, lookahead=True):
        """StepPlan of step J: the update by panel J of every local tile of
        columns > J (column J+1 first, gated), and, on process column
        (J+1) mod Pc, the factorization of (J+1, J+1) and the solve of this
        rank's panel-(J+1) tiles inside the same launch (not with
        lookahead=False: the last step before the gathered tail)."""
        K = J + 1
        items = self.update_items(J, slot)
        d = self.factor_tile(K) if lookahead else -1
        s, c = self.my_panel(K)
        if d < 0:
            return StepPlan(items, 0, -1, K * self.b, (s, 0))
        gate = np.full(len(items), -1, dtype=np.int64)
        gate[items[:, 0] == d] = 0
        for t in range(c):
            gate[items[:, 0] == s + t] = 1 + t
        items = items.copy()
        col = gate >= 0
        items[col, 3] |= ((gate[col] + 1) << 8).astype(np.int32)
        order = np.concatenate([np.nonzero(col)[0][np.argsort(gate[col], kind="stable")],
                                np.nonzero(~col)[0]])
        return StepPlan(items[order], int(col.sum()), d, K * self.b, (s, c))

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


# steps whose update work (tiles) is below this run the fused TRSM's column
# passes as independent tasks (the chain-bound regime; capi.cu bgp_potrf)
_PAR_PASS_TILES = {128: 48 * 49 // 2, 256: 26 * 27 // 2, 384: 22 * 23 // 2, 512: 18 * 19 // 2}


def dist_cholesky(dist, local, ops, comm):
    """Right-looking tiled Cholesky of a distributed matrix, in place, with
    the look-ahead inside each step's launch.

    `local` is this rank's (storage_count, b, b) tile stack (owned tiles,
    then shadow diagonal tiles).  Returns the first failing pivot row
    (1-based, LAPACK info) agreed by all ranks, or 0.

    Step J is ONE launch per rank (ops.step -> bgp_dist_step) on one stream:
    the update of all its tiles by panel J, column J+1 first; on process
    column (J+1) mod Pc the launch also factors and inverts (J+1, J+1) --
    every such rank its own copy (the owner's tile or its shadow), so no
    kernel waits on another GPU -- and solves the rank's panel-(J+1) tiles
    as gated tasks, storing each solved block into every rank's panel
    buffer over NVLink (PanelExchange).  One stream-ordered barrier between
    step launches orders the exchange: after it, panel J+1 is complete on
    every rank and every rank has finished reading the buffer that step J+1
    overwrites (double-buffered panels).  Without peer mappings the panel
    goes out by NCCL broadcasts after the launch instead (one per process
    row).  The host enqueues the whole sweep without waiting on the GPU; a
    failing pivot stays in the device status, which skips later launches.
    """
    b, T, me = dist.b, dist.T, dist.rank
    # tail: the last tile rows, where a step's update is shorter than the
    # look-ahead chain on any number of GPUs, are gathered to every rank and
    # finished there on 128 tiles (the single-GPU tail re-tiling)
    tail = ops.tail_tiles(T) if hasattr(ops, "tail_tiles") else 0
    J0 = T - tail if 0 < tail and 2 * tail < T else T
    nsteps = min(T - 1, J0)
    ops.sweep_begin(T)
    layouts = [dist.panel_layout(J) for J in range(T - 1)]
    plans = [dist.step_plan(J, layouts[J][1], lookahead=J + 1 < J0) for J in range(nsteps)]
    dev = ops.prepare_items([p.items for p in plans])
    par_tiles = _PAR_PASS_TILES.get(b, 0)
    # fused panel exchange (the TRSM epilogue stores into every rank's panel
    # buffer over NVLink), or None: NCCL broadcasts after each step's launch
    xchg = ops.panel_exchange(comm, T) if hasattr(ops, "panel_exchange") else None
    panels = [None, None]

    def buffer(K, ntot):
        if xchg is not None:
            return xchg.bufs[K % 2]
        if panels[K % 2] is None or panels[K % 2].shape[0] < ntot:
            panels[K % 2] = ops.empty((max(ntot, 1), b, b))
        return panels[K % 2]

    def push_args(K):
        """Destinations of my panel-K tiles: (xchg, which buffer, first slot)."""
        if xchg is None or K >= T - 1:
            return None
        chunks = layouts[K][0]
        off = next((o for root, o, cnt in chunks if root == me and cnt), 0)
        return (xchg, K % 2, off)

    def broadcast_panel(K):
        """Fallback exchange of panel K (after its solve): one broadcast per
        process-row chunk into every rank's panel buffer."""
        chunks, _, ntot = layouts[K]
        panel = buffer(K, ntot)
        for root, off, cnt in chunks:
            if cnt == 0:
                continue
            view = panel[off:off + cnt]
            if me == root:
                ps, pcount = dist.my_panel(K)
                assert pcount == cnt
                ops.copy_tiles(view, local, ps, cnt)
            comm.broadcast(view, root)

    # panel 0: factor (0, 0) (every rank of process column 0 its own copy),
    # solve and deliver my panel-0 tiles
    d0 = dist.factor_tile(0)
    s0, c0 = dist.my_panel(0)
    if d0 >= 0:
        ops.first_panel(local, d0, (s0, c0), push_args(0))
    if T > 1:
        if xchg is None:
            broadcast_panel(0)
    for J in range(nsteps):
        if xchg is not None:
            comm.barrier_stream()  # panel J complete everywhere; buffer (J+1) % 2 free
        plan = plans[J]
        par = plan.trsm[1] > 0 and len(plan.items) <= par_tiles
        ops.step(J, local, buffer(J, layouts[J][2]), dev[J], plan, par,
                 push_args(J + 1) if J + 1 < J0 else None)
        if xchg is None and J + 1 < min(T - 1, J0):
            broadcast_panel(J + 1)
    info = comm.min_nonzero(ops.end())
    # resident tiles at the peak (reported by distla.cholesky): my storage,
    # the two panel buffers, and the gathered tail triangle (+ my share)
    pbuf = 2 * xchg.tiles if xchg is not None else sum(p.shape[0] for p in panels if p is not None)
    T2 = T - J0
    ops.peak_tiles = dist.storage_count + pbuf + (T2 * (T2 + 1) // 2 + T2 * T2 // max(dist.grid.G, 1)
                                                  if J0 < T else 0)
    if J0 < T and not info:
        info = comm.min_nonzero(factor_tail(dist, local, ops, comm, J0))
    return info


def factor_tail(dist, local, ops, comm, J0):
    """Finish the factorization of the trailing tile rows J0.. (all panels
    < J0 applied): every rank gathers the trailing triangle (one all-gather
    of the ranks' trailing tiles, contiguous in their column-packed
    storage), factors it itself (ops.factor_tail: single-GPU look-ahead
    factorization re-tiled to 128) and keeps its own tiles.  Returns the
    failing pivot row (1-based, global) or 0."""
    b, T = dist.b, dist.T
    T2 = T - J0
    G = dist.grid.G
    shares = []
    for r in range(G):
        d = dist if r == dist.rank else TileDist(dist.n, b, dist.grid, r)
        first = int(d.col_start[J0])
        t = d.tiles[first:]
        I2, C2 = t[:, 0].astype(np.int64) - J0, t[:, 1].astype(np.int64) - J0
        shares.append((first, C2 * T2 - C2 * (C2 - 1) // 2 + (I2 - C2)))
    width = max(len(idx) for _, idx in shares)
    first, mine = shares[dist.rank]
    part = ops.empty((max(width, 1), b, b))
    if len(mine):
        part[:len(mine)].copy_(local[first:first + len(mine)])
    sub = ops.empty((T2 * (T2 + 1) // 2, b, b))
    import torch
    for (_, idx), piece in zip(shares, comm.all_gather(part)):
        if len(idx):
            sub.index_copy_(0, torch.from_numpy(idx).to(sub.device), piece[:len(idx)])
    info = ops.factor_tail(sub, T2, dist.n - J0 * b, J0 * b)
    if len(mine):
        local[first:first + len(mine)].copy_(sub.index_select(0, torch.from_numpy(mine).to(sub.device)))
    return info


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
        # per step, in issue order: each step launch ("compute") and each
        # barrier / broadcast ("comm") -- a step whose launch is short and
        # whose barrier long waited for another rank or for its own chain
        return {"comm_ms": comm, "collectives": len(iv["comm"]),
                "exposed_comm_ms": exposed_time(iv["comm"], iv["compute"]),
                "step_launch_ms": [round(b - a, 4) for a, b in iv["compute"]],
                "comm_span_ms": [round(b - a, 4) for a, b in iv["comm"]]}


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

    def all_gather_object(self, value):
        if self.world == 1:
            return [value]
        out = [None] * self.world
        self.dist.all_gather_object(out, value, group=self.group)
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

    def end(self, info=0):
        import ctypes
        dev = ctypes.c_int64(0)
        self.cl.call("bgp_info_read", ctypes.byref(dev), self.cl.stream)
        return int(info or dev.value)

    def copy_tiles(self, dst, local, start, count):
        dst.copy_(local[start:start + count])

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
        # (one push destination per rank, at most BGP_MAX_PUSH = 8: one node)
        if comm.world == 1 or comm.world > 8 or os.environ.get("BGP_PANEL_XFER", "push") != "push":
            return None
        cache = self.cl.__dict__.setdefault("_panel_xchg", {})
        x = cache.get("x")
        if x is None or x.tiles < T:
            if x is not None:
                x.close()
            x = PanelExchange(self.cl, comm, T)
            cache["x"] = x
        return x if x.ok else None

    def tail_tiles(self, T):
        """Trailing tile rows finished gathered on every rank:
        about 6,000 rows, where a step's update on any number of GPUs is
        shorter than the one-CTA POTRF + inverse chain at b = 256 / 512."""
        return {256: 24, 384: 16, 512: 12}.get(self.b, 0)

    def factor_tail(self, sub, T2, n2, row0):
        """Factor the packed trailing triangle `sub` (T2 tile rows of b, n2
        live rows) in place on this GPU: re-tiled to 128 and run through
        bgp_potrf (look-ahead inside the update launches).  Returns the
        failing row (global, 1-based) or 0."""
        import ctypes

        import torch
        b, f = self.b, self.b // 128
        T1 = T2 * f
        key = (T2, b)
        if getattr(self, "_tail_idx", (None,))[0] != key:
            i1 = np.array([i for j in range(T1) for i in range(j, T1)])
            j1 = np.array([j for j in range(T1) for i in range(j, T1)])
            I, J = i1 // f, j1 // f
            big = J * T2 - J * (J - 1) // 2 + (I - J)
            dev = lambda a: torch.from_numpy(a).to(self.cl.device)  # noqa: E731
            self._tail_idx = (key, dev(big), dev(j1 % f), dev(i1 % f))
        _, big, cj, ci = self._tail_idx
        view = sub.view(-1, f, 128, f, 128)  # [tile][cj][cc][ci][rr] (column-major tiles)
        small = view[big, cj, :, ci, :].contiguous()
        info = ctypes.c_int64(0)
        self.cl.call("bgp_potrf", self._p(small), n2, 128, ctypes.byref(info), self.cl.stream)
        view[big, cj, :, ci, :] = small
        return row0 + int(info.value) if info.value else 0

    def sweep_begin(self, T):
        self._T = T
        self.cl.call("bgp_dist_begin", T, self.b, self.cl.stream)
        if getattr(self, "_linv", None) is None:
            self._linv = self.cl.empty((self.b, self.b))

    @staticmethod
    def _dst(push, count):
        """(dst array, ndst, first slot, buffer tiles) of a panel push."""
        if push is None or count == 0:
            return None, 0, 0, 1
        xchg, which, slot0 = push
        return xchg.dst[which], len(xchg.dst[which]), slot0, xchg.tiles

    def first_panel(self, local, d, trsm, push):
        """Factor local tile d (panel 0's diagonal, or its shadow), invert it,
        solve my panel-0 tiles and (push) deliver them to every rank."""
        s, c = trsm
        self.cl.call("bgp_tile_potrf_async", self._p(local[d]), self.b, 0,
                     self._p(self._linv) if c else None, self.cl.stream)
        if c == 0:
            return
        dst, ndst, slot0, tiles = self._dst(push, c)
        if ndst:
            self.cl.call("bgp_panel_trsm_push", self._p(self._linv), self._p(local[s]), c, self.b,
                         dst, ndst, slot0, tiles, self.cl.stream)
        else:
            self.cl.call("bgp_panel_trsm_inv", self._p(self._linv), self._p(local[s]), c, self.b,
                         self.cl.stream)

    def step(self, J, local, panel, items, plan, par, push):
        """Step J of the sweep on this rank: one bgp_dist_step launch."""
        dev, count = items
        s, c = plan.trsm
        if count == 0 and plan.diag < 0:
            return
        dst, ndst, slot0, tiles = self._dst(push, c)
        diag = self._p(local[plan.diag]) if plan.diag >= 0 else None
        args = ("bgp_dist_step", J, self._p(local), local.shape[0], self._p(panel), panel.shape[0],
                self._p(dev) if count else None, count, plan.col_items, diag, plan.diag_row0, s, c,
                1 if par else 0, dst, ndst, slot0, tiles, self.b, self.cl.stream)
        if self.timeline is not None:
            with self.timeline.span("compute"):
                self.cl.call(*args)
        else:
            self.cl.call(*args)

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

"""Device implementations of the reference's distla operation ids.

Each function here is registered under the same op id as the reference's
worker SPMD function (bg/distla/kernels.py) and is invoked through
`B200Cluster.run(op_id, **kwargs)` with the same keyword arguments.  The
`ctx` argument is the cluster (the GPU is the worker).  All arithmetic is in
libbgp (include/bgp.h); these functions allocate buffers, check shapes and
map device status codes onto the reference's exceptions.
"""

import ctypes

import numpy as np

from .. import _lib, registry
from ..errors import (DimensionMismatch, GeneratorError, NotPositiveDefinite,
                      SingularDiagonal, UnknownFunction, UnsupportedSmoothness)
from ..grid import BlockLayout
from .objects import DevObj

HALF_INTEGER_NU = (0.5, 1.5, 2.5)


def _ntiles(n, b):
    return -(-n // b)


def _alloc(ctx, kind, n, m=None):
    b = ctx.tile
    T = _ntiles(n, b)
    if kind == "triangular":
        return ctx.empty((T * (T + 1) // 2, b, b))
    if kind == "rectangular":
        return ctx.empty((T * _ntiles(m, b), b, b))
    return ctx.empty((T * b,))


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _need(ctx, name, kind, full=True):
    obj = ctx.fetch(name)
    if not isinstance(obj, DevObj) or obj.kind != kind:
        raise DimensionMismatch(f"object {name!r} is not a device {kind} object")
    return _full(ctx, obj) if full else obj


def _packed_index(dist, tiles=None):
    """Packed-triangle index of a rank's tiles (default: the owned ones)."""
    import torch
    tiles = dist.tiles if tiles is None else tiles
    I = tiles[:, 0].astype(np.int64)
    J = tiles[:, 1].astype(np.int64)
    T = dist.T
    return torch.from_numpy(J * T - J * (J - 1) // 2 + (I - J))


def _rank_maps(ctx, n):
    """(count, packed index on the device) of every rank's tiles, cached per n."""
    cache = ctx.__dict__.setdefault("_rank_tile_maps", {})
    key = (n, ctx.tile)
    if key not in cache:
        from ..parallel import TileDist
        maps = []
        for r in range(ctx.G):
            td = TileDist(n, ctx.tile, ctx.grid, r)
            maps.append((td.count, _packed_index(td).to(ctx.device)))
        cache[key] = maps
    return cache[key]


def _full(ctx, obj):
    """Replicated packed copy of a distributed triangular object (for the
    operations that run on one GPU's full copy: collect, kriging solves,
    crossproducts, elementwise helpers): one all-gather of every rank's
    tiles (padded to the largest share), scattered to packed order."""
    if obj.dist is None:
        return obj
    d = obj.dist
    maps = _rank_maps(ctx, obj.n)
    width = max(c for c, _ in maps)
    part = ctx.empty((max(width, 1), obj.tile, obj.tile))
    if d.count:
        part[:d.count].copy_(obj.data[:d.count])
    full = ctx.empty((d.T * (d.T + 1) // 2, obj.tile, obj.tile))
    for (count, idx), piece in zip(maps, ctx.comm.all_gather(part)):
        if count:
            full.index_copy_(0, idx, piece[:count])
    return DevObj(obj.kind, obj.row_layout, obj.col_layout, obj.tile, full)


def _my_cols(ctx, m):
    """Column shards of an m-column object over the job's GPUs (tile rows of
    the transposed storage) and this rank's (r0, r1)."""
    from ..parallel import col_shards
    shards = col_shards(_ntiles(m, ctx.tile), ctx.G)
    return shards, shards[ctx.rank - 1]


def _gather_rect(ctx, X, Tn, Tm, shards):
    """All-gather column shards (Tn, r1 - r0, b, b) into a replicated
    (Tn * Tm, b, b) transposed rectangular object."""
    from ..parallel import gather_col_shards
    b = ctx.tile
    width = max(r1 - r0 for r0, r1 in shards)
    part = ctx.zeros((Tn, width, b, b))
    part[:, :X.shape[1]].copy_(X)
    full = ctx.empty((Tn * Tm, b, b))
    view = full.view(Tn, Tm, b, b)

    def fill(r0, r1, piece):
        view[:, r0:r1].copy_(piece)
    gather_col_shards(ctx.comm, part, shards, fill)
    return full


def _gather_vec(ctx, w, shards):
    """All-gather per-rank m-vector shards (tile rows r0..r1) into one vector."""
    from ..parallel import gather_col_shards
    b = ctx.tile
    width = max(r1 - r0 for r0, r1 in shards)
    part = ctx.zeros((1, width * b))
    part[0, :w.shape[0]].copy_(w)
    full = ctx.zeros((shards[-1][1] * b,))

    def fill(r0, r1, piece):
        full[r0 * b:r1 * b].copy_(piece.reshape(-1)[:(r1 - r0) * b])
    gather_col_shards(ctx.comm, part.view(1, width, b), shards, fill)
    return full


def _tile_ops(ctx, n):
    from ..parallel import LibTileOps
    return LibTileOps(ctx, n)


# ---------------------------------------------------------------------------
# construction (bg/distla/kernels.py:35-75)

def _device_generator(ctx, gen_id, params, inputs, kind):
    g = registry.device_generator(gen_id)
    params = np.asarray(params, dtype=float).ravel()
    desc = _lib.Generator()
    desc.family, desc.part, desc.nugget = g.family, g.part, int(g.nugget)
    desc.nparams = len(params)
    if len(params) > 8:
        raise DimensionMismatch("at most 8 kernel parameters")
    for i, v in enumerate(params):
        desc.params[i] = float(v)
    desc.nu = float(inputs.get("nu", inputs.get("nu1", 0.5))) if inputs else 0.5
    desc.nu2 = float(inputs.get("nu2", 0.5)) if inputs else 0.5
    fam = g.family
    try:
        if fam in (_lib.GEN_MATERN, _lib.GEN_SQEXP, _lib.GEN_PRODUCT) and g.part != _lib.PART_PREDVAR:
            # the reference's generators raise inside the worker; those
            # errors surface as GeneratorError (bg/distla/kernels.py:66-69)
            if fam == _lib.GEN_PRODUCT:
                nus = (desc.nu, desc.nu2)
                rhos = params[1:3]
            else:
                nus = (desc.nu,) if fam == _lib.GEN_MATERN else ()
                rhos = params[1:2]
            for nu in nus:
                if nu not in HALF_INTEGER_NU:
                    raise UnsupportedSmoothness(
                        f"nu={nu} not supported; use one of {HALF_INTEGER_NU}")
            if fam == _lib.GEN_MATERN or fam == _lib.GEN_PRODUCT:
                for rho in rhos:
                    if rho <= 0:
                        raise ValueError(f"range must be positive, got {rho}")
        if fam == _lib.GEN_LINEAR_INDEX:
            desc.params[0] = float(inputs["n"])
            desc.nparams = 1
    except Exception as exc:
        raise GeneratorError(ctx.rank, exc) from exc
    return g, desc


@registry.register("distla.construct")
def construct(ctx, name, kind, generator, params, inputs_name, row_layout, col_layout=None):
    inputs = ctx.fetch(inputs_name) if inputs_name else {}
    g, desc = _device_generator(ctx, generator, params, inputs, kind)
    n = row_layout.n
    m = col_layout.n if (kind == "rectangular" and col_layout is not None) else None
    if kind == "rectangular" and col_layout is None:
        raise DimensionMismatch("rectangular construction needs a column layout")
    needs_points = g.family in (_lib.GEN_MATERN, _lib.GEN_SQEXP, _lib.GEN_PRODUCT) \
        and g.part != _lib.PART_PREDVAR and kind != "vector"
    X = Y = None
    dim = 1
    if needs_points:
        key_x = "pred_coords" if g.part == _lib.PART_PRED else "coords"
        X = ctx.device_input(inputs_name, key_x)
        dim = X.shape[1]
        if X.shape[0] < n:
            raise GeneratorError(ctx.rank, IndexError(
                f"{key_x} has {X.shape[0]} points, layout needs {n}"))
        if g.part == _lib.PART_CROSS:
            Y = ctx.device_input(inputs_name, "pred_coords")
            if Y.shape[1] != dim or Y.shape[0] < m:
                raise GeneratorError(ctx.rank, IndexError("pred_coords do not conform"))
        keys = ("coords", "pred_coords") if g.part == _lib.PART_CROSS else (key_x,)
        desc.span = ctx.input_span(inputs_name, keys)
    if name in ctx.store:
        del ctx.store[name]
    if kind == "triangular" and ctx.G > 1:
        from ..parallel import TileDist
        td = TileDist(n, ctx.tile, ctx.grid, ctx.rank - 1)
        # owned tiles, then the shadow diagonal tiles (parallel.TileDist)
        out = ctx.empty((max(td.storage_count, 1), ctx.tile, ctx.tile))
        tij = ctx.upload_int32(td.storage_tiles)
        ctx.call("bgp_construct_tiles", ctypes.byref(desc), _ptr(X) if X is not None else None, n, dim,
                 ctx.tile, _ptr(tij), td.storage_count, _ptr(out), ctx.stream)
        ctx.store[name] = DevObj(kind, row_layout, col_layout or row_layout, ctx.tile, out, td)
        ctx.log_event("construct")
        return
    out = _alloc(ctx, kind, n, m)
    ctx.call("bgp_construct", _lib.KIND_CODE[kind], ctypes.byref(desc),
             _ptr(X) if X is not None else None, n,
             _ptr(Y) if Y is not None else None, m or 0, dim, ctx.tile, _ptr(out), ctx.stream)
    cl = (col_layout or row_layout) if kind != "vector" else None
    ctx.store[name] = DevObj(kind, row_layout, cl, ctx.tile, out)
    ctx.log_event("construct")


@registry.register("distla.split")
def split(ctx, name, kind, array, row_layout, col_layout=None):
    """Upload a master-side dense array (bg/distla/kernels.py:538-544)."""
    a = np.asarray(array, dtype=float)
    n = row_layout.n
    if kind == "vector":
        if a.shape != (n,):
            raise DimensionMismatch(f"vector length {a.shape} != {n}")
        m = None
    elif kind == "triangular":
        if a.shape != (n, n):
            raise DimensionMismatch(f"triangular array {a.shape} != ({n}, {n})")
        m = n
    else:
        if col_layout is None or a.shape != (n, col_layout.n):
            raise DimensionMismatch("rectangular array does not match its layouts")
        m = col_layout.n
    dense = ctx.upload(a)
    out = _alloc(ctx, kind, n, m)
    ld = a.shape[1] if a.ndim == 2 else 1
    ctx.call("bgp_pack", _lib.KIND_CODE[kind], _ptr(dense), n, m or 1, ld, ctx.tile,
             _ptr(out), ctx.stream)
    cl = (col_layout or row_layout) if kind != "vector" else None
    td = None
    if kind == "triangular" and ctx.G > 1:
        from ..parallel import TileDist
        td = TileDist(n, ctx.tile, ctx.grid, ctx.rank - 1)
        out = out.index_select(0, _packed_index(td, td.storage_tiles).to(out.device)).contiguous()
    ctx.store[name] = DevObj(kind, row_layout, cl, ctx.tile, out, td)


# ---------------------------------------------------------------------------
# Cholesky (bg/distla/kernels.py:110-194)

@registry.register("distla.cholesky")
def cholesky(ctx, name, out_name):
    obj = _need(ctx, name, "triangular", full=False)
    if out_name != name:
        ctx.store[out_name] = obj
        del ctx.store[name]
    info = ctypes.c_int64(0)
    try:
        if obj.dist is not None:
            import time
            from ..parallel import LibTileOps, Timeline, dist_cholesky
            # ctx.comm_timeline: record comm / compute spans (exposed-comm report)
            tl = Timeline(ctx.device) if getattr(ctx, "comm_timeline", False) else None
            ctx.comm.timeline = tl
            ctx.synchronize()
            t0 = time.perf_counter()
            ops = LibTileOps(ctx, obj.n, tl)
            try:
                info.value = dist_cholesky(obj.dist, obj.data, ops, ctx.comm)
                peak_tiles = getattr(ops, "peak_tiles", obj.dist.storage_count)
            finally:
                ctx.comm.timeline = None
            ctx.synchronize()
            ctx.last_cholesky_ms = 1e3 * (time.perf_counter() - t0)
            ctx.last_comm = tl.summary() if tl is not None else None
        else:
            ctx.call("bgp_potrf", _ptr(obj.data), obj.n, obj.tile, ctypes.byref(info), ctx.stream)
    except BaseException:
        ctx.store.pop(out_name, None)  # no partial factor is retained
        raise
    if info.value:
        ctx.store.pop(out_name, None)
        raise NotPositiveDefinite((info.value - 1) // obj.row_layout.block_size + 1)
    ctx.log_event("factor")
    # peak_blocks in the reference's unit (row-layout blocks, bg/distla/
    # kernels.py: blocks resident at the peak): this rank's resident device
    # elements / block_size^2.  Distributed: owned tiles, shadow diagonal
    # tiles, the two panel-exchange buffers and the gathered tail; the
    # panel buffers (2 x T tiles) dominate at small n
    bs2 = float(obj.row_layout.block_size) ** 2
    t2 = float(obj.tile) ** 2
    if obj.dist is not None:
        return {"peak_blocks": peak_tiles * t2 / bs2, "owned_blocks": obj.dist.count * t2 / bs2,
                "tile": obj.tile, "peak_tiles": int(peak_tiles), "storage_tiles": obj.dist.storage_count,
                "owned_tiles": obj.dist.count}
    nt = obj.data.shape[0]
    return {"peak_blocks": nt * t2 / bs2, "owned_blocks": nt * t2 / bs2, "tile": obj.tile, "peak_tiles": nt,
            "storage_tiles": nt, "owned_tiles": nt}


@registry.register("distla.loglik_many")
def loglik_many(ctx, thetas, cov_fn, mean_fn, inputs_name, y_name, row_layout, lanes=2):
    """logdet, sumsq and status of log_density at every theta of a list
    (one GPU), pipelined: evaluation k runs on lane k mod `lanes` (its own
    library context and stream), so the covariance build and first panels of
    evaluation k+1 fill the SMs the latency-bound tail of evaluation k's
    Cholesky leaves idle.  Each evaluation is the path of
    bg/gp/problem.py:119-142 (construct, Cholesky, y - mu, forward solve,
    logdet, sumsq) with the stream-ordered entry points; one host
    synchronization at the end.  Returns [(logdet, ssq, info)] in order."""
    import torch
    if ctx.G > 1:
        raise DimensionMismatch("loglik_many runs on one GPU (use log_density per theta)")
    inputs = ctx.fetch(inputs_name)
    y = _need(ctx, y_name, "vector")
    n, b = row_layout.n, ctx.tile
    T = _ntiles(n, b)
    gens = []
    for th in thetas:
        g, desc = _device_generator(ctx, cov_fn, th, inputs, "triangular")
        _, mdesc = _device_generator(ctx, mean_fn, th, inputs, "vector")
        gens.append((g, desc, mdesc))
    X = None
    dim = 1
    if gens and gens[0][0].family in (_lib.GEN_MATERN, _lib.GEN_SQEXP, _lib.GEN_PRODUCT):
        X = ctx.device_input(inputs_name, "coords")
        dim = X.shape[1]
        span = ctx.input_span(inputs_name, ("coords",))
        for _, desc, _ in gens:
            desc.span = span
    lanes = ctx.lanes(max(1, int(lanes)))
    # every lane's GEMM launches leave a few SMs free, so a lane in its
    # latency-bound tail is not starved by the other lane's full-width
    # launches (C2 at tile 256: 21.6 -> 22.1 evals/s with 8; BGP_LANE_RESERVE)
    import os
    reserve = int(os.environ.get("BGP_LANE_RESERVE", "8"))
    for lc, _ in lanes:
        ctx.lib.bgp_set_grid_cap(lc, ctx.num_sms - reserve if reserve and len(lanes) > 1 else 0)
    key = (n, b, len(lanes))
    bufs = ctx.__dict__.get("_many_bufs")
    if bufs is None or bufs[0] != key:
        bufs = (key, [(ctx.empty((T * (T + 1) // 2, b, b)), ctx.empty((T * b,)), ctx.empty((T * b,)))
                      for _ in lanes])
        ctx.__dict__["_many_bufs"] = bufs
    res = ctx.zeros((max(len(thetas), 1), 2))
    info = torch.zeros(max(len(thetas), 1), dtype=torch.int64, device=ctx.device)
    cur = torch.cuda.current_stream(ctx.device)
    for _, st in lanes:
        st.wait_stream(cur)
    for k, (g, desc, mdesc) in enumerate(gens):
        lc, st = lanes[k % len(lanes)]
        C, mu, x = bufs[1][k % len(lanes)]
        s = st.cuda_stream
        ctx.call_on(lc, "bgp_construct", _lib.BGP_TRI, ctypes.byref(desc),
                    _ptr(X) if X is not None else None, n, None, 0, dim, b, _ptr(C), s)
        ctx.call_on(lc, "bgp_potrf_async", _ptr(C), n, b, s)
        ctx.call_on(lc, "bgp_construct", _lib.BGP_VEC, ctypes.byref(mdesc), None, n, None, 0, 1, b,
                    _ptr(mu), s)
        ctx.call_on(lc, "bgp_sub", _ptr(y.data), _ptr(mu), _ptr(x), T * b, s)
        ctx.call_on(lc, "bgp_trsv_async", _ptr(C), n, b, _ptr(x), 0, s)
        ctx.call_on(lc, "bgp_logdet_async", _ptr(C), n, b, _ptr(res[k, 0:1]), s)
        ctx.call_on(lc, "bgp_sumsq_async", _ptr(x), n, _ptr(res[k, 1:2]), s)
        ctx.call_on(lc, "bgp_info_copy", _ptr(info[k:k + 1]), s)
    for _, st in lanes:
        cur.wait_stream(st)
    out = res.cpu().numpy()
    inf = info.cpu().numpy()
    return [(float(out[k, 0]), float(out[k, 1]), int(inf[k])) for k in range(len(thetas))]


# ---------------------------------------------------------------------------
# triangular solves (bg/distla/kernels.py:200-307)

@registry.register("distla.solve_vector")
def solve_vector(ctx, l_name, rhs_name, out_name, forward=True):
    L = _need(ctx, l_name, "triangular", full=False)
    rhs = _need(ctx, rhs_name, "vector")
    if rhs.data.shape[0] != L.tile * _ntiles(L.n, L.tile) or rhs.n != L.n:
        raise DimensionMismatch("rhs does not conform to L")
    info = ctypes.c_int64(0)
    if L.dist is not None:
        from ..parallel import dist_trsv
        x, info.value = dist_trsv(L.dist, L.data, rhs.data, _tile_ops(ctx, L.n), ctx.comm, forward)
    else:
        x = rhs.data.clone()
        ctx.call("bgp_trsv", _ptr(L.data), L.n, L.tile, _ptr(x), 0 if forward else 1,
                 ctypes.byref(info), ctx.stream)
    if info.value:
        raise SingularDiagonal(f"zero diagonal at row {info.value}")
    ctx.store[out_name] = DevObj("vector", rhs.row_layout, None, rhs.tile, x)
    ctx.log_event("solve")


@registry.register("distla.solve_rect")
def solve_rect(ctx, l_name, rhs_name, out_name, forward=True):
    L = _need(ctx, l_name, "triangular")
    B = _need(ctx, rhs_name, "rectangular")
    if B.n != L.n:
        raise DimensionMismatch("rhs rows do not conform to L")
    info = ctypes.c_int64(0)
    if ctx.G > 1:
        # columns are independent: each GPU solves its shard of the RHS
        # columns against the replicated L, then the shards are all-gathered
        #
        b = ctx.tile
        Tm, Tn = _ntiles(B.m, b), _ntiles(B.n, b)
        shards, (r0, r1) = _my_cols(ctx, B.m)
        X = B.data.view(Tn, Tm, b, b)[:, r0:r1].contiguous()
        mloc = max(0, min(B.m, r1 * b) - r0 * b)
        if mloc:
            ctx.call("bgp_trsm_rect", _ptr(L.data), L.n, L.tile, _ptr(X), mloc, 0 if forward else 1,
                     ctypes.byref(info), ctx.stream)
        info.value = ctx.comm.min_nonzero(info.value)
        if not info.value:
            X = _gather_rect(ctx, X, Tn, Tm, shards)
    else:
        X = B.data.clone()
        ctx.call("bgp_trsm_rect", _ptr(L.data), L.n, L.tile, _ptr(X), B.m, 0 if forward else 1,
                 ctypes.byref(info), ctx.stream)
    if info.value:
        raise SingularDiagonal(f"zero diagonal at row {info.value}")
    ctx.store[out_name] = DevObj("rectangular", B.row_layout, B.col_layout, B.tile, X)
    ctx.log_event("solve")


# ---------------------------------------------------------------------------
# crossproducts (bg/distla/kernels.py:387-487)

@registry.register("distla.xprod_mat_vec")
def xprod_mat_vec(ctx, v_name, u_name, out_name):
    V = _need(ctx, v_name, "rectangular")
    u = _need(ctx, u_name, "vector")
    if u.n != V.n:
        raise DimensionMismatch("u does not conform to V")
    if ctx.G > 1:
        w = _sharded_cols(ctx, V, lambda Vs, mloc, ws: ctx.call(
            "bgp_xprod_mat_vec", _ptr(Vs), V.n, mloc, V.tile, _ptr(u.data), _ptr(ws), ctx.stream))
    else:
        w = _alloc(ctx, "vector", V.m)
        ctx.call("bgp_xprod_mat_vec", _ptr(V.data), V.n, V.m, V.tile, _ptr(u.data), _ptr(w), ctx.stream)
    ctx.store[out_name] = DevObj("vector", V.col_layout, None, V.tile, w)


def _sharded_cols(ctx, V, kernel):
    """Per-column reduction of a replicated rectangular V on G > 1 GPUs: each
    rank runs `kernel(V shard, local columns, out shard)` on its column shard
    and the m-vector shards are all-gathered in rank order."""
    b = ctx.tile
    Tm, Tn = _ntiles(V.m, b), _ntiles(V.n, b)
    shards, (r0, r1) = _my_cols(ctx, V.m)
    mloc = max(0, min(V.m, r1 * b) - r0 * b)
    ws = ctx.zeros(((r1 - r0) * b,))
    if mloc:
        Vs = V.data.view(Tn, Tm, b, b)[:, r0:r1].contiguous()
        kernel(Vs, mloc, ws)
    return _gather_vec(ctx, ws, shards)


@registry.register("distla.xprod_self")
def xprod_self(ctx, v_name, out_name):
    V = _need(ctx, v_name, "rectangular")
    S = _alloc(ctx, "triangular", V.m)
    ctx.call("bgp_xprod_self", _ptr(V.data), V.n, V.m, V.tile, _ptr(S), ctx.stream)
    ctx.store[out_name] = DevObj("triangular", V.col_layout, V.col_layout, V.tile, S)


@registry.register("distla.xprod_self_diag")
def xprod_self_diag(ctx, v_name, out_name):
    V = _need(ctx, v_name, "rectangular")
    if ctx.G > 1:
        d = _sharded_cols(ctx, V, lambda Vs, mloc, ds: ctx.call(
            "bgp_xprod_self_diag", _ptr(Vs), V.n, mloc, V.tile, _ptr(ds), ctx.stream))
    else:
        d = _alloc(ctx, "vector", V.m)
        ctx.call("bgp_xprod_self_diag", _ptr(V.data), V.n, V.m, V.tile, _ptr(d), ctx.stream)
    ctx.store[out_name] = DevObj("vector", V.col_layout, None, V.tile, d)


# ---------------------------------------------------------------------------
# reductions (bg/distla/kernels.py:493-522)

@registry.register("distla.logdet")
def logdet(ctx, l_name):
    L = _need(ctx, l_name, "triangular", full=False)
    if L.dist is not None:
        # this rank's partial over its diagonal tiles; run() gathers the
        # partials and the master sums them in rank order (__init__.py:157)
        value, info = _tile_ops(ctx, L.n).logdet_partial(L.data, L.dist.diag_items())
        info = ctx.comm.min_nonzero(info)
        if info:
            raise SingularDiagonal(f"non-positive diagonal at row {info}")
        return value
    out = ctypes.c_double(0.0)
    info = ctypes.c_int64(0)
    ctx.call("bgp_logdet", _ptr(L.data), L.n, L.tile, ctypes.byref(out), ctypes.byref(info),
             ctx.stream)
    if info.value:
        raise SingularDiagonal(f"non-positive diagonal at row {info.value}")
    return out.value


@registry.register("distla.sumsq")
def sumsq(ctx, name):
    x = _need(ctx, name, "vector")
    if ctx.G > 1 and ctx.rank != 1:
        return 0.0  # vectors are replicated: rank 1 holds the whole sum
    out = ctypes.c_double(0.0)
    ctx.call("bgp_sumsq", _ptr(x.data), x.n, ctypes.byref(out), ctx.stream)
    return out.value


# ---------------------------------------------------------------------------
# collection (bg/distla/kernels.py:525-535, objects.py:108-123)

def dense_of(ctx, obj):
    """Unpadded host array of a device object (lower-triangular for
    triangular objects)."""
    torch = __import__("torch")
    obj = _full(ctx, obj)
    if obj.kind == "vector":
        return obj.data[:obj.n].cpu().numpy().copy()
    n, m = obj.n, (obj.m if obj.kind == "rectangular" else obj.n)
    dense = torch.zeros((n, m), dtype=torch.float64, device=obj.data.device)
    ctx.call("bgp_unpack", _lib.KIND_CODE[obj.kind], _ptr(obj.data), n, m, obj.tile,
             _ptr(dense), m, ctx.stream)
    return dense.cpu().numpy()


def diagonal_of(ctx, obj):
    torch = __import__("torch")
    obj = _full(ctx, obj)
    d = torch.empty((obj.n,), dtype=torch.float64, device=obj.data.device)
    ctx.call("bgp_tri_diagonal", _ptr(obj.data), obj.n, obj.tile, _ptr(d), ctx.stream)
    return d.cpu().numpy()


def _blocks_of(dense, kind, rl, cl, diagonal_only):
    """Reference-format {(I, J): block} pieces of an unpadded dense array."""
    if kind == "vector":
        bs = rl.block_size
        x = np.zeros(rl.padded_n)
        x[:rl.n] = dense
        return {J: x[(J - 1) * bs:J * bs].copy() for J in range(1, rl.B + 1)}
    cl = cl or rl
    bsr, bsc = rl.block_size, cl.block_size
    A = np.zeros((rl.padded_n, cl.padded_n))
    A[:rl.n, :cl.n] = dense
    if kind == "triangular":
        for t in range(rl.n, rl.padded_n):
            A[t, t] = 1.0
    out = {}
    for J in range(1, cl.B + 1):
        for I in range(J if kind == "triangular" else 1, rl.B + 1):
            blk = A[(I - 1) * bsr:I * bsr, (J - 1) * bsc:J * bsc]
            if diagonal_only:
                if I == J:
                    out[(I, J)] = np.diag(blk).copy()
            else:
                out[(I, J)] = blk.copy()
    return out


@registry.register("distla.collect")
def collect_blocks(ctx, name, diagonal_only=False):
    """Operator-level collect: pieces in the object's API layout."""
    obj = ctx.fetch(name)
    if not isinstance(obj, DevObj):
        raise DimensionMismatch(f"{name!r} is not a distributed object")
    return _blocks_of(dense_of(ctx, obj), obj.kind, obj.row_layout, obj.col_layout,
                      diagonal_only)


# ---------------------------------------------------------------------------
# elementwise helpers used through remote_apply (bg/distla/kernels.py:550-564)

def _conform(a, b):
    if not (isinstance(a, DevObj) and isinstance(b, DevObj) and a.kind == b.kind
            and a.data.shape == b.data.shape and a.tile == b.tile):
        raise DimensionMismatch("local pieces do not align")


def _sub(ctx, a, b):
    _conform(a, b)
    out = ctx.empty(a.data.shape)
    ctx.call("bgp_sub", _ptr(a.data), _ptr(b.data), _ptr(out), a.data.numel(), ctx.stream)
    return DevObj(a.kind, a.row_layout, a.col_layout, a.tile, out)


def _negate(ctx, a):
    zero = DevObj(a.kind, a.row_layout, a.col_layout, a.tile, ctx.zeros(a.data.shape))
    return _sub(ctx, zero, a)


def _add(ctx, a, b):
    return _sub(ctx, a, _negate(ctx, b))


_ELEMENTWISE = {"sub": _sub, "add": _add, "negate": _negate}


@registry.register("core.apply")
def apply(ctx, op_id, input_names, output_name):
    fn = _ELEMENTWISE.get(op_id)
    if fn is None:
        registry.lookup(op_id)  # UnknownFunction for ids that do not exist at all
        raise UnknownFunction(f"{op_id!r} has no device implementation")
    ctx.store[output_name] = fn(ctx, *[_full(ctx, ctx.fetch(n)) if isinstance(ctx.fetch(n), DevObj)
                                        else ctx.fetch(n) for n in input_names])


@registry.register("distla.mult_vector")
def mult_vector(ctx, l_name, x_name, out_name):
    """y = L x (bg/distla/kernels.py:313-343)."""
    L = _need(ctx, l_name, "triangular")
    x = _need(ctx, x_name, "vector")
    if x.n != L.n:
        raise DimensionMismatch("x does not conform to L")
    y = ctx.empty(x.data.shape)
    ctx.call("bgp_tri_mv", _ptr(L.data), L.n, L.tile, _ptr(x.data), _ptr(y), 0, ctx.stream)
    ctx.store[out_name] = DevObj("vector", x.row_layout, None, x.tile, y)


@registry.register("distla.rnorm")
def construct_rnorm(ctx, name, kind, row_layout, col_layout=None, fill="normal"):
    """i.i.d. N(0,1) object from this rank's stream (bg/distla/kernels.py:78-104).

    The stream is the reference's (bg/rng.py:18-28): Philox4x64-10 keyed by
    (seed << 64) + rank, one draw per element of every owned block, padding
    included, in the reference's block order.  At G = 1 (rank 1, the same
    API layout as the reference's P = 1) the draws equal the reference's up
    to the inverse-CDF ulps; with G > 1 every rank draws the rank-1 stream
    (objects are replicated).  fill="zeros" draws nothing.
    """
    from ..errors import StreamsUninitialized
    if kind not in ("vector", "rectangular"):
        raise DimensionMismatch(f"rnorm fills vectors or rectangular objects, not {kind!r}")
    n = row_layout.n
    m = col_layout.n if kind == "rectangular" else 0
    out = _alloc(ctx, kind, n, m).zero_()
    if fill != "zeros":
        if ctx.seed is None:
            raise StreamsUninitialized("no master seed installed")
        bs_r = row_layout.block_size
        bs_c = col_layout.block_size if kind == "rectangular" else 1
        nblocks = row_layout.B * (col_layout.B if kind == "rectangular" else 1)
        ctx.call("bgp_rnorm", n, m, bs_r, bs_c, int(ctx.seed), 1, ctx.stream_pos, ctx.tile,
                 _ptr(out), ctx.stream)
        ctx.stream_pos += nblocks * bs_r * bs_c
    cl = col_layout if kind == "rectangular" else None
    ctx.store[name] = DevObj(kind, row_layout, cl, ctx.tile, out)


@registry.register("distla.mult_rect")
def mult_rect(ctx, l_name, x_name, out_name):
    """Y = L X for a rectangular X (bg/distla/kernels.py:346-381), on the DMMA GEMM."""
    L = _need(ctx, l_name, "triangular")
    X = _need(ctx, x_name, "rectangular")
    if X.n != L.n:
        raise DimensionMismatch("X rows do not conform to L")
    Y = ctx.empty(X.data.shape)
    ctx.call("bgp_trmm_rect", _ptr(L.data), L.n, L.tile, _ptr(X.data), X.m, _ptr(Y), ctx.stream)
    ctx.store[out_name] = DevObj("rectangular", X.row_layout, X.col_layout, X.tile, Y)
for _op in ("sub", "add", "negate"):
    registry.register(_op, _op)

__all__ = ["BlockLayout", "dense_of", "diagonal_of"]

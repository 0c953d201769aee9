"""Multi-GPU sharding of the candidate grid (one process per GPU).

The grid is split into contiguous latitude slabs (lat-major flat index, so a
slab is a contiguous flat range and slab order equals global order). Every
rank stages all snapshots' captures, solves its slab with no communication,
and the only exchange is the final peak: an all-gather of each rank's exact
(value, flat index), reduced to the global maximum with the reference's
lowest-index tie-break (std::max_element). The accumulated
surface can optionally be gathered to one rank for detect_emitters, which
needs global mean/sigma and the 3x3 neighbourhoods across slab edges.

torch.distributed is the plumbing: NCCL over NVLink on GPUs, gloo in the CPU
tests (tests/test_sharding.py).
"""
from __future__ import annotations


def slab_rows(n_lat: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) owned by `rank`; balanced to within one row."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"slab_rows: bad rank {rank} of {world}")
    return rank * n_lat // world, (rank + 1) * n_lat // world


def merge_argmax(pairs):
    """Global peak from per-slab (value, global_index) pairs: the maximum value,
    lowest flat index among equal values (the first maximum wins)."""
    best = None
    for v, i in pairs:
        if i < 0:
            continue  # empty slab
        if best is None or v > best[0] or (v == best[0] and i < best[1]):
            best = (float(v), int(i))
    return best if best is not None else (0.0, 0)


def exchange_argmax(value: float, index: int, device="cpu", group=None):
    """All-gather each rank's exact peak and reduce with merge_argmax."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    v = torch.tensor([value], dtype=torch.float64, device=device)
    i = torch.tensor([index], dtype=torch.int64, device=device)
    vs = [torch.empty_like(v) for _ in range(world)]
    ix = [torch.empty_like(i) for _ in range(world)]
    dist.all_gather(vs, v, group=group)
    dist.all_gather(ix, i, group=group)
    return merge_argmax((float(a.item()), int(b.item())) for a, b in zip(vs, ix))


def gather_surface(local, sizes, dst: int = 0, group=None):
    """Concatenate per-rank slab surfaces (1-D float64 tensors of `sizes[r]`
    elements) in rank order on every rank (all_gather with padding to the
    largest slab); returns the full surface."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    m = max(sizes)
    buf = torch.zeros(m, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[r][: sizes[r]] for r in range(world)])


def geolocate_sharded(grid, states, captures, sample_rate_hz, center_freq_hz, options=None,
                      gather=True, group=None):
    """Solve the full grid across the ranks of the default process group.

    Returns (argmax_value, argmax_index, full_surface_or_None, detections) on
    every rank; detections are computed on the gathered surface (rank-local GPU).
    """
    import torch
    import torch.distributed as dist

    from . import _capi
    from .geolocate import EmitterEstimate, GeolocateOptions, geolocate_staged, StagedSnapshots
    from .geodesy import GeodeticCoord

    options = options or GeolocateOptions()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    r0, r1 = slab_rows(grid.lat.count, rank, world)
    slab = grid.slab(r0, r1)
    staged = StagedSnapshots(states, captures, sample_rate_hz, center_freq_hz, engine=grid.engine)
    local = torch.empty(max(slab.size(), 1), dtype=torch.float64, device="cuda")
    opts = GeolocateOptions(**{**options.__dict__, "detect": False})
    if slab.size() > 0:
        res = geolocate_staged(slab, staged, opts, want_surface=False,
                               accumulated_device=local.data_ptr())
        peak = (res.argmax_value, res.argmax_index)
    else:
        peak = (0.0, -1)
    value, index = exchange_argmax(peak[0], peak[1], device=local.device, group=group)
    full, dets = None, []
    if gather:
        sizes = [(slab_rows(grid.lat.count, r, world)[1] - slab_rows(grid.lat.count, r, world)[0])
                 * grid.lon.count for r in range(world)]
        full = gather_surface(local[: slab.size()], sizes, group=group)
        if options.detect:
            import ctypes as C
            cap = 4096
            out = (_capi.dg_emitter_estimate * cap)()
            n = C.c_int64()
            _capi.check(_capi.lib.dg_detect_emitters(
                grid.engine.handle, grid.handle, C.c_void_p(full.data_ptr()), 1,
                float(options.k_sigma), int(options.exclusion_radius_cells), out, cap,
                C.byref(n)))
            dets = [EmitterEstimate(GeodeticCoord(e.lat_deg, e.lon_deg, e.alt_m),
                                    int(e.grid_index), e.score, e.score_zsigma)
                    for e in out[: min(n.value, cap)]]
    return value, index, full, dets

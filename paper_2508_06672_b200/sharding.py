"""Multi-GPU sharding of a geolocation run (one process per GPU).

The work of a run is (snapshot, pair) steps, each over the whole candidate
grid, and every step is independent. Sharding the *grid* would
repeat each step's per-TDOA-bucket block moments on every GPU (a slab still
crosses almost every TDOA contour), so the run is sharded by *snapshot*:

1. rank r correlates snapshots [s0_r, s1_r) over the whole grid
   (dg_correlate_steps): geometry, block moments, candidate evaluation, exact
   refinement, pair sums, optional median scaling — no communication;
2. one all-to-all moves every per-snapshot surface to the owner of its
   latitude slab (contiguous flat range, so slab order equals global order):
   rank j receives [S][slab_j] in snapshot order;
3. rank j accumulates its slab over all S snapshots in the reference's order
   (dg_accumulate_peak), so each cell's accumulated value is bit-identical to
   the single-GPU solve, and finds the slab's exact peak;
4. the only other exchanges are the peak (all-gather of (value, flat index),
   first-maximum tie-break = std::max_element) and, for detect_emitters, the
   accumulated surface (global mean/sigma, 3x3 neighbourhoods across slabs).

torch.distributed is the plumbing: NCCL over NVLink on GPUs, gloo in the CPU
tests (tests/test_sharding.py).
"""
from __future__ import annotations


def slab_rows(n_lat: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) owned by `rank`; balanced to within one row."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"slab_rows: bad rank {rank} of {world}")
    return rank * n_lat // world, (rank + 1) * n_lat // world


def step_range(n_snapshots: int, rank: int, world: int) -> tuple[int, int]:
    """Snapshots [s0, s1) correlated by `rank`; balanced to within one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"step_range: bad rank {rank} of {world}")
    return rank * n_snapshots // world, (rank + 1) * n_snapshots // world


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
    if _host_collectives(group):
        device = "cpu"
    v = torch.tensor([value], dtype=torch.float64, device=device)
    i = torch.tensor([index], dtype=torch.int64, device=device)
    vs = [torch.empty_like(v) for _ in range(world)]
    ix = [torch.empty_like(i) for _ in range(world)]
    dist.all_gather(vs, v, group=group)
    dist.all_gather(ix, i, group=group)
    return merge_argmax((float(a.item()), int(b.item())) for a, b in zip(vs, ix))


def _host_collectives(group=None) -> bool:
    """gloo moves CPU tensors only: device tensors take a host round trip (the
    multi-process tests on one GPU); NCCL works on them in place."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def exchange_steps(local, n_snapshots: int, n_lat: int, n_lon: int, group=None):
    """All-to-all of per-snapshot surfaces: `local` is [s1-s0][n_lat*n_lon]
    (this rank's snapshots, full grid); returns [n_snapshots][slab] for this
    rank's latitude slab, snapshots in global order."""
    import torch
    import torch.distributed as dist

    if local.is_cuda and _host_collectives(group):
        return exchange_steps(local.cpu(), n_snapshots, n_lat, n_lon, group).to(local.device)

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    s0, s1 = step_range(n_snapshots, rank, world)
    if tuple(local.shape) != (s1 - s0, n_lat * n_lon):
        raise ValueError("exchange_steps: local surfaces have the wrong shape")
    cols = [tuple(c * n_lon for c in slab_rows(n_lat, j, world)) for j in range(world)]
    send = torch.cat([local[:, a:b].reshape(-1) for a, b in cols]) if local.numel() else \
        local.new_empty(0)
    send_split = [(s1 - s0) * (b - a) for a, b in cols]
    mine = cols[rank][1] - cols[rank][0]
    steps = [step_range(n_snapshots, i, world) for i in range(world)]
    recv_split = [(b - a) * mine for a, b in steps]
    recv = local.new_empty(sum(recv_split))
    dist.all_to_all_single(recv, send.contiguous(), recv_split, send_split, group=group)
    return recv.view(n_snapshots, mine)


def gather_vector(local, sizes, group=None):
    """Concatenate per-rank 1-D tensors of `sizes[r]` elements in rank order on
    every rank (all_gather with padding to the largest)."""
    import torch
    import torch.distributed as dist

    if local.is_cuda and _host_collectives(group):
        return gather_vector(local.cpu(), sizes, group).to(local.device)
    world = dist.get_world_size(group)
    m = max(max(sizes), 1)
    buf = torch.zeros(m, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[r][: sizes[r]] for r in range(world)])


gather_surface = gather_vector  # the accumulated slabs -> full surface


def geolocate_sharded(grid, staged, options=None, gather=True, group=None, stream=None,
                      profile=False):
    """Solve the full grid over the ranks of `group` (snapshot-sharded).

    `staged`: every rank's StagedSnapshots of the whole run (captures are
    small next to the surfaces). Returns (argmax_value, argmax_index,
    full_surface_or_None, detections, correlation stats of this rank) on
    every rank.
    """
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _capi
    from .geodesy import GeodeticCoord
    from .geolocate import EmitterEstimate, GeolocateOptions, accumulate_peak, correlate_steps

    options = options or GeolocateOptions()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    S = staged.shape[0]
    n_lat, n_lon = grid.lat.count, grid.lon.count
    s0, s1 = step_range(S, rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    local = torch.empty((s1 - s0, grid.size()), dtype=torch.float64, device=dev)
    med = torch.empty(max(s1 - s0, 1), dtype=torch.float64, device=dev)
    norm = bool(options.normalize_per_snapshot)
    stats = dict(n_refined=0, sum_overlap_samples=0.0, correlate_ms=0.0, moments_ms=0.0,
                 evaluate_ms=0.0, moment_ffma2=0.0, evaluate_ffma2=0.0, direct_steps=0,
                 evaluate_tc_flop=0.0,
                 kernel_launches=0, correlate_launches=0)
    if s1 > s0:
        stats = correlate_steps(grid, staged, s0, s1, local.data_ptr(),
                                med.data_ptr() if norm else None, options, stream=stream,
                                profile=profile)
    slab_all = exchange_steps(local, S, n_lat, n_lon, group=group)
    medians = None
    if norm:
        medians = gather_vector(med[: s1 - s0], [b - a for a, b in
                                                 (step_range(S, r, world) for r in range(world))],
                                group=group)
    r0, r1 = slab_rows(n_lat, rank, world)
    slab = grid.slab(r0, r1)
    acc = torch.empty(max(slab.size(), 1), dtype=torch.float64, device=dev)
    opts = GeolocateOptions(**{**options.__dict__, "detect": False})
    if slab.size() > 0:
        res = accumulate_peak(slab, staged, slab_all.data_ptr(),
                              medians.data_ptr() if medians is not None else None, opts,
                              want_surface=False, accumulated_device=acc.data_ptr(),
                              stream=stream)
        peak = (res.argmax_value, res.argmax_index)
    else:
        peak = (0.0, -1)
    value, index = exchange_argmax(peak[0], peak[1], device=dev, group=group)
    full, dets = None, []
    if gather:
        sizes = [(b - a) * n_lon for a, b in (slab_rows(n_lat, r, world) for r in range(world))]
        full = gather_vector(acc[: slab.size()], sizes, group=group)
        if options.detect:
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
    return value, index, full, dets, stats

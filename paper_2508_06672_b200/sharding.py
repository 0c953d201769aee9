"""Multi-GPU sharding of a geolocation run, one process per GPU (DESIGN.md
section 7; the same plan drives the one-process multi-GPU engine of
dg_engine_create_multi).

The work of a run is (snapshot, pair) steps, each over the whole candidate
grid, and every step is independent. Sharding the *grid* would
repeat each step's per-TDOA-bucket block moments on every GPU (a slab still
crosses almost every TDOA contour), so the run is sharded by *work unit*
(dg_shard_plan): rank r gets the whole steps [r q, (r + 1) q), q = steps //
world, and part r of each of the last steps % world steps, a cost-balanced range
of that step's TDOA buckets (the other candidates left 0). Every rank then
holds q + (steps % world) / world steps of work.

1. rank r correlates its units over the whole grid (dg_correlate_units):
   geometry, block moments, candidate evaluation, exact refinement — no
   communication;
2. one all-to-all moves every unit's columns to the owner of each latitude
   slab (contiguous flat range, so slab order equals global order);
3. rank j sums the parts of each step (exact: disjoint candidates), adds the
   pairs in the reference's order and accumulates its slab over all S
   snapshots (dg_accumulate_peak), so each accumulated value is
   bit-identical to the single-GPU solve;
4. the exact peak is two-stage: every slab's fast maximum is all-reduced, then
   each slab re-ranks its cells above the band of that global maximum, the
   same cells on every partition; the (value, index) pairs are all-gathered
   and merged with the first-maximum rule (std::max_element);
5. the accumulated slabs are gathered (every rank gets the surface) and
   rank 0 runs detect_emitters on it and broadcasts the list.

With median normalisation (geolocate.hpp:115-122) a whole snapshot's surface
is needed for its median, so units are whole snapshots (dg_correlate_steps)
and the all-to-all moves per-snapshot slabs.

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


def shard_plan(n_snapshots: int, n_receivers: int, world: int, whole_snapshots: bool = False):
    """dg_shard_plan: [(step, part, parts, rank)] of every work unit, in plan order."""
    import ctypes as C

    from . import _capi
    n = C.c_int64()
    _capi.check(_capi.lib.dg_shard_plan(int(n_snapshots), int(n_receivers), int(world),
                                        int(bool(whole_snapshots)), None, 0, C.byref(n)))
    buf = (_capi.dg_work_unit * max(n.value, 1))()
    _capi.check(_capi.lib.dg_shard_plan(int(n_snapshots), int(n_receivers), int(world),
                                        int(bool(whole_snapshots)), buf, n.value, C.byref(n)))
    return [(int(u.step), int(u.part), int(u.parts), int(u.rank)) for u in buf[:n.value]]


def exchange_units(local, plan, rank: int, world: int, n_lat: int, n_lon: int, n_rows: int,
                   group=None):
    """All-to-all of unit surfaces: `local` [n_mine][n_lat*n_lon] (this rank's units in
    plan order) -> [n_rows][slab] for this rank's latitude slab, where every unit
    is added into row `step` (parts of a step: disjoint, so the sum is exact)."""
    import torch
    import torch.distributed as dist

    if local.is_cuda and _host_collectives(group):
        return exchange_units(local.cpu(), plan, rank, world, n_lat, n_lon, n_rows,
                              group).to(local.device)
    cols = [tuple(c * n_lon for c in slab_rows(n_lat, j, world)) for j in range(world)]
    counts = [sum(1 for u in plan if u[3] == r) for r in range(world)]
    if tuple(local.shape) != (counts[rank], n_lat * n_lon):
        raise ValueError("exchange_units: local surfaces have the wrong shape")
    mine = cols[rank][1] - cols[rank][0]
    # one send buffer laid out by destination (each destination's slab columns of
    # every local unit): a strided copy per destination, no concatenation
    send = local.new_empty(counts[rank] * n_lat * n_lon)
    off, send_split = 0, []
    for a, b in cols:
        n = counts[rank] * (b - a)
        send[off:off + n].view(counts[rank], b - a).copy_(local[:, a:b])
        send_split.append(n)
        off += n
    recv_split = [counts[r] * mine for r in range(world)]
    recv = local.new_empty(sum(recv_split))
    dist.all_to_all_single(recv, send, recv_split, send_split, group=group)
    rows = torch.zeros((n_rows, mine), dtype=local.dtype, device=local.device)
    off = 0
    for r in range(world):
        for u in (u for u in plan if u[3] == r):
            rows[u[0]] += recv[off:off + mine]
            off += mine
    return rows


def geolocate_sharded(grid, staged, options=None, gather=True, group=None, stream=None,
                      profile=False):
    """Solve the full grid over the ranks of `group` (work-unit sharded).

    `staged`: every rank's StagedSnapshots of the whole run (captures are
    small next to the surfaces). Returns (argmax_value, argmax_index,
    full_surface_or_None, detections, correlation stats of this rank) on
    every rank. The engine calls, the torch ops and the collectives all run
    in order on one CUDA stream (`stream`, a raw cudaStream_t, or the current
    torch stream).
    """
    import torch

    ext = (torch.cuda.ExternalStream(stream) if stream is not None
           else torch.cuda.current_stream())
    with torch.cuda.stream(ext):
        return _geolocate_sharded(grid, staged, options, gather, group, ext.cuda_stream, profile)


def _geolocate_sharded(grid, staged, options, gather, group, stream, profile):
    import torch
    import torch.distributed as dist

    from .geolocate import (CorrelationGrid, GeolocateOptions, accumulate_peak,
                            correlate_steps, correlate_units, detect_emitters)

    options = options or GeolocateOptions()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    S, R = staged.shape[0], staged.shape[1]
    pairs = R * (R - 1) // 2
    n_lat, n_lon = grid.lat.count, grid.lon.count
    norm = bool(options.normalize_per_snapshot)
    plan = shard_plan(S, R, world, whole_snapshots=norm)
    mine = [u for u in plan if u[3] == rank]
    dev = torch.device("cuda", torch.cuda.current_device())
    local = torch.empty((len(mine), grid.size()), dtype=torch.float64, device=dev)
    med = torch.empty(max(len(mine), 1), dtype=torch.float64, device=dev)
    stats = dict(n_refined=0, sum_overlap_samples=0.0, correlate_ms=0.0, moments_ms=0.0,
                 evaluate_ms=0.0, moment_ffma2=0.0, evaluate_ffma2=0.0, direct_steps=0,
                 evaluate_tc_flop=0.0, moment_fft_flop=0.0, kernel_launches=0,
                 correlate_launches=0)
    if mine and norm:
        stats = correlate_steps(grid, staged, mine[0][0], mine[0][0] + len(mine),
                                local.data_ptr(), med.data_ptr(), options, stream=stream,
                                profile=profile)
    elif mine:
        stats = correlate_units(grid, staged, [u[:3] for u in mine], local.data_ptr(), options,
                                stream=stream, profile=profile)
    medians = None
    if norm:
        slab_all = exchange_units(local, plan, rank, world, n_lat, n_lon, S, group=group)
        sizes = [sum(1 for u in plan if u[3] == r) for r in range(world)]
        medians = gather_vector(med[: len(mine)], sizes, group=group)
    else:
        steps = exchange_units(local, plan, rank, world, n_lat, n_lon, S * pairs, group=group)
        # pairs summed in the reference's order (correlate_snapshot_all_pairs)
        steps = steps.view(S, pairs, -1)
        slab_all = steps[:, 0].clone()
        for q in range(1, pairs):
            slab_all += steps[:, q]
    del local
    r0, r1 = slab_rows(n_lat, rank, world)
    slab = grid.slab(r0, r1)
    acc = torch.empty(max(slab.size(), 1), dtype=torch.float64, device=dev)
    opts = GeolocateOptions(**{**options.__dict__, "detect": False})
    mptr = medians.data_ptr() if medians is not None else None
    fast = 0.0
    if slab.size() > 0:
        fast = accumulate_peak(slab, staged, slab_all.data_ptr(), mptr, opts, want_surface=False,
                               accumulated_device=acc.data_ptr(), stream=stream,
                               peak_stage=1).argmax_value
    m = torch.tensor([fast], dtype=torch.float64, device="cpu" if _host_collectives(group) else dev)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    peak = (0.0, -1)
    if slab.size() > 0:
        res = accumulate_peak(slab, staged, slab_all.data_ptr(), mptr, opts, want_surface=False,
                              accumulated_device=acc.data_ptr(), stream=stream, peak_stage=2,
                              peak_max=float(m.item()))
        peak = (res.argmax_value, res.argmax_index)
    value, index = exchange_argmax(peak[0], peak[1], device=dev, group=group)
    full, dets = None, []
    if gather or options.detect:
        sizes = [(b - a) * n_lon for a, b in (slab_rows(n_lat, r, world) for r in range(world))]
        full = gather_vector(acc[: slab.size()], sizes, group=group)
        if options.detect:
            torch.cuda.current_stream().synchronize()  # dg_detect_emitters: engine stream
            box = [None]
            if rank == 0:
                box[0] = detect_emitters(CorrelationGrid(grid, None), options.k_sigma,
                                         options.exclusion_radius_cells,
                                         values_device=full.data_ptr()) if full.is_cuda else \
                    detect_emitters(CorrelationGrid(grid, full.numpy()), options.k_sigma,
                                    options.exclusion_radius_cells)
            dist.broadcast_object_list(box, src=0, group=group)
            dets = box[0]
        if not gather:
            full = None
    return value, index, full, dets, stats

"""CPU, world_size 2 over gloo: the multi-GPU host logic (slab partition,
peak exchange with the reference's first-maximum tie-break, surface gather)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_06672_b200.sharding import (exchange_argmax, exchange_units, gather_surface,
                                            merge_argmax, shard_plan, slab_rows, step_range)


def test_slab_rows_partition():
    for n_lat in (1, 7, 81, 2001):
        for world in (1, 2, 3, 4, 8):
            rows = [slab_rows(n_lat, r, world) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == n_lat
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_rows(10, 2, 2)


def test_step_range_partition():
    for S in (1, 3, 10, 50, 100):
        for world in (1, 2, 3, 4, 8):
            rng = [step_range(S, r, world) for r in range(world)]
            assert rng[0][0] == 0 and rng[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))


@pytest.mark.parametrize("S,R", [(50, 2), (100, 2), (10, 3), (3, 4), (1, 2)])
def test_shard_plan_balance(S, R):
    """dg_shard_plan: every step is covered once (a whole unit, or all `world`
    parts), whole steps are contiguous per rank, and every rank holds the same
    work to within one whole step when steps >= world."""
    pairs = R * (R - 1) // 2
    steps = S * pairs
    for world in (1, 2, 3, 4, 8):
        plan = shard_plan(S, R, world)
        cover = {}
        for step, part, parts, rank in plan:
            cover.setdefault(step, []).append((part, parts, rank))
        assert sorted(cover) == list(range(steps))
        for step, c in cover.items():
            if len(c) == 1:
                assert c[0][:2] == (0, 1)
            else:
                assert sorted(p for p, _, _ in c) == list(range(world))
                assert all(n == world and p == r for p, n, r in c)
        work = [sum(1.0 / n for _, _, n, r in plan if r == k) for k in range(world)]
        assert max(work) - min(work) < 1e-9
        assert abs(sum(work) - steps) < 1e-9
        whole = shard_plan(S, R, world, whole_snapshots=True)
        assert [u[0] for u in whole] == list(range(S))
        assert all(u[3] == k for k in range(world) for u in whole
                   if step_range(S, k, world)[0] <= u[0] < step_range(S, k, world)[1])


def test_merge_argmax_tie_break():
    assert merge_argmax([(3.0, 10), (5.0, 7), (5.0, 2), (1.0, 0)]) == (5.0, 2)
    assert merge_argmax([(0.0, -1), (2.0, 9)]) == (2.0, 9)
    assert merge_argmax([(0.0, -1)]) == (0.0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # global surface with a tie between the two slabs' maxima
        n_lat, n_lon = 5, 3
        full = torch.arange(n_lat * n_lon, dtype=torch.float64) % 7
        r0, r1 = slab_rows(n_lat, rank, world)
        local = full[r0 * n_lon:r1 * n_lon].clone()
        lv, li = local.max().item(), int(torch.argmax(local).item()) + r0 * n_lon
        # torch.argmax returns the first maximum, like std::max_element
        peak = exchange_argmax(lv, li)
        sizes = [(slab_rows(n_lat, r, world)[1] - slab_rows(n_lat, r, world)[0]) * n_lon
                 for r in range(world)]
        got = gather_surface(local, sizes)
        # unit-sharded surfaces -> latitude slabs: whole steps and the disjoint
        # parts of the remainder steps sum back to every step exactly
        S = 5
        allsteps = torch.arange(S * n_lat * n_lon, dtype=torch.float64).view(S, -1) + 0.5
        plan = shard_plan(S, 2, world)
        mine = [u for u in plan if u[3] == rank]
        local = torch.zeros((len(mine), n_lat * n_lon), dtype=torch.float64)
        cells = torch.arange(n_lat * n_lon)
        for i, (step, part, parts, _) in enumerate(mine):
            keep = (cells % parts) == part
            local[i][keep] = allsteps[step][keep]
        slab = exchange_units(local, plan, rank, world, n_lat, n_lon, S)
        ok_steps = bool(torch.equal(slab, allsteps[:, r0 * n_lon:r1 * n_lon]))
        q.put((rank, peak, bool(torch.equal(got, full)) and ok_steps))
    finally:
        dist.destroy_process_group()


def test_exchange_and_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = torch.arange(15, dtype=torch.float64) % 7
    want = (6.0, 6)  # values 6 at flat 6 and 13: the first one wins across slabs
    assert full[6] == 6.0 and full[13] == 6.0
    for rank, peak, same in res:
        assert peak == want
        assert same

"""CPU, world_size 2 over gloo: the multi-GPU host logic (slab partition,
peak exchange with the reference's first-maximum tie-break, surface gather)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_06672_b200.sharding import (exchange_argmax, exchange_steps, gather_surface,
                                            merge_argmax, slab_rows, step_range)


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
        # snapshot-sharded surfaces -> latitude slabs, snapshots in order
        S = 5
        allsteps = torch.arange(S * n_lat * n_lon, dtype=torch.float64).view(S, -1)
        s0, s1 = step_range(S, rank, world)
        slab = exchange_steps(allsteps[s0:s1].clone(), S, n_lat, n_lon)
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

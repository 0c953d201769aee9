"""GPU: the snapshot-sharded multi-process solve (sharding.geolocate_sharded),
world size 2 and 3, both ranks on the one GPU of the box (gloo carries the
collectives through the host), against the 1-process solve: same accumulated
surface bit for bit, same exact peak, same detections."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2508_06672_b200 as b2
    import scenes
    from oracle.bindings import RefLib
    from paper_2508_06672_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        sc = RefLib().simulate(scenes.render(scenes.DESK_FOURJAM))
        grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
        staged = b2.StagedSnapshots(sc.states, sc.captures, sc.fs, sc.fc)
        opts = b2.GeolocateOptions(patch_peak=False)
        value, index, full, dets, _ = sharding.geolocate_sharded(grid, staged, opts)
        q.put((rank, value, index, full.cpu().numpy(), [d.grid_index for d in dets]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_processes_match_single(b2, ref, world):
    import scenes
    sc = ref.simulate(scenes.render(scenes.DESK_FOURJAM))
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    single = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc,
                                 b2.GeolocateOptions(patch_peak=False))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, value, index, full, dets in res:
        assert (value, index) == (single.argmax_value, single.argmax_index)
        assert np.array_equal(full, single.accumulated.values)
        assert dets == [d.grid_index for d in single.detections]

"""The N>1 host path on CPU: world-size-2 gloo process group (127.0.0.1), the bench's slot
sharding (contiguous ranges, no data-path collective) and its max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, slots, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2409_15097_b200 as bbm

        s0, s1 = bbm.shard_slots(slots, world, rank)
        # every rank "times" a different elapsed value; the reported one is the max
        got = bench.max_over_ranks(1.5 + rank * 2.25)
        # the bench's one-time metadata hand-over: rank 0's IPC blob reaches every rank intact
        blob = [bytes(range(256)) * 3 if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        dist.barrier()
        q.put((rank, s0, s1, got, blob[0] == bytes(range(256)) * 3))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("slots", [256, 7, 1])
def test_two_rank_sharding_and_max_over_ranks(slots):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, slots, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[3] for r in res] == [1.5 + 2.25] * world  # max over ranks, seen by every rank
    assert all(r[4] for r in res)
    ranges = [(r[1], r[2]) for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == slots
    assert ranges[0][1] == ranges[1][0]  # contiguous, disjoint, covering


def test_strong_sharding_covers_every_config_slot_once():
    """bench.py --gpus G (strong scaling): the config's B*H slots split into G contiguous ranges."""
    import bench
    import paper_2409_15097_b200 as bbm

    for name, (B, H, *_rest) in bench.CONFIGS.items():
        for world in (1, 2, 4, 8):
            ranges = [bbm.shard_slots(B * H, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == B * H, name
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:])), name
            assert max(e - s for s, e in ranges) - min(e - s for s, e in ranges) <= 1, name

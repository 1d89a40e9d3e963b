"""CPU (gloo, world size 2): the multi-process host plumbing — ring
neighbour wiring and blob exchange used by open_ring_shard / bench.py."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_08282_b200.dist import exchange_ring, ring_neighbours


def test_ring_neighbours():
    assert ring_neighbours(0, 1) == (0, 0)
    assert ring_neighbours(0, 2) == (1, 1)
    assert ring_neighbours(0, 4) == (3, 1)
    assert ring_neighbours(3, 4) == (2, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    left, right = exchange_ring(f"blob-{rank}".encode(), rank, world)
    q.put((rank, left, right))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_ring_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, left, right = q.get(timeout=120)
        res[rank] = (left, right)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        l, rt = ring_neighbours(r, world)
        assert res[r] == (f"blob-{l}".encode(), f"blob-{rt}".encode())

"""Config 5 host logic on CPU: two gloo ranks each run the streaming region's
oracle on their shard of the element range (counter-based inputs generated
per shard, as on the GPUs) and all-reduce the checksum; the gathered value
must equal the checksum of the whole range computed in one piece."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_10413_b200 import sharding

N = 100_003
COEF = np.array([k / 8 for k in range(1, 9)])


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
    from oracle import oracle as O
    lo, hi = sharding.shard_range(N, rank, world)
    n = hi - lo
    x = np.empty(n)
    y = np.empty(n)
    O.lib().orc_fill(1, O.ptr(x), n, 0x5eed01ab, lo)
    O.lib().orc_fill(1, O.ptr(y), n, 0x5eed01ac, lo)
    O.lib().orc_stream(1, n, O.ptr(x), O.ptr(y), O.ptr(COEF), 1)
    local = O.lib().orc_checksum(1, O.ptr(y), n)
    total = sharding.allreduce_checksum(local)
    q.put((rank, lo, hi, total))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_checksum_equals_whole(world):
    from oracle import oracle as O
    O.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # ranges tile [0, N) exactly
    assert res[0][1] == 0 and res[-1][2] == N
    assert all(res[i][2] == res[i + 1][1] for i in range(world - 1))
    x = np.empty(N)
    y = np.empty(N)
    O.lib().orc_fill(1, O.ptr(x), N, 0x5eed01ab, 0)
    O.lib().orc_fill(1, O.ptr(y), N, 0x5eed01ac, 0)
    O.lib().orc_stream(1, N, O.ptr(x), O.ptr(y), O.ptr(COEF), 1)
    whole = O.lib().orc_checksum(1, O.ptr(y), N)
    assert all(r[3] == whole for r in res)


def test_split_join_roundtrip():
    for c in [0, 1, (1 << 64) - 1, 0x37fbe6030960972d, 1 << 63]:
        lo, hi = sharding.split64(c)
        assert sharding.join64(lo, hi) == c
    # sums of halves recombine mod 2^64
    a, b = 0xffffffffffffffff, 0x8000000000000001
    la, ha = sharding.split64(a)
    lb, hb = sharding.split64(b)
    assert sharding.join64(la + lb, ha + hb) == (a + b) & sharding.MASK64

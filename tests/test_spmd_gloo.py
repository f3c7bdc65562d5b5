"""One-process-per-GPU exchange steps (spmd.py) over gloo with world size 2 on CPU: the
NCCL all-reduce of reduce partials and the all-gather of scan totals -> carry.  Device
work is not involved; each rank's partial comes from its block of a host array."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2406_00158_b200 import spmd

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        g = spmd.Group()
        data = (np.arange(1, 101, dtype=np.int64) * 3) - 40
        blocks = np.array_split(data, world)
        mine = blocks[rank]
        res = {}
        res["sum"] = int(spmd.allreduce_partial(np.int64(mine.sum()), "add", np.int64, g))
        res["min"] = int(spmd.allreduce_partial(np.int64(mine.min()), "minimum", np.int64, g))
        res["max_f"] = float(spmd.allreduce_partial(np.float64(mine.max()), "maximum", np.float64, g))
        res["none_sum"] = spmd.allreduce_partial(None, "add", np.float64, g)
        part = None if rank == 0 else np.float64(2.5)
        res["one_empty"] = float(spmd.allreduce_partial(part, "add", np.float64, g))
        res["totals"] = [None if t is None else int(t) for t in spmd.gather_totals(np.int64(mine.sum()), np.int64, g)]
        carry = spmd.exclusive_carry(np.int64(mine.sum()), "add", np.int64, g)
        res["carry"] = None if carry is None else int(carry)
        # scan check: local cumsum + carry == global cumsum block
        local = np.cumsum(mine) + (0 if carry is None else carry)
        res["scan_ok"] = bool(np.array_equal(local, np.cumsum(data)[sum(len(b) for b in blocks[:rank]):][:len(mine)]))
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))


def test_exchange_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    data = (np.arange(1, 101, dtype=np.int64) * 3) - 40
    for r in range(world):
        res = out[r]
        assert isinstance(res, dict), res
        assert res["sum"] == int(data.sum())
        assert res["min"] == int(data.min())
        assert res["max_f"] == float(data.max())
        assert res["none_sum"] is None
        assert res["one_empty"] == 2.5
        assert res["totals"] == [int(b.sum()) for b in np.array_split(data, world)]
        assert res["scan_ok"]
    assert out[0]["carry"] is None
    assert out[1]["carry"] == int(np.array_split(data, world)[0].sum())

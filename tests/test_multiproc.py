"""Multi-process host logic of the one-process-per-GPU path, on CPU with gloo
(world sizes 2 and 4): every rank derives its block, plan and arena layout
independently, and the pairs must agree message for message (the receiver's
entry for each send, sizes, variable order and depths — what k_pack relies on
when it writes into the neighbour's slab), plus the handle exchange and the
max-over-ranks timing reduction bench.py performs."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, grid, mode, strategy, q):
    import sys
    sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    from paper_2006_02602_b200 import capi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = capi.choose_dims(world, mode)
        ext = capi.partition(grid, dims)[rank]
        n = tuple(ext[1][a] - ext[0][a] for a in range(3))
        rank_at = capi.neighbors(dims, rank)
        plan = capi.build_plan(n, rank_at, strategy)
        node, owner = capi.center_owner(grid, dims)
        mine = {"rank": rank, "n": n, "rank_at": rank_at, "plan": plan, "owner": owner,
                "handle": bytes([rank]) * 64}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        # every send entry has exactly one matching receive entry on the neighbour
        for e in plan:
            peer = allp[e["neighbor"]]
            assert peer["rank_at"][e["face"] ^ 1] == rank
            match = [r for r in peer["plan"] if r["face"] == e["face"] ^ 1 and
                     len(r["vars"]) == len(e["vars"]) and r["vars"][0][0] == e["vars"][0][0]]
            assert len(match) == 1
            assert match[0]["vars"] == e["vars"] and match[0]["scalars"] == e["scalars"]
            assert match[0]["recv_tag"] == e["send_tag"]
        # all ranks agree on the centre owner; handles arrive intact
        assert all(p["owner"] == owner for p in allp)
        assert [p["handle"] for p in allp] == [bytes([r]) * 64 for r in range(world)]
        t = torch.tensor([1.0 + rank, 10.0 - rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.tolist() == [float(world), 10.0]
        q.put((rank, "ok"))
    except Exception as ex:  # surface the failure to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,grid,mode,strategy", [
    (2, (16, 16, 16), "1d-k", "v3"), (2, (20, 16, 16), "1d-i", "baseline"),
    (4, (24, 20, 20), "2d", "v2"), (4, (32, 32, 32), "3d", "v1")])
def test_ranks_agree_on_messages(world, grid, mode, strategy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, mode, strategy, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {r: "ok" for r in range(world)}, results


def test_bench_weak_grids():
    """bench.py's N>1 workloads follow grow_grid(256^3, N, 3d, 2) (C4)."""
    import argparse
    import bench
    args = argparse.Namespace(grid=[256], scaling="weak", mode="3d")
    assert [bench.grid_of(args, n) for n in (1, 2, 4, 8)] == [
        (256, 256, 256), (256, 256, 512), (256, 512, 512), (512, 512, 512)]
    args.scaling = "strong"
    args.grid = [512]
    assert bench.grid_of(args, 8) == (512, 512, 512)

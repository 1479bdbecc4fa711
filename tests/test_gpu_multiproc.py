"""The one-process-per-GPU path (what bench.py runs under torchrun): each
process owns one block, the exchange arenas travel as CUDA IPC handles over a
gloo group, and halos/scalars then move device-to-device with no host
staging. On a one-GPU box both processes share cuda:0 (IPC between processes
on one device), which exercises the same code; results must equal the
oracle's serial run bitwise."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, grid, dims, strategy, overlap, steps, q):
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2006_02602_b200 import capi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = rank % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        b = capi.Block(rank, world, grid, dims, strategy=strategy, overlap=overlap, device=dev,
                       timeout_ms=20000)
        handles = [None] * world
        dist.all_gather_object(handles, b.arena_ipc())
        for r in range(world):
            if r != rank:
                b.connect(r, ipc=handles[r])
        b.initialize()
        dist.barrier()
        _, checks = b.run(steps, check_every=5, want_norms=True)
        store = b.download()
        lo = b.lo
        n = b.n
        interior = store[:, 2:n[2] + 2, 2:n[1] + 2, 2:n[0] + 2].copy()
        q.put((rank, "ok", lo, interior, [(it, d.copy()) for it, d, _ in checks]))
        dist.barrier()
        b.close()
    except Exception as ex:
        q.put((rank, repr(ex), None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid,dims,strategy,overlap", [
    ((20, 14, 12), (2, 1, 1), "v3", 1), ((16, 14, 20), (1, 1, 2), "baseline", 0)])
def test_two_processes_over_cuda_ipc(grid, dims, strategy, overlap):
    import torch.multiprocessing as mp
    from oracle.refbind import Oracle
    from paper_2006_02602_b200 import capi

    steps = 20
    world = dims[0] * dims[1] * dims[2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, dims, strategy, overlap, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, status, *_ in got:
        assert status == "ok", (rank, status)
    fields = np.zeros((5, grid[2], grid[1], grid[0]))
    digits = {}
    for rank, _, lo, interior, checks in got:
        nz, ny, nx = interior.shape[1:]
        fields[:, lo[2]:lo[2] + nz, lo[1]:lo[1] + ny, lo[0]:lo[0] + nx] = interior
        for it, d in checks:
            digits.setdefault(it, []).append(d)
    want = Oracle.run_case(capi.default_config(grid=grid, steps=steps, check_every=5),
                           collect_fields=True, collect_history=True)
    np.testing.assert_array_equal(fields.view(np.uint64), want["fields"].view(np.uint64))
    # exact norms: merge the per-rank digit partials, as global_norms does
    n_glob = grid[0] * grid[1] * grid[2]
    its = sorted(digits)
    assert its == [int(x) for x in want["history_iter"]]
    for row, it in enumerate(its):
        for v in range(5):
            total = sum(int(x) << (32 * d) for part in digits[it] for d, x in enumerate(part[v].tolist()))
            value = capi._round_scaled(total, 1140) if total else 0.0
            assert np.sqrt(value / n_glob) == want["history"][row, v]

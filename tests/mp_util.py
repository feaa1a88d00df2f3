"""Process plumbing of the multi-process GPU tests.

Each test spawns one process per rank, each on its own GPU.  Ranks never
share a device: the commit's barrier kernels spin on flags that peers
write, and two such kernels of different processes on one GPU are not
guaranteed to be co-scheduled (B200_PROFILING.md: 2-4 spinning ranks on one
B200 raised Xid 109, context-switch timeout).  A test whose world exceeds
the box's GPUs is skipped (the host logic of every world size runs on the
CPU, tests/test_dist_host.py)."""

import os
import socket
import traceback

import torch


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def init_rank(rank: int, world: int, port: int, backend: str = "") -> bool:
    """Bind this process to its device and join the group; True when ranks
    share devices."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    n = torch.cuda.device_count()
    if world > n:
        raise RuntimeError("%d ranks need %d GPUs, %d visible (ranks never share a GPU)"
                           % (world, world, n))
    dev = rank
    torch.cuda.set_device(dev)
    shared = False
    backend = backend or ("gloo" if shared else "nccl")
    kw = {"device_id": torch.device("cuda", dev)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return shared


def _entry(fn, rank, world, port, q, args):
    import torch.distributed as dist
    try:
        init_rank(rank, world, port)
        q.put((rank, fn(rank, world, *args)))
    except BaseException:
        q.put((rank, "ERROR\n" + traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def need_gpus(world: int) -> None:
    """Skip the calling test unless every rank gets its own GPU."""
    import pytest
    if torch.cuda.device_count() < world:
        pytest.skip("%d ranks need %d GPUs (ranks never share a GPU)" % (world, world))


def spawn(fn, world: int, *args, timeout: float = 600.0):
    """Run fn(rank, world, *args) in `world` processes; {rank: result}.  A
    result that is a string starting with ERROR is a worker's traceback."""
    if torch.cuda.device_count() < world:
        raise RuntimeError("%d ranks need %d GPUs (ranks never share a GPU)" % (world, world))
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=timeout) for _ in procs)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return res


def failed(res) -> dict:
    return {r: v for r, v in res.items() if isinstance(v, str) and v.startswith("ERROR")}

"""Process plumbing of the multi-process GPU tests.

Each test spawns one process per rank.  With fewer GPUs than ranks the ranks
share devices round-robin (rank r on cuda:r % n): time-sliced contexts, the
same CUDA IPC / VMM peer mappings and the same data path, so the
multi-process commit is exercised on a one-GPU box too.  NCCL refuses two
ranks on one device, so shared layouts use gloo for the host handshakes
(the data path never touches the process group)."""

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
    dev = rank % n
    torch.cuda.set_device(dev)
    shared = world > n
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


def spawn(fn, world: int, *args, timeout: float = 600.0):
    """Run fn(rank, world, *args) in `world` processes; {rank: result}.  A
    result that is a string starting with ERROR is a worker's traceback."""
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

"""NVLink P2P probe (2+ GPUs, torchrun): bandwidth of the access patterns the
commit kernels can use, measured with CUDA events on each rank, max over
ranks.  Prints one JSON line per pattern.  Used to choose the combine design
(profiles/r1/p2p_probe.txt)."""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200 import _lib  # noqa: E402
from paper_2605_11215_b200.dist import PeerBuffers  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n = 64 << 20  # 256 MB of fp32
    src = torch.randn(n, device="cuda")
    dst = torch.empty(n, device="cuda")
    pb = PeerBuffers(rank, world)
    src_p = pb.share(src)
    dst_p = pb.share(dst)
    peer = (rank + 1) % world
    stream = torch.cuda.current_stream().cuda_stream

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        z.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(z) / reps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def fold_plan(in_ptr, out_ptr, variant):
        return _lib.TreePlan([(in_ptr, 0, 0, _lib.F32)], 1, [out_ptr], _lib.F32, 0.0, variant)

    res = []
    for name, in_ptr, out_ptr in [("pull", src_p[peer], dst.data_ptr()),
                                  ("push", src.data_ptr(), dst_p[peer]),
                                  ("local", src.data_ptr(), dst.data_ptr())]:
        for vname, v in (("tma", _lib.VARIANT_TMA), ("direct", _lib.VARIANT_DIRECT)):
            plan = fold_plan(in_ptr, out_ptr, v)
            ms = timeit(lambda: plan.run(0, 0, n, stream))
            res.append({"pattern": name, "variant": vname, "ms": ms,
                        "gbs_per_direction": n * 4 / ms / 1e6,
                        "note": "every rank moves 256 MB at once (both directions loaded)"})
    # the combine's shapes: fold one slice from every rank (peers over NVLink)
    # into a local output; store one local slice into every rank; both at once
    peers = [r for r in range(world) if r != rank]
    sl = n // world
    for vname, v in (("tma", _lib.VARIANT_TMA), ("direct", _lib.VARIANT_DIRECT)):
        blocks = [(src_p[r] + rank * sl * 4, r, 0, _lib.F32) for r in range(world)]
        width = 1 << max(0, (world - 1).bit_length())
        pull = _lib.TreePlan(blocks, width, [dst.data_ptr() + rank * sl * 4], _lib.F32, 0.0, v)
        ms = timeit(lambda: pull.run(0, 0, sl, stream))
        res.append({"pattern": "allgather-pull-fold", "variant": vname, "ms": ms,
                    "nvlink_in_gbs": len(peers) * sl * 4 / ms / 1e6})
        push = _lib.TreePlan([(src.data_ptr() + rank * sl * 4, 0, 0, _lib.F32)], 1,
                             [dst_p[r] + rank * sl * 4 for r in range(world)], _lib.F32, 0.0, v)
        ms = timeit(lambda: push.run(0, 0, sl, stream))
        res.append({"pattern": "push-to-all", "variant": vname, "ms": ms,
                    "nvlink_out_gbs": len(peers) * sl * 4 / ms / 1e6})
        both = _lib.TreePlan(blocks, width, [dst_p[r] + rank * sl * 4 for r in range(world)],
                             _lib.F32, 0.0, v)
        ms = timeit(lambda: both.run(0, 0, sl, stream))
        res.append({"pattern": "combine(pull-all+push-all)", "variant": vname, "ms": ms,
                    "nvlink_gbs_per_direction": len(peers) * sl * 4 / ms / 1e6})
    # copy engine
    ms = timeit(lambda: torch.cuda.current_stream().synchronize() if False else
                _lib.load().rcv_copy(dst_p[peer], src.data_ptr(), n * 4, stream))
    res.append({"pattern": "push", "variant": "copy-engine", "ms": ms,
                "gbs_per_direction": n * 4 / ms / 1e6})
    # NCCL all_reduce busBW on the same buffers (the comparison bar)
    for mb in (25, 256):
        t = torch.randn(mb * (1 << 20) // 4, device="cuda")
        ms = timeit(lambda: dist.all_reduce(t))
        s = t.numel() * 4
        res.append({"pattern": "nccl_all_reduce", "bytes": s, "ms": ms,
                    "busbw_gbs": 2 * (world - 1) / world * s / ms / 1e6})
    if rank == 0:
        for r in res:
            print(json.dumps(dict(r, world=world)))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""BASELINE configs[3]: Llama-style 1B HSDP commit (torchrun, 4 GPUs = 2-way
shard x 2 replicas; the config's 4 replicas need 8 GPUs, gpurun offers 4).

Per rank: its shard (1,235,814,400 / 2 params) of each microbatch's
gradient in bf16 (the FSDP reduce-scatter output), committed in fp32 by the
canonical engine over its replicate group (HSDPCommit); M = 32 microbatches
(G = 16 per replica), K = 20 buckets; replica 1 (both of its shard ranks)
is lost during_sync on bucket 7 in the middle of the timed region and the
quota is redistributed to the survivor.  One JSON line (rank 0).
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

D_LLAMA_1B = 1_235_814_400
TOKENS_PER_MB = 4096


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--numel", type=int, default=D_LLAMA_1B)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2605_11215_b200.dist import HSDPCommit
    shards = 2
    reps = world // shards
    g = 32 // reps
    hsdp = HSDPCommit(args.numel, shards, reps, g, 20)
    lo, hi = hsdp.bounds[hsdp.shard]
    n = hi - lo
    gen = torch.Generator(device="cuda").manual_seed(77 + hsdp.shard)
    leaves = [torch.randn(n, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(32)]
    fail_step = args.warmup + args.steps // 2

    class Kill:
        def __init__(self):
            self.t = -1

        def fire(self, phase, bucket=None):
            if self.t == fail_step and phase == "during_sync" and bucket == 7:
                return [reps - 1]
            return []

    kill = Kill()
    for t in range(args.warmup):
        kill.t = t
        hsdp.step(t, lambda m, rid: leaves[m], kill)
    torch.cuda.synchronize()
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    outs = []
    for i, t in enumerate(range(args.warmup, args.warmup + args.steps)):
        kill.t = t
        ev[i].record()
        outs.append(hsdp.step(t, lambda m, rid: leaves[m], kill))
    ev[-1].record()
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    tot = torch.tensor([sum(ms)], device="cuda")
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    committed = sum(o.contrib_total for o in outs)
    if rank == 0:
        fail_i = [i for i, o in enumerate(outs) if o.events]
        print(json.dumps({
            "config": "configs[3]: Llama-style 1B HSDP, %d-way shard x %d replicas, bf16 "
                      "microbatch shard gradients, fp32 commit, M=32, K=20, replica %d lost "
                      "during_sync:7" % (shards, reps, reps - 1),
            "numel": args.numel, "shard_numel": n, "n_gpus": world,
            "committed_tokens_per_s": committed * TOKENS_PER_MB / (total_ms / 1e3),
            "ms_per_step": total_ms / args.steps,
            "step_ms": [round(x, 3) for x in ms],
            "failure_step_ms": ms[fail_i[0]] if fail_i else None,
            "events": outs[fail_i[0]].events if fail_i else None,
            "hbm_bytes_per_rank_per_step_failure_free":
                (32 // reps) * n * 2 + n * 4 + 3 * n * 4,
        }))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

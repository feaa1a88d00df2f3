"""Debug driver for the multi-process runtime: bench-shaped steps, one at a
time, with a device sync and a status-word check after each, so a hang or a
timed-out wait is pinned to its step and phase.
  torchrun --nproc-per-node N tools/gate_debug.py NUMEL [STEPS] [FAIL_STEP]"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200.dist import DistributedGradientCommit  # noqa: E402


class Kill:
    def __init__(self, at):
        self.at, self.step = at, -1

    def fire(self, phase, bucket=None):
        if self.step == self.at and phase == "during_sync" and bucket == 7:
            return [3]
        return []


def main():
    numel = int(sys.argv[1])
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    fail = int(sys.argv[3]) if len(sys.argv) > 3 else -1
    local = int(os.environ["LOCAL_RANK"])
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev).manual_seed(1234)
    leaves = [torch.randn(numel, generator=gen, device=dev) for _ in range(32)]
    eng = DistributedGradientCommit(numel, 8, 4, 20)
    kill = Kill(fail)
    for s in range(steps):
        timing = s in (2, 3)
        if timing:
            eng.start_timing()
        kill.step = s
        t0 = time.perf_counter()
        eng.step(s, lambda m, rid: leaves[m], kill)
        torch.cuda.synchronize()
        st = int(eng.status.item())
        if timing:
            eng.drain_timing()
        print("rank %d step %d timing %d: %.1f ms status 0x%x" % (
            dist.get_rank(), s, timing, (time.perf_counter() - t0) * 1e3, st), flush=True)
        if st:
            break
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

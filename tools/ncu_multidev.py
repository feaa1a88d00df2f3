"""Single-process, 2-GPU masked all-reduce of a 1 GiB fp32 bucket through the
drop-in (the configs[2] shape) — a target for ncu: no cross-GPU spin flags,
streams are ordered with events, so kernel replay is safe."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200.comm import Communicator  # noqa: E402

n = (1 << 30) // 4
views = {r: torch.randn(n, device="cuda:%d" % r) for r in range(2)}
for _ in range(int(os.environ.get("REPS", "4"))):
    Communicator([0, 1]).ulfm_allreduce(views)
for d in range(2):
    torch.cuda.synchronize(d)
print("ok")

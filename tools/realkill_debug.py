"""Debug driver for real-kill mode (torchrun): per-rank progress to stderr."""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def log(*a):
    print("[rank %s %.2f]" % (os.environ.get("RANK"), time.time() % 1000), *a, file=sys.stderr, flush=True)

if len(sys.argv) > 1 and sys.argv[1] == "--spawn":
    # plain launcher: torchrun's agent would SIGTERM the survivors
    import subprocess
    n = int(sys.argv[2])
    ps = [subprocess.Popen([sys.executable, os.path.abspath(__file__)], env=dict(os.environ, RANK=str(r), LOCAL_RANK=str(r),
          WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT="29544")) for r in range(n)]
    for p in ps:
        try:
            p.wait(timeout=90)
        except subprocess.TimeoutExpired:
            print("rank pid", p.pid, "hung; killing", file=sys.stderr, flush=True)
            p.kill()
    print("exit codes", [p.returncode for p in ps], file=sys.stderr, flush=True)
    sys.exit(0)
local = int(os.environ["LOCAL_RANK"]); world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
from paper_2605_11215_b200.dist import DeadPeerDetector, DistributedGradientCommit, RealKill
from oracle import fold
shrink = os.environ.get("SHRINK", "0") == "1"
w, g = 2 * world, 2
b = w * g
numel = 4 * 64 * 97 + 64
host = [np.random.default_rng(900 + m).standard_normal(numel).astype(np.float32) for m in range(b)]
dev = [torch.from_numpy(h).cuda() for h in host]
want = fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b)
log("init engine")
eng = DistributedGradientCommit(numel, w, g, 4, real_kill=True, barrier_timeout_s=1.0)
log("engine ready")
inj = RealKill(1, "during_sync", 2) if rank == 1 else DeadPeerDetector(eng, shrink=shrink)
for t in range(4):
    inj.step = t
    log("step", t, "start")
    out = eng.step(t, lambda m, rid: dev[m], inj)
    log("step", t, "enqueued")
    torch.cuda.synchronize()
    ok = all(eng.grads[r].cpu().numpy().tobytes() == want.tobytes() for r in eng.comm.members if eng._holds(r))
    log("step", t, "ok", ok, out.contrib_total, out.w_cur, out.events, getattr(inj, "detections", None))
log("done")
os._exit(0)

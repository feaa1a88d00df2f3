"""HSDP training step: FSDP2 inside a replica, the fault-tolerant canonical
commit across replicas.

The paper runs ULFM on the replicate process group and NCCL on the shard
group.  Here:

* **shard group** (the GPUs of one replica): ``torch.distributed.fsdp.
  fully_shard`` over a 1-D mesh, bf16 parameters for compute
  (MixedPrecisionPolicy), fp32 sharded master parameters, and a bf16 NCCL
  reduce-scatter of every microbatch's gradient.  FSDP's gradient divide is
  switched off (``set_gradient_divide_factor(1.0)``, sum reduction): the
  divisor B of the step belongs to the commit, as in the reference
  (trainer.py:446 ``flat / B``).
* **replicate group** (one rank per replica at the same shard position):
  ``DistributedGradientCommit`` over that group.  Each microbatch's
  reduce-scattered bf16 shard gradient is pushed, in place (one segment per
  parameter shard), onto the rank's K-ACC stack (kacc.py, fp32), and the
  commit evaluates the canonical tree over the replicas' stack nodes and
  divides by B — bitwise the same result whichever replica computed which
  microbatch, so a replica's death changes nothing in the committed bits.

A replica is atomic: every shard rank of it runs the same replicated control
plane over the same failure schedule, so both compute the same microbatches
in the same order (their FSDP collectives pair up) and drop out together.

Global rank = replica * shards + shard.
"""

from __future__ import annotations

from typing import Callable, List, Optional

import torch
import torch.distributed as dist
import torch.nn as nn

from . import kacc as _kacc
from .commit import CommitOutcome
from .dist import DistributedGradientCommit


class HSDPTrainer:
    """One rank of an HSDP group of `replicas` x `shards` ranks.

    model_fn() builds the (random-initialised) model on this rank's device;
    batch_fn(t, m) returns step t's microbatch m (identical on every rank,
    a pure function of (t, m)); loss_fn(model, batch) -> scalar loss."""

    def __init__(self, model_fn: Callable[[], nn.Module], batch_fn: Callable, loss_fn: Callable,
                 shards: int, replicas: int, g_init: int, k_buckets: int, lr: float = 0.05,
                 param_dtype: torch.dtype = torch.bfloat16,
                 reduce_dtype: torch.dtype = torch.bfloat16, **engine_kw):
        from torch.distributed.device_mesh import DeviceMesh
        from torch.distributed.fsdp import MixedPrecisionPolicy, fully_shard
        rank, world = dist.get_rank(), dist.get_world_size()
        if world != shards * replicas:
            raise ValueError("world %d != %d shards x %d replicas" % (world, shards, replicas))
        self.shards, self.replicas = shards, replicas
        self.replica, self.shard = divmod(rank, shards)
        self.device = torch.device("cuda", torch.cuda.current_device())
        # every rank creates every group, in the same order
        shard_groups = [dist.new_group([r * shards + s for s in range(shards)])
                        for r in range(replicas)]
        rep_groups = [dist.new_group([r * shards + s for r in range(replicas)])
                      for s in range(shards)]
        self.shard_pg, self.rep_pg = shard_groups[self.replica], rep_groups[self.shard]
        mesh = DeviceMesh.from_group(self.shard_pg, "cuda")
        model = model_fn().to(self.device)
        mp = MixedPrecisionPolicy(param_dtype=param_dtype, reduce_dtype=reduce_dtype)
        blocks = getattr(getattr(model, "model", model), "layers", None)
        for blk in (blocks or []):
            fully_shard(blk, mesh=mesh, mp_policy=mp)
        fully_shard(model, mesh=mesh, mp_policy=mp)
        model.set_gradient_divide_factor(1.0)  # the commit divides by B
        self.model = model
        self.params = [p for p in model.parameters() if p.requires_grad]
        self.local = [p.to_local() for p in self.params]
        bad = [tuple(t.shape) for t in self.local if t.numel() % 4]
        if bad:
            raise ValueError("K-ACC needs parameter shards of whole 4-element vectors: %s" % bad[:4])
        self.numel = sum(t.numel() for t in self.local)
        self.engine = DistributedGradientCommit(self.numel, replicas, g_init, k_buckets,
                                                group=self.rep_pg, **engine_kw)
        self.pool = _kacc.SlotPool(self.numel, self.device)
        self.acc = _kacc.KAccumulator(self.pool)
        self.batch_fn, self.loss_fn, self.lr = batch_fn, loss_fn, lr
        self.b = replicas * g_init
        self.computed: List[tuple] = []
        self.capture: Optional[dict] = None  # test hook: {m: host copy of the shard leaf}

    def _shard_leaf(self) -> List[torch.Tensor]:
        segs = []
        for p in self.params:
            g = p.grad.to_local()
            segs.append(g.reshape(-1) if g.is_contiguous() else g.contiguous().reshape(-1))
        return segs

    def step(self, t: int, injector=None):
        """One optimizer step; returns (CommitOutcome, this replica's mean
        microbatch loss)."""
        self.acc.reset()
        losses = {}
        done = {}

        def leaf(m: int, rid: int):
            if rid != self.replica:
                raise RuntimeError("replica %d asked for replica %d's microbatch" % (self.replica, rid))
            if m not in done:
                for p in self.params:
                    p.grad = None
                loss = self.loss_fn(self.model, self.batch_fn(t, m))
                loss.backward()
                segs = self._shard_leaf()
                if self.capture is not None:
                    self.capture[m] = torch.cat([s.float() for s in segs]).cpu()
                self.acc.push(m, segs)
                losses[m] = loss.detach().float()
                done[m] = _kacc.Pending(self.acc, m)
                self.computed.append((t, m))
            return done[m]

        out: CommitOutcome = self.engine.step(t, leaf, injector)
        # per-microbatch losses of this replica's computations (the run's
        # committed loss is the fold over all replicas' admitted ones)
        self.last_losses = {m: float(v) for m, v in losses.items()
                            if m in out.admitted.get(self.replica, ())}
        for p in self.params:
            p.grad = None
        loss = float("nan")
        if self.replica in self.engine.comm.members:
            grad = self.engine.grads[self.replica]
            off = 0
            with torch.no_grad():
                for t_local in self.local:
                    n = t_local.numel()
                    t_local.sub_(grad[off:off + n].view_as(t_local), alpha=self.lr)
                    off += n
            # this replica's share of the committed loss (a fixed left fold
            # over the microbatches it admitted; informational)
            mine = sorted(m for m in losses if m in out.admitted.get(self.replica, ()))
            tot = torch.zeros((), dtype=torch.float64, device=self.device)
            for m in mine:
                tot = tot + losses[m].double()
            loss = float(tot) / max(1, len(mine))
        return out, loss

    @property
    def grad(self) -> torch.Tensor:
        return self.engine.grads[self.replica]

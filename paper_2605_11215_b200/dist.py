"""Multi-process canonical commit: one process per GPU over NVLink P2P.

The control plane (membership, epoch, roles, quotas, the whole step state
machine of ``GradientCommit``) runs replicated on every rank: it is a pure
function of the shared failure schedule, so every rank reaches the same
decisions without exchanging a byte — the reference's agreement property
(comm.py:1-9) by construction, as in its simulator.  Only the data plane
crosses GPUs:

1. *local pre-reduce* — each rank folds the canonical-tree nodes whose
   microbatch gradients all live on it into its slot of a partial pool
   (rcv_tree_commit, HBM-bound, no NVLink);
2. *flag barrier* among the live ranks (rcv_barrier: release/acquire flags in
   IPC-shared memory, every wait bounded by %globaltimer);
3. *combine* — each live rank owns one 64-element-aligned slice of the
   bucket: it reads every cover node's partial slice (peers' over NVLink),
   evaluates the top of the canonical tree, divides by B and stores the
   slice into the primary replica buffer of every live rank (peers' over
   NVLink) — reduce-scatter and all-gather fused in one launch;
4. *local broadcast* — after the next barrier each rank copies the bucket
   from its primary replica into its other replicas (HBM), so NVLink carries
   one copy per rank, not one per replica.

Partial pools are double-buffered by call parity, so one barrier per bucket
suffices (a rank passing barrier k+1 has finished combine k); one more
barrier closes the step.  Dead replicas' microbatches are not in the cover,
so their memory is never read; a rank whose replicas all died stops taking
part in barriers and launches.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import torch
import torch.distributed as dist

from . import _lib
from .comm import Communicator
from .commit import GradientCommit, aligned_bounds, block_cover
from .policy import assign_roles, initial_state, policy_advancement


def owner_slice(n: int, q: int, nr: int, align: int = 64):
    """[a, z) of a bucket of n elements owned by the q-th of nr live ranks:
    contiguous, align-element granular, covering [0, n) exactly."""
    units = (n + align - 1) // align
    return (min(n, units * q // nr * align), min(n, units * (q + 1) // nr * align))


def plan_bucket(owner: Dict[int, int], n_leaves: int, live_ranks: Sequence[int],
                pool_slots: int):
    """Host plan of one bucket commit, identical on every rank.

    owner maps each admitted microbatch index to the rank holding its
    gradient.  Returns (cover, slot_of) where cover is the list of canonical
    tree nodes (lo, level) pre-reduced locally and slot_of maps each node to
    (producing rank, pool slot).  Raises if a rank needs more slots."""
    cover = block_cover(owner, n_leaves)
    slot_of: Dict[tuple, tuple] = {}
    used: Dict[int, int] = {}
    for blo, blev in cover:
        rk = owner[min(m for m in owner if blo <= m < blo + (1 << blev))]
        if rk not in live_ranks:
            raise RuntimeError("microbatch owned by a dead rank %d" % rk)
        j = used.get(rk, 0)
        if j >= pool_slots:
            raise RuntimeError("partial pool exhausted (%d slots)" % pool_slots)
        used[rk] = j + 1
        slot_of[(blo, blev)] = (rk, j)
    return cover, slot_of


class PeerBuffers:
    """Exchange CUDA IPC handles of one buffer per rank; returns every
    rank's device pointer to it, valid in this process."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def share(self, t: torch.Tensor) -> List[int]:
        h, off = _lib.ipc_export(t)
        got: List[Optional[tuple]] = [None] * self.world
        dist.all_gather_object(got, (h, off), group=self.group)
        return [t.data_ptr() if r == self.rank else _lib.ipc_import(hh, oo)
                for r, (hh, oo) in enumerate(got)]


class DistributedGradientCommit(GradientCommit):
    """``GradientCommit`` with replicas spread over the ranks of a process
    group, (w_init + spares) / world consecutive replicas per rank."""

    def __init__(self, numel: int, w_init: int, g_init: int, k_buckets: int,
                 rank: Optional[int] = None, world: Optional[int] = None,
                 group=None, dtype: torch.dtype = torch.float32,
                 policy_kind: str = "static", spares: int = 0,
                 variant: int = _lib.VARIANT_AUTO,
                 combine_variant: int = _lib.VARIANT_AUTO,
                 pool_slots: int = 8, barrier_timeout_s: float = 30.0):
        if policy_kind not in ("static", "adaptive"):
            raise ValueError("unknown policy kind %r" % (policy_kind,))
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        members = list(range(w_init + spares))
        if len(members) % self.world:
            raise ValueError("%d replicas do not split over %d ranks" % (len(members), self.world))
        per = len(members) // self.world
        self.rank_of = {r: r // per for r in members}
        self.state = initial_state(w_init, g_init)
        if spares:
            self.state = policy_advancement(self.state, w_cur=len(members))
        self.comm = Communicator(members, assign_roles(self.state, members))
        self.policy_kind = policy_kind
        self.numel = numel
        self.bounds = aligned_bounds(numel, k_buckets)
        self.dtype = dtype
        self.variant = variant
        self.combine_variant = combine_variant
        self.alive = {r: True for r in members}
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.placement = {r: self.device for r in members if self.rank_of[r] == self.rank}
        self.timing: Optional[list] = None
        self._code = {torch.float32: _lib.F32, torch.float64: _lib.F64}[dtype]
        self._es = torch.tensor([], dtype=dtype).element_size()

        local = [r for r in members if self.rank_of[r] == self.rank]
        store = torch.zeros(per * numel, dtype=dtype, device=self.device)
        self.grads = {r: store[i * numel:(i + 1) * numel] for i, r in enumerate(local)}
        self.lmax = max(hi - lo for lo, hi in self.bounds)
        self.pool_slots = pool_slots
        self.pool = torch.empty(2 * pool_slots * self.lmax, dtype=dtype, device=self.device)
        self.flags = torch.zeros(64, dtype=torch.int64, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.timeout_ns = int(barrier_timeout_s * 1e9)
        pb = PeerBuffers(self.rank, self.world, group)
        store_ptr = pb.share(store)
        self.grad_ptr = {r: store_ptr[self.rank_of[r]] + (r % per) * numel * self._es
                         for r in members}
        self.pool_ptr = pb.share(self.pool)
        self.flag_ptr = pb.share(self.flags)
        self._seq = 0
        self._calls = 0
        self._pending = None  # (lo, hi) of the last combined bucket to broadcast locally
        self._plan_cache = None
        # pre-reduce stream: bucket k+1's HBM-bound pre-reduce overlaps bucket
        # k's NVLink-bound combine on the caller's stream
        self.pstream = torch.cuda.Stream(self.device)
        self._set_free = [None, None]   # event: pool set reusable (all peers done)
        self._in_step = False
        self.barriers = 0  # barrier kernels launched (for launch accounting)
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)

    # ---- hooks of GradientCommit.step ----

    def _holds(self, rid: int) -> bool:
        return self.rank_of[rid] == self.rank

    def _live_ranks(self) -> List[int]:
        return sorted({self.rank_of[r] for r in self.comm.members})

    def _primary(self, rank: int) -> Optional[int]:
        """Lowest live replica on `rank`: the one the combine stores into."""
        return next((r for r in self.comm.members if self.rank_of[r] == rank), None)

    def _flush_broadcast(self) -> None:
        """Copy the last combined bucket from this rank's primary replica to
        its other live replicas (HBM only).  Runs after a barrier, so every
        peer's stores into the primary have landed."""
        if self._pending is None:
            return
        lo, hi = self._pending
        self._pending = None
        mine = [r for r in self.comm.members if self._holds(r)]
        if len(mine) < 2:
            return
        src = self.grads[mine[0]][lo:hi]
        outs = [self.grads[r][lo:hi] for r in mine[1:]]
        self._timed_launch("broadcast", (1 + len(outs)) * (hi - lo) * self._es,
                           lambda: _lib.fold([src], [0], outs, variant=self.variant))

    def _barrier(self) -> None:
        ranks = self._live_ranks()
        if self.rank not in ranks or len(ranks) < 2:
            self._flush_broadcast()
            return
        self._seq += 1
        self.barriers += 1
        mask = 0
        for r in ranks:
            mask |= 1 << r
        self._timed_launch("barrier", 0, lambda: _lib.barrier(
            self.flags, self.flag_ptr, self.rank, mask, self._seq,
            self.timeout_ns, self.status))
        self._flush_broadcast()

    def _end_of_step(self) -> None:
        self._barrier()
        self._in_step = False
        self._set_free = [None, None]

    def check_peers(self) -> None:
        """Raise if any barrier so far timed out on a peer (reads the device
        status word: a host sync, so callers do it off the hot path)."""
        bad = int(self.status.item())
        if bad:
            raise RuntimeError("peer ranks timed out in the commit barrier: mask 0x%x" % bad)

    def _pool_at(self, rank: int, set_idx: int, slot: int, elem: int) -> int:
        return self.pool_ptr[rank] + ((set_idx * self.pool_slots + slot) * self.lmax + elem) * self._es

    def _timed_launch(self, kind: str, nbytes: int, launch, nvlink=(0, 0)) -> None:
        """Launch; with timing on, bracket it with CUDA events and record
        its algorithmic HBM bytes and NVLink (in, out) bytes."""
        if self.timing is None:
            launch()
            return
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch()
        z.record()
        self.timing.append((a, z, nbytes, kind, nvlink))

    def _dist_plan(self, leaves):
        """Per leaf set (cached): the local pre-reduce plans, the combine
        plan over every cover node's pool slot, and NVLink byte counts."""
        members = tuple(self.comm.members)
        cached = self._plan_cache
        if cached is not None and cached[0] is leaves and cached[1] == members:
            return cached[2]
        b = self.state.b
        ranks = self._live_ranks()
        owner = {m: self.rank_of[rid] for m, (rid, _) in leaves.items()}
        cover, slot_of = plan_bucket(owner, b, ranks, self.pool_slots)
        pre = []
        for blo, blev in cover:
            rk, j = slot_of[(blo, blev)]
            if rk != self.rank:
                continue
            span = [m for m in sorted(leaves) if blo <= m < blo + (1 << blev)]
            sub = [(leaves[m][1].data_ptr(), m - blo, 0, self._code) for m in span]
            dst = self.pool_ptr[self.rank] + j * self.lmax * self._es
            pre.append((_lib.TreePlan(sub, 1 << blev, [dst], self._code, 0.0, self.variant),
                        len(sub)))
        combine = None
        if self.rank in ranks:
            blocks = [(self.pool_ptr[rk] + j * self.lmax * self._es, blo, blev, self._code)
                      for (blo, blev), (rk, j) in sorted(slot_of.items())]
            prim = [self._primary(rk) for rk in ranks]
            outs = [self.grad_ptr[r] for r in prim]
            combine = (_lib.TreePlan(blocks, b, outs, self._code, float(b), self.combine_variant),
                       sum(1 for rk, _ in slot_of.values() if rk != self.rank),
                       sum(1 for r in prim if not self._holds(r)), len(blocks), len(outs))
        plan = (pre, combine, ranks)
        self._plan_cache = (leaves, members, plan)
        return plan

    def _reduce_bucket(self, k: int, leaves) -> int:
        lo, hi = self.bounds[k]
        n = hi - lo
        if n == 0:
            return 0
        if not leaves:
            for r in self.comm.members:
                if self._holds(r):
                    _lib.zero_(self.grads[r][lo:hi])
            return 1
        pre, combine, ranks = self._dist_plan(leaves)
        sidx = self._calls % 2
        set_off = sidx * self.pool_slots * self.lmax
        self._calls += 1
        main = torch.cuda.current_stream(self.device)
        stream = main.cuda_stream
        if not self._in_step:
            # the leaves were produced on the caller's stream
            self._in_step = True
            self.pstream.wait_stream(main)
        if self._set_free[sidx] is not None:
            self.pstream.wait_event(self._set_free[sidx])
        with torch.cuda.stream(self.pstream):
            for tp, n_leaf in pre:
                self._timed_launch("prereduce", (n_leaf + 1) * n * self._es,
                                   lambda: tp.run(lo, set_off, n, self.pstream.cuda_stream))
        ready = torch.cuda.Event()
        ready.record(self.pstream)
        main.wait_event(ready)
        self._barrier()
        # every live peer passed this barrier after its previous combine, so
        # the other pool set (read by that combine) may be overwritten
        free = torch.cuda.Event()
        free.record(main)
        self._set_free[1 - sidx] = free
        launches = len(pre)
        if combine is not None:
            tp, r_in, r_out, n_in, n_out = combine
            a, z = owner_slice(n, ranks.index(self.rank), len(ranks))
            if z > a:
                sl = (z - a) * self._es
                local = (n_in - r_in) + (n_out - r_out)
                self._timed_launch("combine", local * sl,
                                   lambda: tp.run(set_off + a, lo + a, z - a, stream),
                                   nvlink=(r_in * sl, r_out * sl))
                launches += 1
        self._pending = (lo, hi)
        return launches

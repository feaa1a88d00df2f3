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
4. *local broadcast* — two barriers later each rank copies the bucket
   from its primary replica into its other replicas (HBM), so NVLink carries
   one copy per rank, not one per replica.

Barriers run on their own stream, barrier k behind this rank's combine k-2
(so it overlaps combine k-1), and partial pools rotate through four sets by
call index, so one barrier per bucket suffices (a rank passing barrier k has
finished pre-reduce k and combine k-2) and the pre-reduce stream may run a
bucket ahead of the barriers; one more barrier closes the step.  Pre-reduces run on a side stream, so bucket k+1's
HBM-bound pre-reduce overlaps bucket k's NVLink-bound combine.  The whole
per-bucket schedule lives in the native runtime (rcv_ctx / rcv_plan in
librcv.so): a plan is prepared once per leaf cover and each bucket costs the
host one call.  Dead replicas' microbatches are not in the cover, so their
memory is never read; a rank whose replicas all died stops taking part in
barriers and launches.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import ctypes
import os
import time

import torch
import torch.distributed as dist

from . import _lib
from .comm import Communicator
from .commit import GradientCommit, aligned_bounds, block_cover, input_nodes
from .policy import assign_roles, initial_state, policy_advancement


# per-rank flag words in peer memory: [0, 64) the barrier sequence written by
# each peer, [64, 67) this rank's pool-set integrity stamps (include/rcv.h)
FLAG_SLOTS = 128


class CommitIntegrityError(RuntimeError):
    """A combine read a pool partial whose stamp was not its call's, or that
    was invalidated while it was being read, or a barrier peer timed out
    outside real-kill mode: the committed bits of that step are not to be
    trusted (never silently committed)."""


def owner_slice(n: int, q: int, nr: int, align: int = 64):
    """[a, z) of a bucket of n elements owned by the q-th of nr live ranks:
    contiguous, align-element granular, covering [0, n) exactly.  Equal
    slices: every owner reads every cover node's partial, so the combine's
    work per element is the same on every owner (NVLink-direction-balanced
    unequal slices measured slower: profiles/r1/slice_weights.txt)."""
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


class VmmBuffers:
    """Shared buffers for real-kill mode: cuMem VMM allocations exported as
    POSIX file descriptors, passed to every peer over a Unix socket
    (SCM_RIGHTS) and mapped there.  An importer's mapping holds a reference
    on the physical memory, so a dead peer's buffers never become invalid
    addresses for the survivors.

    The abstract socket is visible to every local process, so the server
    hands the descriptor only to a peer whose SO_PEERCRED pid is one of the
    group's and which presents the job's secret (exchanged over the process
    group); accept, connect and receive are bounded by `timeout_s`."""

    def __init__(self, rank: int, world: int, group=None, timeout_s: float = 60.0):
        import secrets
        self.rank, self.world, self.group = rank, world, group
        self.timeout_s = timeout_s
        got = [None] * world
        mine = (secrets.token_hex(4), secrets.token_hex(16)) if rank == 0 else None
        dist.all_gather_object(got, (os.getpid(), mine), group=group)
        self.pids = {pid for pid, _ in got}
        self.job, secret = got[0][1]
        self.secret = secret.encode()
        self.dev = torch.cuda.current_device()
        self._keep = []  # fds and tensors that must outlive the mappings

    def _serve(self, srv, fd, errors) -> None:
        import socket
        import struct
        served = 0
        try:
            while served < self.world - 1:
                conn, _ = srv.accept()
                with conn:
                    conn.settimeout(self.timeout_s)
                    cred = conn.getsockopt(socket.SOL_SOCKET, socket.SO_PEERCRED,
                                           struct.calcsize("3i"))
                    pid, uid, _ = struct.unpack("3i", cred)
                    if pid not in self.pids or uid != os.getuid():
                        continue  # not a rank of this group: refuse
                    if conn.recv(len(self.secret)) != self.secret:
                        continue
                    socket.send_fds(conn, [b"f"], [fd])
                    served += 1
        except Exception as exc:  # surfaced by share()
            errors.append(exc)

    def broadcast_fd(self, fd: Optional[int], root: int = 0) -> int:
        """Hand rank `root`'s descriptor `fd` to every other rank (the same
        peer checks as share()); returns this rank's descriptor of it."""
        import socket
        import threading
        name = "\0rcv-%s-b%d-%d" % (self.job, root, len(self._keep))
        if self.rank == root:
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(name)
            srv.listen(self.world)
            srv.settimeout(self.timeout_s)
            errors: List[Exception] = []
            th = threading.Thread(target=self._serve, args=(srv, fd, errors), daemon=True)
            th.start()
        dist.barrier(group=self.group)  # the root listens before anyone connects
        if self.rank == root:
            th.join(timeout=self.timeout_s)
            srv.close()
            if errors or th.is_alive():
                raise RuntimeError("descriptor broadcast failed: %r" % (errors or "timeout"))
            self._keep.append((fd, None))
            return fd
        c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        c.settimeout(self.timeout_s)
        c.connect(name)
        c.sendall(self.secret)
        _, fds, _, _ = socket.recv_fds(c, 1, 1)
        c.close()
        if not fds:
            raise RuntimeError("rank %d refused its descriptor" % root)
        self._keep.append((fds[0], None))
        return fds[0]

    def share(self, nbytes: int, dtype: torch.dtype):
        """Allocate nbytes here; returns (local tensor, [ptr of every rank])."""
        import socket
        import threading
        ptr, size, fd = _lib.vmm_alloc(nbytes)
        name = "\0rcv-%s-%d-%d"
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name % (self.job, self.rank, len(self._keep)))
        srv.listen(self.world)
        srv.settimeout(self.timeout_s)
        errors: List[Exception] = []
        th = threading.Thread(target=self._serve, args=(srv, fd, errors), daemon=True)
        th.start()
        meta = [None] * self.world
        dist.all_gather_object(meta, (size, self.dev), group=self.group)
        ptrs = []
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(ptr)
                continue
            c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            c.settimeout(self.timeout_s)
            c.connect(name % (self.job, r, len(self._keep)))
            c.sendall(self.secret)
            _, fds, _, _ = socket.recv_fds(c, 1, 1)
            c.close()
            if not fds:
                raise RuntimeError("rank %d refused its VMM descriptor" % r)
            ptrs.append(_lib.vmm_import(fds[0], meta[r][0], meta[r][1]))
            os.close(fds[0])
        th.join(timeout=self.timeout_s)
        srv.close()
        if errors or th.is_alive():
            raise RuntimeError("VMM descriptor exchange failed: %r" % (errors or "timeout"))
        es = torch.tensor([], dtype=dtype).element_size()
        local = _lib.tensor_at(ptr, nbytes // es, dtype, torch.device("cuda", self.dev))
        self._keep.append((fd, local))
        return local, ptrs


class DeadPeerDetector:
    """Injector for real-kill mode on the survivors: they are not told the
    schedule; they find out, at the protocol's poll points, which ranks the
    hardware saw die — the crash-stop detection and agreement of
    comm.py:129-172 driven by the machine instead of the simulator.

    With the engine's node liveness (``rcv_liveness``: native heartbeats in
    shared memory, a dead word every GPU's barrier kernel reads), a poll is
    one host read and a compare-and-swap: poll point n of the replicated
    control flow is decided by the first rank that reaches it, and every
    survivor acts on that same failed set (``Liveness.decide``).  No device
    synchronisation, so it polls before every bucket's collective
    ("during_sync", trainer.py:425) as well as at before_sync / after_sync.

    Without liveness it falls back to the barrier timeout: a poll
    synchronises the device and reads the status word (only at
    before/after_sync unless per_bucket=True, since each poll serialises
    the bucket pipeline).

    shrink=True re-forms the torch process group without the dead ranks
    (ncclCommShrink via torch.distributed.shrink_group), timed."""

    def __init__(self, engine: "DistributedGradientCommit", inner=None, shrink: bool = False,
                 per_bucket: Optional[bool] = None):
        self.engine, self.inner, self.shrink = engine, inner, shrink
        lv = getattr(engine, "liveness", None)
        self.per_bucket = lv is not None if per_bucket is None else per_bucket
        self.known = 0
        self.seq = 0
        self.detections: List[dict] = []
        self.shrinker = None

    def fire(self, phase, bucket=None):
        import time
        out = list(self.inner.fire(phase, bucket)) if self.inner is not None else []
        polls = ("after_sync", "before_sync", "during_sync") if self.per_bucket else \
            ("after_sync", "before_sync")
        if phase not in polls:
            return out
        t0 = time.perf_counter()
        lv = getattr(self.engine, "liveness", None)
        rec = {}
        if lv is not None:
            self.seq += 1
            mask, decided_ns = lv.decide(self.seq)
            bits = mask & ~self.known
            if bits:
                rec["poll"] = self.seq
                rec["decided_ns"] = decided_ns
        else:
            torch.cuda.synchronize(self.engine.device)
            bits = int(self.engine.status[0].item()) & ~self.known
        if bits:
            self.known |= bits
            dead_ranks = [r for r in range(self.engine.world) if (bits >> r) & 1]
            victims = [rid for rid in self.engine.comm.members
                       if self.engine.rank_of[rid] in dead_ranks]
            rec.update(phase=phase, bucket=bucket, ranks=dead_ranks, replicas=victims,
                       poll_ms=(time.perf_counter() - t0) * 1e3)
            if lv is not None:
                st = lv.stats(dead_ranks[0])
                rec.update(dead_ns=st["dead_ns"], kill_ns=st["kill_ns"], seen_ns=st["now_ns"])
                if st["kill_ns"] and st["dead_ns"]:
                    rec["detect_ms"] = (st["dead_ns"] - st["kill_ns"]) / 1e6
                if st["dead_ns"] and rec.get("decided_ns"):
                    rec["agree_ms"] = max(0, rec["decided_ns"] - st["dead_ns"]) / 1e6
            if self.shrink and hasattr(dist, "shrink_group"):
                # NCCL is off the commit's data path: re-form the torch group
                # in the background, timed, while the step recovers
                import threading

                def shrink(rec=rec, ranks=list(dead_ranks)):
                    t1 = time.perf_counter()
                    try:
                        dist.shrink_group(ranks)
                        rec["shrink_ms"] = (time.perf_counter() - t1) * 1e3
                    except Exception as exc:  # reported, not fatal
                        rec["shrink_error"] = repr(exc)[:200]
                self.shrinker = threading.Thread(target=shrink, daemon=True)
                self.shrinker.start()
            self.detections.append(rec)
            out += victims
        return out


class RealKill:
    """Victim-side injector: at (step, phase, bucket) this process dies by
    SIGKILL (the paper's failure simulator) — at once, with
    its queued and running kernels, unless drain_s > 0 asks it to finish its
    GPU work first.  Survivors never read a dead rank's memory after the
    agreed detection; what it left half-written before is re-reduced (every
    bucket tagged before the failure is stale)."""

    def __init__(self, step: int, phase: str, bucket=None, drain_s: float = 0.0,
                 liveness=None):
        self.at = (step, phase, bucket)
        self.step = -1
        self.drain_s = drain_s
        self.liveness = liveness

    def fire(self, phase, bucket=None):
        if (self.step, phase, bucket if phase == "during_sync" else None) == self.at:
            import signal
            import time
            if self.drain_s > 0:
                torch.cuda.synchronize()
                time.sleep(self.drain_s)
            if self.liveness is not None:
                self.liveness.note_kill()
            os.kill(os.getpid(), signal.SIGKILL)
        return []


class DistributedGradientCommit(GradientCommit):
    """``GradientCommit`` with replicas spread over the ranks of a process
    group, (w_init + spares) / world consecutive replicas per rank."""

    def __init__(self, numel: int, w_init: int, g_init: int, k_buckets: int,
                 rank: Optional[int] = None, world: Optional[int] = None,
                 group=None, dtype: torch.dtype = torch.float32,
                 policy_kind: str = "static", spares: int = 0,
                 variant: int = _lib.VARIANT_AUTO,
                 combine_variant: int = _lib.VARIANT_AUTO,
                 pool_slots: int = 8, barrier_timeout_s: float = 30.0,
                 real_kill: bool = False, liveness_deadline_s: Optional[float] = 10e-3,
                 liveness_period_s: float = 1e-3, multicast: Optional[bool] = None):
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
        self.recovery_events: Optional[list] = None
        self._code = {torch.float32: _lib.F32, torch.float64: _lib.F64}[dtype]
        self._es = torch.tensor([], dtype=dtype).element_size()

        local = [r for r in members if self.rank_of[r] == self.rank]
        self.lmax = max(hi - lo for lo, hi in self.bounds)
        self.pool_slots = pool_slots
        self.real_kill = real_kill
        # [0] peers that timed out in a barrier, [1] pool-stamp mismatches
        self.status = torch.zeros(2, dtype=torch.int32, device=self.device)
        # each step's status words are copied to pinned memory behind the
        # step and checked when the next step ends (no host sync on the path)
        self._status_host = torch.zeros(2, dtype=torch.int32, pin_memory=True)
        self._status_ev: Optional[torch.cuda.Event] = None
        self.integrity_errors = 0
        # RCV_TIMEOUT_S overrides every bounded wait (debugging hangs)
        self.timeout_ns = int(float(os.environ.get("RCV_TIMEOUT_S", barrier_timeout_s)) * 1e9)
        # NVLS multicast all-gather (RCV_MC=1 or multicast=True): the combine
        # stores each owner slice once, through a multicast object bound to
        # every rank's landing slot (its first replica buffer), instead of
        # once per live peer.  Not in real-kill mode (a dead team member's
        # binding is left alone there).
        if multicast is None:
            multicast = os.environ.get("RCV_MC", "0") not in ("", "0")
        self.multicast = bool(multicast) and not real_kill and self.world > 1
        self.mc_ptr: Optional[int] = None
        self._slot = numel  # elements from one replica buffer to the next
        if self.multicast:
            gran = _lib.mc_granularity(self.world)
            self._slot = -(-numel * self._es // gran) * gran // self._es
        if real_kill or self.multicast:
            # VMM memory: survivors' mappings outlive a dead exporter, and a
            # multicast object binds only shareable allocations
            vb = VmmBuffers(self.rank, self.world, group)
            self._shared = vb
            store, store_ptr = vb.share(per * self._slot * self._es, dtype)
            store.zero_()
        if real_kill:
            self.pool, self.pool_ptr = vb.share(_lib.pool_sets() * pool_slots * self.lmax * self._es, dtype)
            self.flags, self.flag_ptr = vb.share(FLAG_SLOTS * 8, torch.int64)
            self.flags.zero_()
        else:
            if not self.multicast:
                store = torch.zeros(per * numel, dtype=dtype, device=self.device)
            self.pool = torch.empty(_lib.pool_sets() * pool_slots * self.lmax, dtype=dtype,
                                        device=self.device)
            self.flags = torch.zeros(FLAG_SLOTS, dtype=torch.int64, device=self.device)
            pb = PeerBuffers(self.rank, self.world, group)
            if not self.multicast:
                store_ptr = pb.share(store)
            self.pool_ptr = pb.share(self.pool)
            self.flag_ptr = pb.share(self.flags)
        sl = self._slot
        self.grads = {r: store[i * sl:i * sl + numel] for i, r in enumerate(local)}
        self.grad_ptr = {r: store_ptr[self.rank_of[r]] + (r % per) * sl * self._es
                         for r in members}
        self._landing = local[0]
        if self.multicast:
            self._mc_setup(store_ptr[self.rank], group)
        self.rt = _lib.BucketRuntime(self.world, self.rank, self.flags, self.flag_ptr,
                                     self.status, self.timeout_ns)
        self.liveness: Optional[_lib.Liveness] = None
        if real_kill and liveness_deadline_s:
            # node-local heartbeats: a dead peer is declared within the
            # deadline and every barrier kernel stops waiting for it at once
            self.liveness = _lib.Liveness("/rcv-live-%s" % vb.job, self.rank, self.world,
                                          liveness_period_s, liveness_deadline_s)
            dist.barrier(group=group)
            if self.rank == 0:  # every rank has it mapped: drop the name
                try:
                    os.unlink("/dev/shm/rcv-live-%s" % vb.job)
                except OSError:
                    pass
            self.rt.set_liveness(self.liveness)
        self._plan_key = None
        self._stream: Optional[int] = None
        # host seconds spent building/looking up plans, enqueueing buckets and
        # waiting for the previous step's status words (bench.py reports them)
        self.host_prof = {"plan_s": 0.0, "bucket_s": 0.0, "wait_s": 0.0}
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)

    def _mc_setup(self, landing_ptr: int, group) -> None:
        """Rank 0 creates the multicast object and hands its descriptor to
        the others; every rank adds its GPU, then (after all have) binds its
        landing slot and maps the object (include/rcv.h, rcv_mc_*)."""
        vb = self._shared
        nbytes = self._slot * self._es
        fd = None
        if self.rank == 0:
            h, size, fd = _lib.mc_create(nbytes, self.world)
        fd = vb.broadcast_fd(fd)
        if self.rank != 0:
            h, size = _lib.mc_import(fd), nbytes
        _lib.mc_add_device(h)
        dist.barrier(group=group)
        _lib.mc_bind(h, landing_ptr, size)
        dist.barrier(group=group)
        self.mc_ptr = _lib.mc_map(h, size)
        self._mc = (h, size)

    # ---- hooks of GradientCommit.step ----

    def _holds(self, rid: int) -> bool:
        return self.rank_of[rid] == self.rank

    def _canonical_ranges(self, counts: List[Tuple[int, int]]) -> Dict[int, List[int]]:
        """Pack each rank's microbatch count into aligned dyadic blocks.

        A rank's leaves enter the commit as the maximal aligned tree nodes
        it owns whole (block_cover), and every owner slice of the combine
        reads every node's partial, so the combine's NVLink bytes grow with
        the cover size.  Contiguous ranges fragment once per-rank counts stop
        being powers of two (10/5/10/7 after a death at N=4: 11 nodes).
        Decomposing each count into its binary digits and placing the blocks
        largest first (buddy order: every start is a multiple of the block
        size, and the packing stays within [0, sum)) reaches sum of
        popcounts (9 there).  Absent leaves past the sum and the per-node
        leaf cap can favour the contiguous layout for large counts, so the
        smaller cover of the two is kept.  The committed bits do not change:
        the canonical tree depends only on the leaf values."""
        key = tuple(counts)
        memo = self.__dict__.setdefault("_ranges_memo", {})
        if key not in memo:
            packed = self._dyadic_ranges(counts)
            plain = GradientCommit._canonical_ranges(self, counts)
            total = sum(q for _, q in counts)

            def nodes(ranges):
                owner = {i: self.rank_of[r] for r, ids in ranges.items() for i in ids}
                return len(block_cover(owner, max(1, total))) if owner else 0
            memo[key] = packed if nodes(packed) < nodes(plain) else plain
        return {r: list(v) for r, v in memo[key].items()}

    def _dyadic_ranges(self, counts: List[Tuple[int, int]]) -> Dict[int, List[int]]:
        per_rank: Dict[int, List[Tuple[int, int]]] = {}
        for rid, q in counts:
            per_rank.setdefault(self.rank_of[rid], []).append((rid, q))
        blocks = []
        for rk, lst in per_rank.items():
            c = sum(q for _, q in lst)
            blocks += [(1 << bit, rk) for bit in range(c.bit_length()) if (c >> bit) & 1]
        blocks.sort(key=lambda x: (-x[0], x[1]))
        ids: Dict[int, List[int]] = {rk: [] for rk in per_rank}
        pos = 0
        for size, rk in blocks:
            ids[rk].extend(range(pos, pos + size))
            pos += size
        ranges: Dict[int, List[int]] = {}
        for rk, lst in per_rank.items():
            k = 0
            for rid, q in lst:
                ranges[rid] = ids[rk][k:k + q]
                k += q
        return ranges

    def _stream_device(self) -> torch.device:
        return self.device

    def _live_ranks(self) -> List[int]:
        return sorted({self.rank_of[r] for r in self.comm.members})

    def _primary(self, rank: int) -> Optional[int]:
        """Lowest live replica on `rank`: the one the combine stores into."""
        return next((r for r in self.comm.members if self.rank_of[r] == rank), None)

    def _live_mask(self):
        ranks = self._live_ranks()
        mask = 0
        for r in ranks:
            mask |= 1 << r
        return ranks, mask

    def _sync_point(self, phase: str) -> None:
        """Real-kill mode, before the after_sync poll: one barrier over the
        live ranks behind the step's last combine, then wait for the device.
        A rank that died with this step's data plane in flight is then seen
        dead by every survivor's device (liveness word or timeout) before the
        protocol decides the step, so its death is decided here at the
        latest and every bucket reduced before it is re-reduced (stale);
        a death the protocol has not decided by now cannot have touched this
        step's data (the rank arrived here after its last combine)."""
        if not self.real_kill or phase != "after_sync":
            return
        ranks, mask = self._live_mask()
        self.rt.poll(mask, self.rank in ranks, torch.cuda.current_stream(self.device).cuda_stream)
        torch.cuda.synchronize(self.device)

    def _end_of_step(self) -> None:
        ranks, mask = self._live_mask()
        stream = torch.cuda.current_stream(self.device)
        self._stream = None  # looked up again at the next step's first bucket
        self.rt.finish(mask, self.rank in ranks, stream.cuda_stream)
        # the previous step's snapshot is complete by now (a step ago);
        # check it, then snapshot this step's words behind its last kernel
        if self._status_ev is not None:
            h0 = time.perf_counter()
            self._status_ev.synchronize()
            self.host_prof["wait_s"] += time.perf_counter() - h0
            self._judge(self._status_host.tolist(), "a previous step")
        self._status_host.copy_(self.status, non_blocking=True)
        self._status_ev = torch.cuda.Event()
        self._status_ev.record(stream)

    def _judge(self, words, when: str) -> None:
        dead, err = int(words[0]) & 0xffffffff, int(words[1]) & 0xffffffff
        if err:
            self.integrity_errors += 1
        if self.real_kill:
            # a peer's death is detected and recovered by the protocol; a
            # combine around it may see a stale stamp, and its bucket is
            # re-reduced over the survivors
            return
        if err:
            raise CommitIntegrityError(
                "rank %d: a combine in %s read a pool partial with a wrong or invalidated "
                "stamp (status 0x%x): the committed gradient is not trustworthy"
                % (self.rank, when, err))
        if dead:
            raise CommitIntegrityError(
                "rank %d: peer ranks 0x%x timed out in a commit barrier in %s (not in "
                "real-kill mode): their partials may have been read unsynchronised"
                % (self.rank, dead, when))

    def check_peers(self) -> None:
        """Raise if any barrier so far timed out on a peer or any combine
        read a partial with a wrong stamp (reads the device status words: a
        host sync, so callers do it off the hot path)."""
        self._judge(self.status.tolist(), "this run")

    def start_timing(self) -> None:
        self.rt.set_timing(True)

    def drain_timing(self):
        """[(kind, ms, hbm_bytes, nvlink_in, nvlink_out)] of every launch
        since start_timing (call after synchronising)."""
        out = self.rt.timings()
        self.rt.set_timing(False)
        return out

    def _set_plan(self, leaves, layout=None) -> None:
        """Build the native plan of a leaf set: local pre-reduce nodes, the
        combine over every cover node's pool slot, the local broadcast."""
        b = self.state.b
        ranks, mask = self._live_mask()
        owner = {m: self.rank_of[rid] for m, (rid, _) in leaves.items()}
        cover, slot_of = plan_bucket(owner, b, ranks, self.pool_slots)
        Block = _lib._Block
        nodes = input_nodes({m: v for m, v in leaves.items() if v[1] is not None})
        pre_blocks, pre_counts, pre_leaves, pre_out = [], [], [], []
        for blo, blev in cover:
            rk, j = slot_of[(blo, blev)]
            if rk != self.rank:
                continue
            span = [n for n in nodes if blo <= n[0] < blo + (1 << blev)]
            pre_blocks += [Block(t.data_ptr(), lo - blo, lev, _lib.dtype_code(t))
                           for lo, lev, t in span]
            pre_counts.append(len(span))
            pre_leaves.append(1 << blev)
            pre_out.append(self.pool_ptr[self.rank] + j * self.lmax * self._es)
        comb = [Block(self.pool_ptr[rk] + j * self.lmax * self._es, blo, blev, self._code)
                for (blo, blev), (rk, j) in sorted(slot_of.items())]
        prim = [self._primary(rk) for rk in ranks]
        mine = [r for r in self.comm.members if self._holds(r)]
        part = self.rank in ranks
        if self.multicast:
            # one multicast store per vector lands in every rank's landing
            # slot (its first replica buffer, live or not); the local
            # broadcast copies it to the rank's other live replicas
            comb_out, n_remote_out = [self.mc_ptr], 1
            src = self._landing if mine else None
            bcast = [r for r in mine if r != self._landing]
        else:
            comb_out = [self.grad_ptr[r] for r in prim]
            n_remote_out = sum(1 for r in prim if not self._holds(r))
            src = mine[0] if mine else None
            bcast = mine[1:]

        def arr(ctype, xs):
            return (ctype * max(1, len(xs)))(*xs)
        keep = dict(pre_blocks=arr(Block, pre_blocks), pre_counts=arr(ctypes.c_int, pre_counts),
                    pre_leaves=arr(ctypes.c_uint32, pre_leaves),
                    pre_out=arr(ctypes.c_void_p, pre_out), comb=arr(Block, comb),
                    comb_out=arr(ctypes.c_void_p, comb_out),
                    bcast_out=arr(ctypes.c_void_p, [self.grads[r].data_ptr() for r in bcast]),
                    comb_rank=arr(ctypes.c_int, [rk for _, (rk, _) in sorted(slot_of.items())]))
        d = _lib.PlanDesc(
            n_pre=len(pre_counts), pre_blocks=keep["pre_blocks"], pre_counts=keep["pre_counts"],
            pre_leaves=keep["pre_leaves"], pre_out=keep["pre_out"],
            set_stride=self.pool_slots * self.lmax,
            n_comb=len(comb) if part else 0, comb_blocks=keep["comb"],
            comb_rank=keep["comb_rank"], n_leaves=b,
            n_comb_out=len(comb_out), comb_out=keep["comb_out"],
            slice_q=ranks.index(self.rank) if part else 0, slice_nr=len(ranks),
            n_bcast=len(bcast) if src is not None else 0,
            bcast_src=self.grads[src].data_ptr() if src is not None else None,
            bcast_out=keep["bcast_out"], acc_dtype=self._code, divisor=float(b),
            variant=self.variant, comb_variant=self.combine_variant,
            live_mask=mask, participate=int(part),
            remote_in=sum(1 for rk, _ in slot_of.values() if rk != self.rank),
            remote_out=n_remote_out,
            guarded=int(self.real_kill), comb_out_mc=int(self.multicast))
        self.rt.set_plan(d, keep, layout)

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
        key = (id(leaves), tuple(self.comm.members))
        if self._plan_key is None or self._plan_key[0] != key or self._plan_key[1] is not leaves:
            h0 = time.perf_counter()
            # the native plan depends only on the leaf layout: which rank
            # holds which microbatch at which address, and the membership
            layout = (tuple(self.comm.members), self.state.b,
                      tuple((m, rid) + _value_key(v) for m, (rid, v) in sorted(leaves.items())))
            if not self.rt.use_cached(layout):
                self._set_plan(leaves, layout)
            self._plan_key = (key, leaves)
            self.host_prof["plan_s"] += time.perf_counter() - h0
        if self._stream is None:
            self._stream = torch.cuda.current_stream(self.device).cuda_stream
        h0 = time.perf_counter()
        self.rt.bucket(lo, n, self._stream)
        self.host_prof["bucket_s"] += time.perf_counter() - h0
        return 1


def _value_key(v) -> tuple:
    """What a native plan captures of one leaf value: its address and dtype
    (a microbatch gradient) or its subtree and address (a K-ACC node)."""
    if v is None:
        return ()
    if isinstance(v, torch.Tensor):
        return (v.data_ptr(), v.dtype)
    return (v.lo, v.level, v.tensor.data_ptr(), v.tensor.dtype)


def shard_bounds(numel: int, shards: int, align: int = 64):
    """Contiguous shard ranges of a flat gradient, cuts on align elements."""
    base = (numel // shards) // align * align
    return [(i * base, numel if i == shards - 1 else (i + 1) * base) for i in range(shards)]


class HSDPCommit:
    """Hybrid-sharded data parallel: every replica spans `shards` GPUs (the
    intra-replica shard group, where FSDP reduce-scatters each microbatch's
    gradient), and the fault-tolerant canonical commit runs per shard
    position over the replicate group of that position (PAPER.md:677-691:
    ULFM on replicate_pg, NCCL on shard_pg).  A replica is atomic: a death
    removes it from every shard position's group at the same logical point,
    because every rank replays the same schedule.

    Global rank = replica * shards + shard.  leaf(m, rid) returns this
    rank's shard of microbatch m's gradient (bf16 or fp32; accumulation is
    fp32)."""

    def __init__(self, numel: int, shards: int, w_init: int, g_init: int,
                 k_buckets: int, spares: int = 0, **kw):
        rank, world = dist.get_rank(), dist.get_world_size()
        n_rep = w_init + spares
        if world != shards * n_rep:
            raise ValueError("world %d != %d shards x %d replicas" % (world, shards, n_rep))
        self.shards = shards
        self.replica, self.shard = divmod(rank, shards)
        groups = [dist.new_group([r * shards + s for r in range(n_rep)]) for s in range(shards)]
        self.bounds = shard_bounds(numel, shards)
        lo, hi = self.bounds[self.shard]
        self.engine = DistributedGradientCommit(hi - lo, w_init, g_init, k_buckets,
                                                group=groups[self.shard], spares=spares, **kw)

    @property
    def grad(self) -> torch.Tensor:
        """This rank's committed shard gradient (its replica's)."""
        return self.engine.grads[self.replica]

    def step(self, t: int, leaf, injector=None):
        return self.engine.step(t, leaf, injector)

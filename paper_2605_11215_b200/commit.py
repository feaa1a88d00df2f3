"""Canonical-order gradient commit engine (the B200 design of the north star).

One optimizer step of a data-parallel replica group: B = W_init * G_init
microbatches are committed exactly once each, in canonical microbatch-index
order, whatever the failures.  Compared with the drop-in ``run_iteration``
(which reproduces the reference's in-place buffers bit for bit), the engine
changes only the data plane:

* **Canonical addressing.**  Step microbatch indices 0..B-1 are handed out
  by the quota policy (majors G, the minor R; ``policy.py``): in contiguous
  ranges, ascending replica id (``_canonical_ranges``; the multi-process
  engine packs each rank's share into aligned dyadic blocks instead).  A spare shadows a counterpart (major-spares
  the highest-id majors, the minor-spare the minor); on promotion it admits
  the vacated replica's range.  In a boundary extension the survivors take
  the orphaned indices (those no live replica admitted), smallest first.
  Per-replica counts, roles, events and counters are exactly the reference's
  (trainer.py:324-487); only *which* example a count refers to changes
  (SURVEY §7.3 R2).
* **Fused commit.**  The committed gradient of every bucket is the canonical
  dyadic tree over the admitted microbatch gradients divided by B, evaluated
  by one rcv_tree_commit launch that reads the microbatch gradients directly
  (accumulation fused into the reduce) and writes every live replica's
  output view.  Because the tree depends only on the leaf values, the result
  is bitwise independent of which replica computed which microbatch — so a
  failure run commits exactly the failure-free gradient.
* **Out of place.**  Inputs are never written by the commit, so the
  reference's pre-reduce snapshot (buckets.py:61-69) is only an epoch tag,
  a rewind is a no-op, and a stale bucket is recovered by re-running the
  launch over the repaired membership.  A dead replica's
  buffers are never read: its microbatches drop out of the leaf set.
* **Committed buckets survive.**  A bucket whose data phase already ran in
  this step over the same microbatch index set holds the canonical tree of
  the same leaf values, so its re-reduce (the second pass after a
  boundary) keeps the protocol call and its accounting but launches
  nothing: only the work the dead replica had not committed is redone
  (north star).  Off in real-kill mode, where a guarded combine may have
  skipped itself, and with RCV_REUSE=0.

Leaves come from a caller-supplied ``leaf(m, rid)`` returning the 1-D CUDA
gradient of microbatch m as computed on replica rid (in the bench: synthetic
per-index gradients resident in HBM).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

import torch

from . import _lib
from .comm import (Communicator, ReplicaRole, SPARE_FOR, SPARE_ROLES,
                   WorkResult, WorkStatus, designate_boundary_minors)
from .policy import (InvariantViolation, PolicyState, adaptive_policy_adjustment,
                     assign_roles, initial_state, policy_adjustment,
                     policy_advancement)
from .trainer import AFTER_SYNC, BEFORE_SYNC, DURING_SYNC, AllReplicasDead, NullInjector

ALIGN = 64  # bucket cuts on 256-byte boundaries: 16-byte vectors, whole sectors


def aligned_bounds(numel: int, k: int, align: int = ALIGN) -> List[Tuple[int, int]]:
    """K contiguous buckets, cuts rounded down to ``align`` elements, the
    last takes the rest (the reference's d//K split, buckets.py:44-58,
    moved onto vector boundaries)."""
    if k < 1:
        raise ValueError("bucket count must be >= 1")
    base = (numel // k) // align * align
    return [(i * base, numel if i == k - 1 else (i + 1) * base) for i in range(k)]


def _height(n: int) -> int:
    return max(0, (n - 1).bit_length())


def block_cover(owner: Dict[int, object], n_leaves: int,
                max_leaves: int = _lib.MAX_IN) -> List[Tuple[int, int]]:
    """Maximal aligned dyadic nodes (lo, level) of the canonical tree whose
    present leaves all sit on one device (``owner`` maps index -> device)
    and number at most ``max_leaves``.  Each node's partial is computed
    locally; the cover is then combined in tree order."""
    out: List[Tuple[int, int]] = []
    present = sorted(owner)

    def visit(level: int, lo: int) -> None:
        hi = lo + (1 << level)
        inside = [m for m in present if lo <= m < hi]
        if not inside:
            return
        if len({owner[m] for m in inside}) == 1 and len(inside) <= max_leaves:
            out.append((lo, level))
            return
        visit(level - 1, lo)
        visit(level - 1, lo + (1 << (level - 1)))

    visit(_height(n_leaves), 0)
    return out


def input_nodes(leaves) -> List[Tuple[int, int, torch.Tensor]]:
    """The commit's inputs, ascending: (lo, level, tensor) per distinct
    canonical-tree node of a leaf set {m: (rid, value)} whose values are
    microbatch gradients (the node (m, 0)) or K-ACC nodes (kacc.KNode: a
    complete subtree, shared by every index it covers)."""
    seen, out = set(), []
    for m in sorted(leaves):
        v = leaves[m][1]
        if isinstance(v, torch.Tensor):
            out.append((m, 0, v))
        elif id(v) not in seen:
            seen.add(id(v))
            out.append((v.lo, v.level, v.tensor))
    return out


@dataclass
class CommitOutcome:
    """Mirror of IterationOutcome (trainer.py:232-252) for the engine."""
    step: int
    contributions: Dict[int, int]
    contrib_total: int
    contrib_regular: int
    contrib_boundary: int
    final_epoch: int
    w_cur: int
    roles: Dict[int, str]
    state: PolicyState
    events: List[dict] = field(default_factory=list)
    admitted: Dict[int, List[int]] = field(default_factory=dict)
    bucket_epochs: List[Optional[int]] = field(default_factory=list)
    rounds: int = 0
    passes: int = 0
    reduces: int = 0
    rewinds: int = 0
    boundary_crossed: bool = False
    launches: int = 0
    failure_wall_s: Optional[float] = None  # host wall from first FAILURE to commit
    reform_host_s: float = 0.0  # host time in the failure handling (repair, policy, roles)


class GradientCommit:
    """Replica group + quota policy + fused canonical commit.

    ``placement`` maps replica id -> CUDA device (default all on cuda:0);
    ``grads[rid]`` is replica rid's committed-gradient buffer (its p.grad).
    """

    def __init__(self, numel: int, w_init: int, g_init: int, k_buckets: int,
                 placement: Optional[Dict[int, object]] = None,
                 dtype: torch.dtype = torch.float32, policy_kind: str = "static",
                 spares: int = 0, variant: int = _lib.VARIANT_AUTO):
        if policy_kind not in ("static", "adaptive"):
            raise ValueError("unknown policy kind %r" % (policy_kind,))
        members = list(range(w_init + spares))
        self.state = initial_state(w_init, g_init)
        if spares:
            self.state = policy_advancement(self.state, w_cur=len(members))
        self.comm = Communicator(members, assign_roles(self.state, members))
        self.policy_kind = policy_kind
        self.numel = numel
        self.bounds = aligned_bounds(numel, k_buckets)
        self.placement = {r: torch.device(placement[r]) if placement else torch.device("cuda:0")
                          for r in members}
        self.dtype = dtype
        self.variant = variant
        self.alive = {r: True for r in members}
        self.grads = {r: torch.empty(numel, dtype=dtype, device=self.placement[r])
                      for r in members}
        self._scratch: Dict[torch.device, List[torch.Tensor]] = {}
        self._plan_cache = None
        # optional launch timing: list of (start_event, end_event, algo_bytes, kind)
        self.timing: Optional[list] = None
        # optional recovery trace: [(name, CUDA event, host time)] marks
        self.recovery_events: Optional[list] = None
        _lib.enable_peer_access(sorted({d.index for d in self.placement.values()}))

    # ---- data plane ----

    def _reuse_committed(self) -> bool:
        """Whether a bucket committed earlier in the step over the same leaf
        index set may keep its outputs instead of being relaunched."""
        return os.environ.get("RCV_REUSE", "1") not in ("", "0") and \
            not getattr(self, "real_kill", False)

    def _holds(self, rid: int) -> bool:
        """Whether this process holds replica rid's buffers (all of them in
        single-process mode; the distributed engine overrides)."""
        return True

    def _canonical_ranges(self, counts: List[Tuple[int, int]]) -> Dict[int, List[int]]:
        """Canonical microbatch indices of each replica, given its quota
        (members in ascending id order): contiguous ranges, ascending id.
        Any partition of [0, sum) commits the same bits; subclasses pick one
        that suits their data placement."""
        ranges: Dict[int, List[int]] = {}
        pos = 0
        for rid, q in counts:
            ranges[rid] = list(range(pos, pos + q))
            pos += q
        return ranges

    def _end_of_step(self) -> None:
        """Hook run after the last bucket of a step is committed."""

    def _sync_point(self, phase: str) -> None:
        """Hook run before the injector's poll at `phase` (the multi-process
        real-kill engine synchronises its data plane before after_sync)."""

    def _stream_device(self) -> torch.device:
        """Device whose current stream carries the commit's tail."""
        return self.placement[self.comm.members[0]] if self.comm.members else \
            next(iter(self.placement.values()))

    def mark(self, name: str) -> None:
        """Record a named CUDA event on the commit stream (recovery trace:
        'fail' at the first FAILURE, 'commit' after the step's last kernel;
        callers add their own, e.g. around recomputed microbatches)."""
        if self.recovery_events is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self._stream_device()))
        self.recovery_events.append((name, ev, time.perf_counter()))

    def _scratch_buf(self, dev: torch.device, i: int) -> torch.Tensor:
        """Full-length partial buffer i on dev (multi-device covers only):
        bucket k's partial lives at the bucket's own offset, so partials and
        leaves share one pointer offset per bucket."""
        pool = self._scratch.setdefault(dev, [])
        while len(pool) <= i:
            pool.append(torch.empty(self.numel, dtype=torch.float32 if self.dtype == torch.bfloat16
                                    else self.dtype, device=dev))
        return pool[i]

    def _plan_for(self, leaves: Dict[int, Tuple[int, torch.Tensor]]):
        """Launch plan of a leaf set (cached while the set is unchanged):
        prebuilt pointer arrays, so each bucket is one or two cheap calls."""
        members = tuple(self.comm.members)
        cached = self._plan_cache
        if cached is not None and cached[0] is leaves and cached[1] == members:
            return cached[2]
        b = self.state.b
        acc = _lib.dtype_code(self.grads[members[0]])
        outs = [self.grads[r] for r in members]
        owner = {m: self.placement[rid] for m, (rid, _) in leaves.items()}
        cover = block_cover(owner, b)
        nodes = input_nodes(leaves)
        pre = []
        if len(cover) == 1:
            # every present leaf on one device: one fused launch per bucket
            ins = [(t.data_ptr(), lo, lev, _lib.dtype_code(t)) for lo, lev, t in nodes]
            top_dev = owner[min(leaves)]
        else:
            ins, used = [], {}
            for blo, blev in cover:
                sub = [n for n in nodes if blo <= n[0] < blo + (1 << blev)]
                dev = owner[sub[0][0]]
                if len(sub) == 1:
                    lo, lev, t = sub[0]
                    ins.append((t.data_ptr(), lo, lev, _lib.dtype_code(t)))
                    continue
                buf = self._scratch_buf(dev, used.get(dev, 0))
                used[dev] = used.get(dev, 0) + 1
                pre.append((dev, _lib.TreePlan(
                    [(t.data_ptr(), lo - blo, lev, _lib.dtype_code(t)) for lo, lev, t in sub],
                    1 << blev, [buf.data_ptr()], acc, 0.0, self.variant)))
                ins.append((buf.data_ptr(), blo, blev, acc))
            top_dev = self.placement[members[0]]
        top = _lib.TreePlan(ins, b, [o.data_ptr() for o in outs], acc, float(b), self.variant)
        others = sorted({o.device for o in outs} | {d for d, _ in pre} | set(owner.values()),
                        key=lambda d: d.index)
        plan = (pre, top, top_dev, [d for d in others if d != top_dev], len(ins), len(outs))
        self._plan_cache = (leaves, members, plan)
        return plan

    def _reduce_bucket(self, k: int, leaves: Dict[int, Tuple[int, torch.Tensor]]) -> int:
        """Commit bucket k from ``leaves`` {m: (rid, tensor)}; returns launches."""
        lo, hi = self.bounds[k]
        n = hi - lo
        if n == 0:
            return 0
        if not leaves:
            for r in self.comm.members:
                _lib.zero_(self.grads[r][lo:hi])
            return len(self.comm.members)
        pre, top, top_dev, others, n_in, n_out = self._plan_for(leaves)
        for dev, tp in pre:
            tp.run(lo, lo, n, torch.cuda.current_stream(dev).cuda_stream)
        es = self.grads[self.comm.members[0]].element_size()
        self._on_device(top_dev, others, lambda: self._timed(
            (n_in + n_out) * n * es,
            lambda: top.run(lo, lo, n, torch.cuda.current_stream(top_dev).cuda_stream)))
        return len(pre) + 1

    def _timed(self, nbytes: int, launch) -> None:
        """Run a fused launch, bracketing it with CUDA events on its stream
        when timing is on; nbytes = every input and output once."""
        if self.timing is None:
            launch()
            return
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch()
        z.record()
        self.timing.append((a, z, nbytes, "fused", (0, 0)))

    def start_timing(self) -> None:
        """Record every fused launch from now on (CUDA events on its stream)."""
        self.timing = []

    def drain_timing(self):
        """[(kind, ms, hbm_bytes, nvlink_in, nvlink_out)] per launch since
        start_timing (call after synchronising); stops recording."""
        out = [(kind, a.elapsed_time(z), nb, nin, nout)
               for a, z, nb, kind, (nin, nout) in (self.timing or [])]
        self.timing = None
        return out

    def _on_device(self, dev, others, launch) -> None:
        """Run ``launch`` on dev's current stream, ordered after the other
        devices' streams (inputs / previous readers) and before them."""
        if not others:
            launch()
            return
        s = torch.cuda.current_stream(dev)
        for d in others:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(d))
            s.wait_event(ev)
        with torch.cuda.device(dev):
            launch()
        ev = torch.cuda.Event()
        ev.record(s)
        for d in others:
            torch.cuda.current_stream(d).wait_event(ev)

    # ---- one step (control flow of trainer.py:324-487) ----

    def step(self, t: int, leaf: Callable[[int, int], torch.Tensor],
             injector=None) -> CommitOutcome:
        inj = injector if injector is not None else NullInjector()
        comm, state, b = self.comm, self.state, self.state.b

        ver = [0]  # bumped whenever admissions, roles or membership change

        def kill(victims):
            if victims:
                ver[0] += 1
            for rid in victims:
                if self.alive.get(rid):
                    self.alive[rid] = False
                    comm.mark_dead(rid)

        kill(inj.fire(BEFORE_SYNC))
        if not any(self.alive[r] for r in comm.members):
            raise AllReplicasDead("no replica survives step %d" % t)
        comm.reset_iteration()

        # canonical ranges (contributor quota) and spare shadows
        counts = []
        for rid in comm.members:
            role = comm.roles[rid]
            counts.append((rid, state.g_cur if role is ReplicaRole.MAJOR else (
                state.r_cur if role is ReplicaRole.MINOR else 0)))
        ranges = self._canonical_ranges(counts)
        cur_range = {r: list(v) for r, v in ranges.items()}
        majors = [r for r in comm.members if comm.roles[r] is ReplicaRole.MAJOR]
        minors = [r for r in comm.members if comm.roles[r] is ReplicaRole.MINOR]
        shadow: Dict[int, int] = {}
        for rid in comm.members:
            role = comm.roles[rid]
            if role is ReplicaRole.MAJOR_SPARE and majors:
                shadow[rid] = majors.pop()
            elif role is ReplicaRole.MINOR_SPARE and minors:
                shadow[rid] = minors[0]

        role_now: Dict[int, ReplicaRole] = {}
        rem_reg: Dict[int, int] = {}
        rem_ext: Dict[int, int] = {}
        admitted: Dict[int, List[int]] = {}
        provisional: Dict[int, List[int]] = {}
        for rid in comm.members:
            if not self.alive[rid]:
                continue
            role = comm.roles[rid]
            role_now[rid] = role
            runs_g = role in (ReplicaRole.MAJOR, ReplicaRole.MAJOR_SPARE)
            rem_reg[rid] = state.g_cur if runs_g else state.r_cur
            rem_ext[rid] = 0
            admitted[rid], provisional[rid] = [], []
        reg_cursor = {rid: 0 for rid in rem_reg}

        tags: Dict[int, int] = {}
        reduced: Dict[int, Optional[int]] = {}
        restore = "skip"
        p_major, m = state.g_cur, 0
        cnt = dict(rounds=0, passes=0, reduces=0, rewinds=0, launches=0)
        events: List[dict] = []
        crossed = False
        after_fired = False
        touched = set()
        t_fail: Optional[float] = None
        reform_s = 0.0

        def live():
            return [r for r in comm.members if self.alive[r]]

        def execute(rid: int) -> None:
            if rem_reg[rid] > 0:
                rem_reg[rid] -= 1
                j = reg_cursor[rid]
                reg_cursor[rid] += 1
                if role_now[rid] in SPARE_ROLES:
                    src = shadow.get(rid)
                    if src is not None and j < len(ranges[src]):
                        provisional[rid].append(ranges[src][j])
                    else:
                        provisional[rid].append(-1)   # nothing to shadow
                elif j < len(ranges[rid]):
                    admitted[rid].append(ranges[rid][j])
                    ver[0] += 1
                    comm.contrib_regular[rid] += 1
                # else: executed and zeroed (trainer.py:229)
            elif rem_ext[rid] > 0:
                rem_ext[rid] -= 1
                taken = {i for r in comm.members if r in admitted for i in admitted[r]}
                nxt = next(i for i in range(b) if i not in taken)
                admitted[rid].append(nxt)
                ver[0] += 1
                comm.contrib_boundary[rid] += 1

        leaf_cache: list = [None, None, None]

        def collect() -> Dict[int, Tuple[int, torch.Tensor]]:
            # the leaf set changes only when admissions, roles or membership
            # do (each bumps ver); reuse the dict (and with it the launch
            # plan) otherwise
            key = (comm.epoch, comm.boundary_latch, ver[0], len(comm.members))
            if leaf_cache[0] == key:
                return leaf_cache[1]
            lv: Dict[int, Tuple[int, torch.Tensor]] = {}
            for rid in comm.members:
                if comm.roles[rid] in SPARE_ROLES and not comm.boundary_latch:
                    continue      # virtual zeroing: spare work never enters
                for i in admitted.get(rid, ()):
                    lv[i] = (rid, leaf(i, rid) if self._holds(rid) else None)
            # K-ACC leaves resolve to their stack node once every admitted
            # microbatch of this leaf set has been pushed
            for i, (rid, v) in lv.items():
                if hasattr(v, "resolve"):
                    lv[i] = (rid, v.resolve())
            leaf_cache[0], leaf_cache[1], leaf_cache[2] = key, lv, frozenset(lv)
            return lv

        committed_keys: Dict[int, frozenset] = {}
        reuse = self._reuse_committed()

        def reduce(k: int) -> WorkResult:
            def data():
                lv = collect()
                keys = leaf_cache[2]
                if reuse and committed_keys.get(k) == keys:
                    return  # same index set, same leaf bits: already committed
                cnt["launches"] += self._reduce_bucket(k, lv)
                committed_keys[k] = keys
            return comm.ulfm_collective(data)

        def on_failure(work: WorkResult) -> None:
            nonlocal p_major, crossed, restore, t_fail, reform_s
            h0 = time.perf_counter()
            ver[0] += 1
            if t_fail is None:
                t_fail = h0
                self.mark("fail")
            rec = work.record
            # promoted spares admit the vacated replica's range (canonical R2)
            vacating = [r for r in sorted(rec.failed_replicas)
                        if roles_before.get(r) in SPARE_FOR]
            for (rid, new_role), dead in zip(rec.promotions, vacating):
                # the vacated replica's current range: a spare promoted
                # earlier in this step holds the range it took over
                cur_range[rid] = list(cur_range.get(dead, []))
                admitted[rid].extend(cur_range[rid])
                comm.contrib_regular[rid] += len(provisional[rid])
                provisional[rid] = []
                role_now[rid] = new_role
            if self.policy_kind == "adaptive":
                decision = adaptive_policy_adjustment(rec)
                state.w_cur = len(comm.members)
                state.n_maj = state.w_cur
                state.n_min = state.n_ms = state.n_mi = 0
            else:
                decision = policy_adjustment(state, rec)
            restore = decision.restore_mode.value
            for kk in list(reduced):
                reduced[kk] = None
            if decision.at_boundary:
                comm.quiesced = True
                comm.boundary_latch = True
                minors_b = set(designate_boundary_minors(comm, decision.n_bdry))
                crossed = True
                p_major = m + decision.g_ext
                for rid in comm.members:
                    g = decision.g_ext - (1 if rid in minors_b else 0)
                    comm.targets[rid] = comm.targets.get(rid, 0) + g
                    rem_ext[rid] = g
            events.append({
                "failed": sorted(rec.failed_replicas), "contrib": rec.contrib,
                "at_boundary": decision.at_boundary, "g_ext": decision.g_ext,
                "n_bdry": decision.n_bdry,
                "promoted": [[r, ro.value] for r, ro in decision.promoted],
                "epoch_after": rec.epoch_after})
            reform_s += time.perf_counter() - h0

        def restoration() -> Optional[WorkResult]:
            nonlocal restore
            if restore == "skip":
                return None
            stale = sorted(k for k, e in tags.items() if e < comm.epoch)
            if restore == "non_blocking":
                cnt["rewinds"] += len(stale)   # rewind = no-op (out of place)
                tags.clear()
                reduced.clear()
                restore = "skip"
                comm.quiesced = False
                return None
            for k in stale:
                cnt["rewinds"] += 1
                work = reduce(k)
                if work.status is WorkStatus.FAILURE:
                    return work
                reduced[k] = work.reduced_epoch
            restore = "skip"
            comm.quiesced = False
            return None

        roles_before = dict(comm.roles)
        while True:
            while m < p_major:
                for rid in live():
                    execute(rid)
                m += 1
                cnt["rounds"] += 1
            cnt["passes"] += 1
            for k in range(len(self.bounds)):
                if k not in touched:
                    touched.add(k)
                    kill(inj.fire(DURING_SYNC, k))
                if not comm.quiesced:
                    tags[k] = comm.epoch          # snapshot_and_tag: tag only
                roles_before = dict(comm.roles)
                work = reduce(k)
                if work.status is WorkStatus.SUCCESS:
                    cnt["reduces"] += 1
                    reduced[k] = work.reduced_epoch
                elif work.status is WorkStatus.FAILURE:
                    on_failure(work)
            if not after_fired:
                after_fired = True
                self._sync_point(AFTER_SYNC)
                kill(inj.fire(AFTER_SYNC))
            roles_before = dict(comm.roles)
            work = comm.ulfm_consensus()
            if work.status is WorkStatus.FAILURE:
                on_failure(work)
            while True:
                roles_before = dict(comm.roles)
                failed = restoration()
                if failed is None:
                    break
                on_failure(failed)
            if m >= p_major:
                break

        self._end_of_step()
        if t_fail is not None:
            self.mark("commit")
        # ---- commit ----
        members = list(comm.members)
        reg, bdy = comm.census_contrib()
        total = reg + bdy
        adm = [i for r in members for i in admitted.get(r, ())]
        if self.policy_kind == "static" and (total != b or len(adm) != b
                                             or len(set(adm)) != b):
            raise InvariantViolation("step %d committed %d microbatches (%d distinct), want %d"
                                     % (t, total, len(set(adm)), b))
        for k in range(len(self.bounds)):
            if reduced.get(k) != comm.epoch:
                raise InvariantViolation("bucket %d reduced under %r, world epoch %d"
                                         % (k, reduced.get(k), comm.epoch))
        new_state = state
        if crossed:
            new_state = policy_advancement(state, w_cur=len(members))
            comm.boundary_latch = False
            comm.prior_roles.clear()
            comm.roles = assign_roles(new_state, members)
        self.state = new_state
        return CommitOutcome(
            step=t,
            contributions={r: comm.contrib_regular[r] + comm.contrib_boundary[r] for r in members},
            contrib_total=total, contrib_regular=reg, contrib_boundary=bdy,
            final_epoch=comm.epoch, w_cur=len(members),
            roles={r: comm.roles[r].value for r in members}, state=new_state,
            events=events, admitted={r: sorted(admitted.get(r, ())) for r in members},
            bucket_epochs=[reduced.get(k) for k in range(len(self.bounds))],
            rounds=cnt["rounds"], passes=cnt["passes"], reduces=cnt["reduces"],
            rewinds=cnt["rewinds"], boundary_crossed=crossed,
            launches=cnt["launches"],
            failure_wall_s=(time.perf_counter() - t_fail) if t_fail else None,
            reform_host_s=reform_s)

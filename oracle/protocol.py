"""numpy restatement of one replica world under the ReCoVer protocol —
TEST INFRASTRUCTURE (see oracle/__init__.py).

Written from the reference's behaviour, not its code: state lives in plain
dicts and the iteration is one method.  Every rule cites the reference line
(paths under /root/reference/pkg/src/steadybatch/) it restates.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import fold

MAJ, MIN, MSP, NSP, BDM = ("major", "minor", "major_spare", "minor_spare",
                           "boundary_minor")
SPARES = (MSP, NSP)
FILLS = {MAJ: MSP, MIN: NSP}  # comm.py:29-32


class OracleInvariant(RuntimeError):
    pass


class OracleAllDead(RuntimeError):
    pass


# ---- policy arithmetic (policy.py:53-166) ----

def ext_rounds(w: int, c: int, b: int) -> int:
    g = 1
    while c + w * g < b:   # smallest g >= 1 covering b (policy.py:53-59)
        g += 1
    return g


def layout(w: int, b: int) -> dict:
    """Steady-state layout (policy.py:110-132)."""
    g = -(-b // w)
    n_maj = b // g
    r = b - n_maj * g
    n_min = 1 if r else 0
    left = w - n_maj - n_min
    n_mi = 1 if (n_min and left >= 2) else 0
    return dict(w_cur=w, g_cur=g, r_cur=r, n_maj=n_maj, n_min=n_min,
                n_ms=left - n_mi, n_mi=n_mi)


def role_map(lay: dict, members: Sequence[int]) -> Dict[int, str]:
    """policy.py:145-166: majors, minor, major-spares, minor-spare."""
    seq = ([MAJ] * lay["n_maj"] + [MIN] * lay["n_min"] + [MSP] * lay["n_ms"]
           + [NSP] * lay["n_mi"])
    ids = sorted(members)
    if len(seq) != len(ids):
        raise OracleInvariant("layout size mismatch")
    return dict(zip(ids, seq))


class ScriptedKills:
    """(phase, bucket, [rids]) entries, each fired once (the reference
    tests' ScriptedInjector contract, test_trainer.py:33-50)."""

    def __init__(self, plan=()):
        self.plan = list(plan)

    def fire(self, phase, bucket=None):
        hit = [e for e in self.plan
               if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan = [e for e in self.plan if e not in hit]
        return [r for e in hit for r in e[2]]


class World:
    """W replicas of a toy model on a partitioned stream, all in one process.

    ``spares`` extra replicas reproduce the reference tests' make_world
    (test_trainer.py:53-63); spares=0 is sim.run_experiment's setup
    (sim.py:379-386).
    """

    def __init__(self, w_init: int, g_init: int, k: int = 2, dim: int = 3,
                 kind: str = "constant", seed: int = 7, spares: int = 0,
                 policy: str = "static", lr: float = 0.05):
        members = list(range(w_init + spares))
        self.b = w_init * g_init
        self.w_init, self.g_init = w_init, g_init
        self.pol = dict(w_cur=w_init, g_cur=g_init, r_cur=0, n_maj=w_init,
                        n_min=0, n_ms=0, n_mi=0)
        if spares:
            self.pol = layout(len(members), self.b)
        self.g_ext: Optional[int] = None
        self.members = members
        self.roles = role_map(self.pol, members)
        self.epoch = 0
        self.quiesced = False
        self.latch = False
        self.prior: Dict[int, str] = {}
        self.pending: set = set()
        self.reg = {r: 0 for r in members}
        self.bdy = {r: 0 for r in members}
        self.kind, self.seed, self.dim = kind, seed, dim
        self.stream_w = len(members)
        self.policy, self.lr, self.k = policy, lr, k
        self.g0 = fold.constant_g0(seed, dim) if kind == "constant" else None
        self.wstar = fold.linear_wstar(seed, dim) if kind == "linear" else None
        self.alive = {r: True for r in members}
        self.params = {r: np.zeros(dim) for r in members}
        self.flat = {r: np.zeros(dim) for r in members}
        self.cursor = {r: 0 for r in members}
        base = dim // k
        self.bounds = [(i * base, dim if i == k - 1 else (i + 1) * base)
                       for i in range(k)]
        self.grad_log: Dict[int, List[Tuple[int, np.ndarray]]] = {}

    # ---- the toy model (trainer.py:103-131, 159-168) ----

    def grad_loss(self, rid: int, i: int):
        if self.kind == "constant":
            x = self.g0
            return x, float(self.params[rid] @ x)
        x, y = fold.linear_example(self.seed, i, self.dim, self.wstar)
        r = self.params[rid] @ x - y
        return r * x, float(r * r)

    # ---- collective phases (comm.py:129-213) ----

    def census_roles(self):
        held = [self.roles[r] for r in self.members]
        return tuple(held.count(x) for x in (MAJ, MIN, MSP, NSP, BDM))

    def detect(self):
        dead = sorted(self.pending & set(self.members))
        if not dead:
            return None
        lost = {r: self.roles[r] for r in dead}
        self.members = [r for r in self.members if r not in lost]
        self.pending -= set(dead)
        for d in (self.roles, self.reg, self.bdy, self.prior):
            for r in dead:
                d.pop(r, None)
        if not self.members:
            raise OracleAllDead("all replicas dead")
        self.epoch += 1
        _, _, ms, mi, _ = self.census_roles()
        boundary = self.latch or (list(lost.values()).count(MAJ) > ms
                                  or list(lost.values()).count(MIN) > mi)
        promos = []
        if not boundary:
            for r in dead:
                if lost[r] in FILLS:
                    pick = [m for m in self.members if self.roles[m] == FILLS[lost[r]]][0]
                    self.roles[pick] = lost[r]
                    promos.append((pick, lost[r]))
        reg = sum(self.reg[r] for r in self.members)
        bdy = sum(self.bdy[r] for r in self.members)
        return dict(failed=dead, counts=self.census_roles(), contrib=reg + bdy,
                    boundary=boundary, epoch_after=self.epoch, promos=promos)

    def allreduce(self, lo: int, hi: int):
        if self.quiesced:
            return "noop", None
        rec = self.detect()
        if rec is not None:
            return "failure", rec
        views = [self.flat[r][lo:hi] for r in self.members]
        contrib = [self.latch or self.roles[r] not in SPARES for r in self.members]
        total = fold.masked_fold(views, contrib)
        for v in views:
            v[:] = total
        return "success", self.epoch

    # ---- one iteration (trainer.py:324-487) ----

    def iterate(self, t: int, kills=None) -> dict:
        kills = kills or ScriptedKills()
        b = self.b

        def kill(rids):
            for r in rids:
                if self.alive.get(r):
                    self.alive[r] = False
                    if r in self.members:
                        self.pending.add(r)

        kill(kills.fire("before_sync"))
        if not any(self.alive[r] for r in self.members):
            raise OracleAllDead("no replica survives iteration %d" % t)
        for r in self.members:
            self.reg[r] = self.bdy[r] = 0
        runs_g = (MAJ, MSP)
        rem_reg, rem_ext, admitted, prov = {}, {}, {}, {}
        loss_adm, loss_prov, role_now = {}, {}, {}
        for r in self.members:
            if not self.alive[r]:
                continue
            role_now[r] = self.roles[r]
            rem_reg[r] = self.pol["g_cur"] if self.roles[r] in runs_g else self.pol["r_cur"]
            rem_ext[r] = 0
            admitted[r], prov[r] = [], []
            loss_adm[r] = loss_prov[r] = 0.0
            self.flat[r][:] = 0.0
        snap: Dict[Tuple[int, int], Tuple[np.ndarray, int]] = {}
        reduced: Dict[Tuple[int, int], Optional[int]] = {}
        restore = {r: "skip" for r in self.members}
        p_major, m = self.pol["g_cur"], 0
        cnt = dict(rounds=0, passes=0, reduces=0, rewinds=0)
        events, crossed, after_fired, touched = [], False, False, set()

        def live():
            return [r for r in self.members if self.alive[r]]

        def microbatch(r):
            i = r + self.stream_w * self.cursor[r]
            self.cursor[r] += 1
            if rem_reg[r] > 0:
                rem_reg[r] -= 1
                g, loss = self.grad_loss(r, i)
                self.flat[r] += g
                if role_now[r] in SPARES:
                    prov[r].append(i)
                    loss_prov[r] += loss
                else:
                    admitted[r].append(i)
                    loss_adm[r] += loss
                    self.reg[r] += 1
            elif rem_ext[r] > 0:
                rem_ext[r] -= 1
                g, loss = self.grad_loss(r, i)
                self.flat[r] += g
                admitted[r].append(i)
                loss_adm[r] += loss
                self.bdy[r] += 1

        def on_failure(rec):
            nonlocal p_major, crossed
            for rid, role in rec["promos"]:           # trainer.py:263-272
                admitted[rid].extend(prov[rid])
                loss_adm[rid] += loss_prov[rid]
                self.reg[rid] += len(prov[rid])
                prov[rid], loss_prov[rid] = [], 0.0
                role_now[rid] = role
            w = len(self.members)
            if self.policy == "adaptive":                # trainer.py:285-289
                self.pol.update(w_cur=w, n_maj=w, n_min=0, n_ms=0, n_mi=0)
                mode, boundary, g_ext, n_b = "blocking", False, None, None
            else:                                        # policy.py:77-107
                self.pol["w_cur"] = w
                if not rec["boundary"]:
                    c = rec["counts"]
                    self.pol.update(n_maj=c[0], n_min=c[1], n_ms=c[2], n_mi=c[3])
                    mode, boundary, g_ext, n_b = "blocking", False, None, None
                else:
                    if rec["contrib"] > b:
                        raise OracleInvariant("census exceeds the batch")
                    g_ext = ext_rounds(w, rec["contrib"], b)
                    n_b = rec["contrib"] + w * g_ext - b
                    self.g_ext = g_ext
                    mode, boundary = "non_blocking", True
            for r in self.members:
                restore[r] = mode
                for kk in range(self.k):
                    reduced[(r, kk)] = None
            if boundary:                                 # trainer.py:297-303
                self.quiesced = self.latch = True
                for r, pr in self.prior.items():         # comm.py:236-239
                    if r in self.roles:
                        self.roles[r] = pr
                self.prior = {}
                chosen = sorted(self.members)[len(self.members) - n_b:] if n_b > 0 else []
                for r in chosen:
                    self.prior[r] = self.roles[r]
                    self.roles[r] = BDM
                crossed = True
                p_major = m + g_ext                      # trainer.py:362-369
                for r in self.members:
                    rem_ext[r] = g_ext - 1 if r in chosen else g_ext
            events.append({"failed": rec["failed"], "contrib": rec["contrib"],
                           "at_boundary": boundary, "g_ext": g_ext,
                           "n_bdry": n_b,
                           "promoted": [[r, ro] for r, ro in
                                        (rec["promos"] if not boundary else [])],
                           "epoch_after": rec["epoch_after"]})

        def stale_of(r):
            return {kk for kk in range(self.k)
                    if (r, kk) in snap and snap[(r, kk)][1] < self.epoch}

        def restoration():                               # buckets.py:103-175
            modes = {restore[r] for r in self.members}
            assert len(modes) == 1
            mode = modes.pop()
            if mode == "skip":
                return None, 0
            if mode == "non_blocking":
                n = None
                for r in self.members:
                    st = stale_of(r)
                    n = len(st) if n is None else n
                    for kk in sorted(st):
                        lo, hi = self.bounds[kk]
                        self.flat[r][lo:hi] = snap[(r, kk)][0]
                    role = self.roles[r]
                    if role == BDM:
                        role = self.prior.get(r, role)
                    if role in SPARES and self.reg[r] == 0 and self.bdy[r] == 0:
                        self.flat[r][:] = 0.0
                    for kk in range(self.k):
                        snap.pop((r, kk), None)
                        reduced[(r, kk)] = None
                    restore[r] = "skip"
                self.quiesced = False
                return None, n or 0
            st = stale_of(self.members[0])
            assert all(stale_of(r) == st for r in self.members)
            n = 0
            for kk in sorted(st):
                lo, hi = self.bounds[kk]
                for r in self.members:
                    self.flat[r][lo:hi] = snap[(r, kk)][0]
                n += 1
                status, val = self.allreduce(lo, hi)
                if status == "failure":
                    return val, n
                for r in self.members:
                    reduced[(r, kk)] = val
            for r in self.members:
                restore[r] = "skip"
            self.quiesced = False
            return None, n

        while True:
            while m < p_major:
                for r in live():
                    microbatch(r)
                m += 1
                cnt["rounds"] += 1
            cnt["passes"] += 1
            for kk in range(self.k):
                lo, hi = self.bounds[kk]
                if kk not in touched:
                    touched.add(kk)
                    kill(kills.fire("during_sync", kk))
                if not self.quiesced:
                    for r in live():
                        snap[(r, kk)] = (self.flat[r][lo:hi].copy(), self.epoch)
                status, val = self.allreduce(lo, hi)
                if status == "success":
                    cnt["reduces"] += 1
                    for r in self.members:
                        reduced[(r, kk)] = val
                elif status == "failure":
                    on_failure(val)
            if not after_fired:
                after_fired = True
                kill(kills.fire("after_sync"))
            rec = self.detect()
            if rec is not None:
                on_failure(rec)
            while True:
                rec, n = restoration()
                cnt["rewinds"] += n
                if rec is None:
                    break
                on_failure(rec)
            if m >= p_major:
                break

        # commit (trainer.py:420-487)
        surv = list(self.members)
        reg = sum(self.reg[r] for r in surv)
        bdy = sum(self.bdy[r] for r in surv)
        total = reg + bdy
        adm = [i for r in surv for i in admitted[r]]
        if self.policy == "static" and (total != b or len(adm) != b or len(set(adm)) != b):
            raise OracleInvariant("iteration %d committed %d" % (t, total))
        for r in surv:
            for kk in range(self.k):
                if reduced.get((r, kk)) != self.epoch:
                    raise OracleInvariant("impure bucket epoch")
        ref = self.flat[surv[0]]
        for r in surv[1:]:
            if not np.array_equal(self.flat[r], ref):
                raise OracleInvariant("replica buffers diverged")
        update = fold.commit_update(ref, b)
        # builtin sum(): compensated (Neumaier) on Python >= 3.12, as in the
        # reference's `sum(rep.loss_admitted ...)` (trainer.py:447)
        loss_sum = sum(loss_adm[r] for r in surv)
        loss = loss_sum / float(total) if total else 0.0
        for r in surv:
            self.params[r] = fold.sgd(self.params[r], self.flat[r], b, self.lr)
        bucket_epochs = [reduced.get((surv[0], kk)) for kk in range(self.k)]
        if crossed:                                      # trainer.py:459-464
            self.pol = layout(len(surv), b)
            self.latch = False
            self.prior = {}
            self.roles = role_map(self.pol, surv)
            self.g_ext = None
        return dict(
            iteration=t, loss=loss, update=update,
            contributions={r: self.reg[r] + self.bdy[r] for r in surv},
            contrib_total=total, contrib_regular=reg, contrib_boundary=bdy,
            final_epoch=self.epoch, w_cur=len(surv),
            roles={r: self.roles[r] for r in surv},
            g_cur=self.pol["g_cur"], events=events,
            admitted=sorted(adm), bucket_epochs=bucket_epochs,
            rounds=cnt["rounds"], passes=cnt["passes"],
            reduces=cnt["reduces"], rewinds=cnt["rewinds"],
            boundary=crossed, params=self.params[surv[0]].copy())

"""Host control plane of the drop-in (no data movement, CPU): the
reference's test_comm.py / test_policy.py cases that never touch a buffer,
plus an exhaustive policy sweep against the oracle."""

import numpy as np
import pytest

from paper_2605_11215_b200.buckets import RestoreMode, bucket_bounds
from paper_2605_11215_b200.comm import (
    Communicator, EmptyMembership, FailureRecord, NoSpareAvailable, ReplicaRole,
    WorkStatus, designate_boundary_minors, elect_promotion)
from paper_2605_11215_b200.policy import (
    InvariantViolation, adaptive_policy_adjustment, assign_roles,
    boundary_minor_count, contribution_quota, extension_rounds, initial_state,
    policy_adjustment, policy_advancement)
from oracle.protocol import layout

M, MI, MS, NS, BM = (ReplicaRole.MAJOR, ReplicaRole.MINOR, ReplicaRole.MAJOR_SPARE,
                     ReplicaRole.MINOR_SPARE, ReplicaRole.BOUNDARY_MINOR)


def rec(failed=(31,), counts=(31, 0, 0, 0, 0), contrib=248, bdy=0, boundary=True,
        epoch=1, promotions=()):
    return FailureRecord(frozenset(failed), counts, contrib, contrib - bdy, bdy,
                         boundary, epoch, promotions)


def test_failure_record_contrib_248():      # test_comm.py:50-66 (control part)
    comm = Communicator(range(32))
    for r in comm.members:
        comm.contrib_regular[r] = 8
    comm.mark_dead(31)
    res = comm.ulfm_allreduce({})           # detection precedes any data access
    assert res.status is WorkStatus.FAILURE
    r = res.record
    assert r.failed_replicas == frozenset({31}) and r.contrib == 248 and r.at_boundary
    assert r.epoch_after == 1 and comm.members == list(range(31))


def test_quiesce_noop_without_detection():  # test_comm.py:69-80
    comm = Communicator(range(4))
    comm.quiesced = True
    comm.mark_dead(2)
    assert comm.ulfm_allreduce({}).status is WorkStatus.NOOP
    assert comm.epoch == 0 and comm.members == [0, 1, 2, 3]
    res = comm.ulfm_consensus()             # test_comm.py:83-90
    assert res.status is WorkStatus.FAILURE and comm.epoch == 1


def test_promotions_and_boundaries():
    comm = Communicator(range(5), {0: M, 1: M, 2: MI, 3: MS, 4: NS})
    comm.mark_dead(0)
    comm.mark_dead(2)
    r = comm.ulfm_consensus().record        # test_comm.py:100-111
    assert not r.at_boundary and r.promotions == ((3, M), (4, MI))
    assert r.role_counts == (2, 1, 0, 0, 0)
    comm = Communicator(range(5), {**{i: M for i in range(4)}, 4: MS})
    comm.mark_dead(1)
    comm.mark_dead(2)
    r = comm.ulfm_consensus().record        # test_comm.py:114-122
    assert r.at_boundary and r.promotions == ()
    comm = Communicator(range(3), {0: M, 1: M, 2: MS})
    comm.mark_dead(2)
    r = comm.ulfm_consensus().record        # test_comm.py:125-133
    assert not r.at_boundary and r.role_counts == (2, 0, 0, 0, 0)
    comm = Communicator(range(4))
    comm.boundary_latch = True
    comm.mark_dead(3)
    assert comm.ulfm_consensus().record.at_boundary  # test_comm.py:136-141


def test_elect_and_designate():
    comm = Communicator([0, 5, 9], {0: M, 5: MS, 9: MS})
    assert elect_promotion(comm, M) == 5 and comm.roles[5] is M
    with pytest.raises(NoSpareAvailable):
        elect_promotion(Communicator(range(3)), M)
    with pytest.raises(ValueError):
        elect_promotion(comm, MS)
    comm = Communicator(range(6))
    assert designate_boundary_minors(comm, 2) == [4, 5]
    assert comm.prior_roles[4] is M
    comm.mark_dead(5)
    comm.boundary_latch = True
    comm.ulfm_consensus()
    assert designate_boundary_minors(comm, 3) == [2, 3, 4]
    assert set(comm.prior_roles) == {2, 3, 4} and comm.roles[0] is M
    with pytest.raises(EmptyMembership):
        c = Communicator(range(1))
        c.mark_dead(0)
        c.ulfm_consensus()


def test_epochs_batch_deaths():
    comm = Communicator(range(8))
    comm.mark_dead(1)
    comm.mark_dead(5)
    assert comm.ulfm_consensus().record.failed_replicas == frozenset({1, 5})
    assert comm.epoch == 1


def test_policy_walkthrough_numbers():      # test_policy.py:44-108
    st = initial_state(32, 8)
    d = policy_adjustment(st, rec())
    assert (d.at_boundary, d.restore_mode, d.g_ext, d.n_bdry, st.w_cur) == \
        (True, RestoreMode.NON_BLOCKING, 1, 23, 31)
    st = initial_state(8, 5)
    st.w_cur = 5
    d = policy_adjustment(st, rec((5, 6, 7), (5, 0, 0, 0, 0), 17))
    assert (d.g_ext, d.n_bdry) == (5, 2)
    st = policy_advancement(initial_state(32, 8), w_cur=31)
    assert (st.n_maj, st.n_min, st.n_ms, st.n_mi, st.g_cur, st.r_cur) == (28, 1, 1, 1, 9, 4)
    d = policy_adjustment(st, rec((28,), (28, 1, 1, 0, 0), 0, boundary=False,
                                  promotions=((30, MI),)))
    assert d.restore_mode is RestoreMode.BLOCKING and d.promoted == ((30, MI),)
    assert (st.n_maj, st.n_min, st.n_ms, st.n_mi, st.w_cur) == (28, 1, 1, 0, 30)
    with pytest.raises(InvariantViolation):
        policy_adjustment(initial_state(4, 2), rec((3,), (3, 0, 0, 0, 0), 9))
    d = adaptive_policy_adjustment(rec())
    assert d.restore_mode is RestoreMode.BLOCKING and d.g_ext is None


def test_quotas_and_roles():                # test_policy.py:142-172
    st = policy_advancement(initial_state(32, 8), w_cur=31)
    roles = assign_roles(st, list(range(31)))
    assert roles[27] is M and roles[28] is MI and roles[29] is MS and roles[30] is NS
    assert [contribution_quota(st, r) for r in (M, MI, MS, NS)] == [9, 4, 0, 0]
    st.g_ext = 2
    assert contribution_quota(st, M, True) == 11
    assert contribution_quota(st, BM, True, prior_role=M) == 10
    with pytest.raises(ValueError):
        contribution_quota(st, BM, True)
    with pytest.raises(InvariantViolation):
        assign_roles(st, list(range(30)))


def test_policy_exhaustive_vs_oracle():
    """Criterion-3-style sweep (test_acceptance.py:160-191): every (w, c, b)
    with w <= 64, b <= 512 for the extension arithmetic (vectorised, like the
    reference), every (w, b) for the layout."""
    bs = np.repeat(np.arange(1, 513, dtype=np.int64), np.arange(2, 514))
    cs = np.concatenate([np.arange(b + 1, dtype=np.int64) for b in range(1, 513)])
    for w in range(1, 65):
        g = np.ones_like(bs)
        short = cs + w * g < bs
        while short.any():
            g[short] += 1
            short = cs + w * g < bs
        pg = extension_rounds(w, cs, bs)
        assert np.array_equal(pg, g)
        assert np.array_equal(boundary_minor_count(w, cs, bs, pg), cs + w * g - bs)
    for w in range(1, 65):
        for b in range(1, 513):
            st = initial_state(w, 1)
            st.b = b
            a = policy_advancement(st, w_cur=w)
            l = layout(w, b)
            assert (a.g_cur, a.n_maj, a.r_cur, a.n_min, a.n_ms, a.n_mi) == \
                (l["g_cur"], l["n_maj"], l["r_cur"], l["n_min"], l["n_ms"], l["n_mi"])


def test_bucket_bounds():                   # test_buckets.py:21-34
    assert [hi - lo for lo, hi in bucket_bounds(10, 3)] == [3, 3, 4]
    assert [hi - lo for lo, hi in bucket_bounds(2, 4)] == [0, 0, 0, 2]
    with pytest.raises(ValueError):
        bucket_bounds(3, 0)

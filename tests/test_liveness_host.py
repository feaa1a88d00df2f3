"""Node-local liveness (live.cpp) on the CPU box: two processes share a
heartbeat segment; when one is SIGKILLed the other's native watcher declares
it dead within the deadline, and every poll point is decided once — a rank
reaching it later gets the same failed set back."""

import multiprocessing as mp
import os
import signal
import time
import uuid

from paper_2605_11215_b200 import _lib


def _victim(name, ready, go):
    lv = _lib.Liveness(name, 1, 2, period_s=1e-3, deadline_s=20e-3)
    ready.set()
    go.wait(30)
    lv.note_kill()
    os.kill(os.getpid(), signal.SIGKILL)


def test_sigkilled_peer_declared_dead_within_deadline():
    name = "/rcv-test-%s" % uuid.uuid4().hex[:12]
    ctx = mp.get_context("spawn")
    ready, go = ctx.Event(), ctx.Event()
    p = ctx.Process(target=_victim, args=(name, ready, go))
    lv = _lib.Liveness(name, 0, 2, period_s=1e-3, deadline_s=20e-3)
    try:
        p.start()
        assert ready.wait(60)
        time.sleep(0.1)                      # both beating: nobody declared
        assert lv.dead() == 0
        assert lv.decide(1) == (0, lv.decide(1)[1])
        go.set()
        p.join(30)
        assert p.exitcode == -signal.SIGKILL
        t0 = time.time()
        while not lv.dead() and time.time() - t0 < 5:
            time.sleep(1e-3)
        assert lv.dead() == 0b10
        st = lv.stats(1)
        detect_ms = (st["dead_ns"] - st["kill_ns"]) / 1e6
        assert 0 <= detect_ms <= 40, detect_ms   # deadline 20 ms + one period
        # poll 1 was decided before the death: it stays "nobody"
        assert lv.decide(1)[0] == 0
        m2, _ = lv.decide(2)
        assert m2 == 0b10 and lv.decide(2)[0] == m2
    finally:
        lv.close(unlink=True)

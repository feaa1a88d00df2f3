"""metrics/v1 rows and the accounting compare.  CPU: file
round trip, compare semantics, the schedule injector's firing rule.  GPU:
replaying the reference's own sim.run_experiment runs (generated schedules,
the Appendix-E trace, the throughput config) on the device drop-in gives
rows whose accounting equals the reference's rows exactly."""

import copy

import pytest

from paper_2605_11215_b200.metrics import (ScheduleInjector, compare_rows,
                                           read_metrics, replay_experiment,
                                           write_metrics)


def test_round_trip_and_compare(tmp_path, golden):
    run = golden["metrics_runs"][0]
    p = tmp_path / "m.jsonl"
    write_metrics(str(p), {"config": run["config"]}, run["rows"])
    meta, rows = read_metrics(str(p))
    assert meta["schema"] == "metrics/v1" and rows == run["rows"]
    assert compare_rows(rows, run["rows"]) == []
    bad = copy.deepcopy(rows)
    bad[1]["contributions"][0][1] += 1
    bad[2]["events"] = []
    diffs = compare_rows(bad, run["rows"])
    assert len(diffs) == 2 and "contributions" in diffs[0]
    # clocks are measured here and simulated there: never compared
    bad = copy.deepcopy(rows)
    bad[0]["elapsed"] = 123.0
    assert compare_rows(bad, run["rows"]) == []


def test_schedule_injector_fires_like_reference():
    inj = ScheduleInjector([(2, 5, "during_sync:1"), (2, 3, "before_sync"), (4, 1, "after_sync")])
    inj.set_step(2)
    assert inj.fire("before_sync") == [3]
    assert inj.fire("during_sync", 0) == [] and inj.fire("during_sync", 1) == [5]
    inj.set_step(4)
    assert inj.fire("after_sync") == [1] and inj.fire("before_sync") == []


@pytest.mark.gpu
def test_replayed_runs_match_reference_rows(golden):
    assert len(golden["metrics_runs"]) >= 12
    for run in golden["metrics_runs"]:
        c = run["config"]
        rows = replay_experiment(c["w_init"], c["g_init"], c["iterations"], c["k_buckets"],
                                 c["dim"], c["model_kind"], c["stream_seed"], c["lr"],
                                 c["policy"], run["entries"])
        assert compare_rows(rows, run["rows"]) == [], run["name"]

"""Host logic of the auto-tuner (paper_2001_04438_b200/tune.py; no GPU needed)."""
import os

import pytest

tune = pytest.importorskip("paper_2001_04438_b200.tune")
tp = pytest.importorskip("paper_2001_04438_b200")


def test_candidates_cover_the_schedules_that_apply():
    one_block = tune.candidates(64, 1000)
    assert {"schedule": tp.SCHED_AUTO} in one_block
    assert all(c["schedule"] != tp.SCHED_CLUSTER for c in one_block)
    assert {c.get("cluster_size") for c in one_block if c["schedule"] == tp.SCHED_SMALL} == {1}
    two_blocks = tune.candidates(64, 32768)  # C2: the small schedule with 1 or 2 CTAs per row
    assert {c.get("cluster_size") for c in two_blocks if c["schedule"] == tp.SCHED_SMALL} == {1, 2}
    c4 = tune.candidates(256, 800000)       # 49 blocks per row: cluster sizes 1..8, look-aheads
    assert {c.get("cluster_size") for c in c4 if c["schedule"] == tp.SCHED_CLUSTER} == {1, 2, 4, 8}
    assert any(c.get("lookahead_rows") == 32 for c in c4)
    huge = tune.candidates(1, 1 << 26)      # 4096 blocks: no cluster schedule, no look-ahead > rows
    assert all(c["schedule"] != tp.SCHED_CLUSTER for c in huge)
    assert all(c.get("lookahead_rows", 0) < 1 or c["lookahead_rows"] < 1 for c in huge)


def test_pick_best_is_the_fastest_and_stable_on_ties():
    t = [({"schedule": 0}, 2.0), ({"schedule": 1}, 1.5), ({"schedule": 3}, 1.5)]
    assert tune.pick_best(t) == {"schedule": 1}


def test_cache_round_trip(tmp_path):
    p = os.path.join(tmp_path, "sub", "tune.json")
    assert tune.load_cache(p) == {}
    tune.save_cache({"k": {"opts": {"schedule": 3, "cluster_size": 4}, "ms": 0.37}}, p)
    assert tune.load_cache(p)["k"]["opts"] == {"schedule": 3, "cluster_size": 4}
    with open(p, "w") as f:
        f.write("{corrupt")
    assert tune.load_cache(p) == {}

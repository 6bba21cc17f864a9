"""Timeline model of the data-parallel step (reference
src/simulator.cpp, tests/test_simulator.cpp). CPU only: the B200 host
implementation against the reference's own simulator on random scenarios
(report text identical, %.17g), the reference tests' known answers, and the
reference tests' rejections of malformed scenario text."""
import random

import pytest

import paper_1904_01038_b200 as sqf
from oracle import ref


def text(w, a, mode, compute, buckets):
    lines = [f"workers {w}", f"accum {a}", f"mode {mode}"]
    lines += [f"compute {i} " + " ".join(repr(x) for x in row) for i, row in enumerate(compute)]
    lines.append("buckets " + " ".join(repr(x) for x in buckets))
    return "\n".join(lines) + "\n"


def test_known_answers():  # test_simulator.cpp:60-104
    r = sqf.simulate_timeline(text(2, 1, "serial_sync", [[1.0], [2.0]], [0.5]))
    assert (r["makespan"], r["idle"], r["exposed_comm"], r["total_compute"]) == (2.5, [1.0, 0.0], 0.5, 3.0)
    assert "makespan 2.5\n" in r["text"] and "idle 0 1\n" in r["text"] and "total_compute 3\n" in r["text"]
    r = sqf.simulate_timeline(text(2, 1, "overlap", [[1.0], [2.0]], [0.25, 0.25]))
    assert r["makespan"] == 2.25 and r["exposed_comm"] == 0.25
    flip = [[1.0, 2.0], [2.0, 1.0]]
    serial = sqf.simulate_timeline(text(2, 2, "serial_sync", flip, [0.5]))
    accum = sqf.simulate_timeline(text(2, 2, "overlap_accum", flip, [0.5]))
    assert serial["makespan"] == 5.0 and serial["idle"] == [1.0, 1.0]
    assert accum["makespan"] == 3.5 and accum["idle"] == [0.0, 0.0] and accum["exposed_comm"] == 0.5
    rt = sqf.simulate_timeline("# toy imbalance\nworkers 2\naccum 2\nmode overlap_accum\n"
                               "compute 0 1.0 2.0   # slow second half\ncompute 1 2.0 1.0\nbuckets 0.5\n")
    assert rt["makespan"] == 3.5


@pytest.mark.parametrize("seed", range(40))
def test_matches_reference_on_random_scenarios(seed):
    if not ref.available():
        pytest.skip("oracle not built")
    rng = random.Random(seed)
    w, a = rng.randint(1, 8), rng.randint(1, 16)
    compute = [[rng.uniform(0.05, 3.0) for _ in range(a)] for _ in range(w)]
    buckets = [rng.uniform(0.001, 0.7) for _ in range(rng.randint(1, 40))]
    for mode in ("serial_sync", "overlap", "overlap_accum"):
        t = text(w, a, mode, compute, buckets)
        mine = sqf.simulate_timeline(t)
        assert mine["text"] == ref.simulate_timeline(w, a, mode, compute, buckets)
    # overlap never loses to the serial barrier (test_simulator.cpp:106-123)
    s = sqf.simulate_timeline(text(w, a, "serial_sync", compute, buckets))["makespan"]
    o = sqf.simulate_timeline(text(w, a, "overlap", compute, buckets))["makespan"]
    assert o <= s + 1e-12


BAD = ["", "workers 1\naccum 1\nmode overlap\ncompute 0 1.0\n",
       "workers 1\naccum 1\nmode sideways\ncompute 0 1.0\nbuckets 0.5\n",
       "workers 2\naccum 1\nmode overlap\ncompute 0 1.0\nbuckets 0.5\n",
       "workers 1\naccum 1\nmode overlap\ncompute 3 1.0\nbuckets 0.5\n",
       "workers 1\naccum 2\nmode overlap\ncompute 0 1.0\nbuckets 0.5\n",
       "workers 1\naccum 1\nmode overlap\ncompute 0 1.0\ncompute 0 1.0\nbuckets 0.5\n",
       "workers 1 9\naccum 1\nmode overlap\ncompute 0 1.0\nbuckets 0.5\n",
       "compute 0 1.0\nworkers 1\naccum 1\nmode overlap\nbuckets 0.5\n",
       "workers 1\naccum 1\nmode overlap\ncompute 0 1.0\nbuckets 0.5\nflux 9\n",
       "workers 1\naccum 1\nmode overlap\ncompute 0 -1.0\nbuckets 0.5\n",
       "workers 1\naccum 1\nmode overlap\ncompute 0 1.0\nbuckets 0.5 zero\n",
       "workers 1\naccum 1\nmode overlap\ncompute 0 0.0\nbuckets 0.5\n"]


@pytest.mark.parametrize("bad", BAD)
def test_rejects_malformed_scenarios_like_the_reference(bad):  # test_simulator.cpp:146-176
    with pytest.raises(Exception, match="ConfigError"):
        sqf.simulate_timeline(bad)

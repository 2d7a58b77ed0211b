"""Append-only JSONL trial log with resume, cost-table mode:
a tuning job killed after its exploration phase resumes from the log without
re-measuring, continues with distinct new points, and ends at the same Droplet result as
an uninterrupted run; lines of another problem are ignored; a malformed line is refused."""
import json
import math

import pytest

from paper_2406_20037_b200 import Tuner, TunerError
from synth import landscape

SK = [[1, 2, 4, 8, 16], [1, 2, 3, 4], [8, 16, 32]]
SHAPE = {"m": 64, "n": 32, "k": 16}


def table():
    return landscape([[len(v) for v in SK]], "rugged", 3, 0.1)


def make(log, shape=SHAPE, seed=0):
    return Tuner("dense", shape, spaces=[(0, SK)], cost_table=table(), seed=seed, trial_log=str(log))


def test_log_lines_and_resume(tmp_path):
    log = tmp_path / "trials.jsonl"
    t = make(log)
    smp = t.sample(20)
    hist = [(s.point, s.cost_ns) for s in t.history()]
    t.close()
    lines = [json.loads(x) for x in log.read_text().splitlines()]
    assert len(lines) == 20
    for ln, (p, c) in zip(lines, hist):
        assert ln["sketch"] == 0 and ln["vals"] == [SK[d][i] for d, i in enumerate(p[1])]
        assert (ln["cost_ns"] is None and not math.isfinite(c)) or ln["cost_ns"] == c
    # resume: the history comes back without a measurement
    r = make(log)
    assert r.stats()["replayed"] == 20 and r.stats()["candidates"] == 0
    assert [(s.point, s.cost_ns) for s in r.history()] == hist
    more = r.sample(10)
    assert len({s.point for s in more} | {p for p, _ in hist}) == 30  # no re-measurement
    assert len(log.read_text().splitlines()) == 30
    # the resumed Droplet from best-of-N equals the uninterrupted run's
    rep_r = r.droplet(r.best().point, 100)
    u = Tuner("dense", SHAPE, spaces=[(0, SK)], cost_table=table(), seed=0)
    u.sample(20)
    u.sample(10)
    rep_u = u.droplet(u.best().point, 100)
    assert rep_r["best"] == rep_u["best"] and rep_r["best_cost"] == rep_u["best_cost"]


def test_other_problem_lines_are_ignored(tmp_path):
    log = tmp_path / "trials.jsonl"
    make(log).sample(12)
    other = make(log, shape={"m": 64, "n": 32, "k": 32})
    assert other.stats()["replayed"] == 0 and other.history() == []


def test_malformed_line_is_refused(tmp_path):
    log = tmp_path / "trials.jsonl"
    log.write_text('{"key": broken\n')
    with pytest.raises(TunerError, match="EINVAL"):
        make(log)

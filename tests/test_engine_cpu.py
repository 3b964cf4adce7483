"""The wall-clock engine's timer API against the reference engine's contract
(pkg/tests/test_engine.py:15-129): (time, seq) dispatch order, tombstone
cancel, no scheduling into the past, run(until) bounds, a deterministic event
log for identical runs, independent reproducible PCG64 streams.  A fake clock
that advances on every read stands in for wall time."""
import pytest

from paper_2404_14691_b200.engine import Engine, EventKind, rng_stream
from paper_2404_14691_b200.resources import SimulationError


class FakeClock:
    def __init__(self, step_us: int = 1):
        self.t, self.step = 0, step_us

    def __call__(self) -> int:
        self.t += self.step
        return self.t


def engine(log: bool = False) -> Engine:
    return Engine(log_events=log, clock=FakeClock(), poll=lambda evs, to: [True] * len(evs))


def collect(eng):
    seen = []
    return seen, lambda tag: seen.append((eng.now, tag))


def test_same_time_events_dispatch_in_schedule_order():
    eng = engine()
    seen, cb = collect(eng)
    eng.schedule(5, EventKind.ARRIVAL, cb, "first")
    eng.schedule(5, EventKind.ARRIVAL, cb, "second")
    eng.run()
    assert seen == [(5, "first"), (5, "second")]


def test_time_then_seq_order():
    eng = engine()
    seen, cb = collect(eng)
    eng.schedule(20, EventKind.ARRIVAL, cb, "a")
    eng.schedule(10, EventKind.ARRIVAL, cb, "b")
    eng.schedule(20, EventKind.ARRIVAL, cb, "c")
    eng.run()
    assert [tag for _, tag in seen] == ["b", "a", "c"]
    assert [t for t, _ in seen] == [10, 20, 20]          # a timer runs at its scheduled instant


def test_cancel_semantics():
    eng = engine()
    seen, cb = collect(eng)
    h = eng.schedule(5, EventKind.STAGE_COMPLETE, cb, "x")
    assert eng.cancel(h) is True
    assert eng.cancel(h) is False                        # twice
    done = eng.schedule(6, EventKind.ARRIVAL, cb, "y")
    eng.run()
    assert seen == [(6, "y")]
    assert eng.cancel(done) is False                     # after dispatch
    with pytest.raises(SimulationError):
        eng.cancel("not-a-handle")
    with pytest.raises(SimulationError):
        engine().cancel(done)                            # another engine's handle


def test_schedule_into_past_aborts():
    eng = engine()
    eng.schedule(10, EventKind.ARRIVAL, lambda p: None)
    eng.run()
    with pytest.raises(SimulationError):
        eng.schedule(9, EventKind.ARRIVAL, lambda p: None)


def test_run_until_and_clock_monotone():
    eng = engine()
    seen, cb = collect(eng)
    eng.schedule(30, EventKind.ARRIVAL, cb, "a")
    eng.schedule(70, EventKind.ARRIVAL, cb, "b")
    eng.run(until=50)
    assert seen == [(30, "a")] and eng.now >= 50
    eng.run()
    assert seen == [(30, "a"), (70, "b")]
    assert eng.run() == 0                                # empty queue


def test_event_log_identical_for_identical_runs():
    def build():
        eng = engine(log=True)
        rng = rng_stream(7, 0)

        def rec(_):
            t = eng.now + int(rng.integers(1, 10))
            if t < 400:
                eng.schedule(t, EventKind.GENERATOR_TICK, rec)
        eng.schedule(0, EventKind.GENERATOR_TICK, rec)
        eng.run()
        return eng.event_log
    assert build() == build()
    with pytest.raises(SimulationError):
        engine().event_log


def test_rng_streams_independent_and_reproducible():
    a1 = rng_stream(42, 0).integers(0, 1000, size=8).tolist()
    a2 = rng_stream(42, 0).integers(0, 1000, size=8).tolist()
    b = rng_stream(42, 1).integers(0, 1000, size=8).tolist()
    assert a1 == a2 and a1 != b

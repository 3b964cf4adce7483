"""ComputeGate on the device (ClusterSpec.compute_concurrency; reference
functions.py:304-327, simulation.py:127-130): with K slots per GPU, at most K
invocations compute at once, FIFO.  Six 3 ms SPIN invocations: K = 1 runs
their COMPUTE stages back to back without overlap; K = 2 never has more than
two at once; without a gate they overlap."""
import pytest

pytestmark = pytest.mark.gpu


def _max_overlap(spans):
    ev = sorted([(b, 1) for b, _ in spans] + [(e, -1) for _, e in spans], key=lambda x: (x[0], x[1]))
    cur = best = 0
    for _, d in ev:
        cur += d
        best = max(best, cur)
    return best


@pytest.mark.parametrize("slots", [1, 2, None])
def test_compute_gate_caps_concurrency(built, slots):
    from conftest import gpu_available
    from paper_2404_14691_b200.functions import Stage, load_spec_table
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table = load_spec_table({"spin": {"ro_mem_mb": 4, "writable_mem_mb": 1, "compute_ms": 3, "body": "spin"}})
    with Simulation(ClusterSpec(gpus=1, compute_concurrency=slots), policy_preset("SAGE"), table, seed=1) as sim:
        sim.submit_many(["spin"])            # warm: resident landed
        sim.drain()
        invs = sim.submit_many(["spin"] * 6)
        sim.drain()
        assert all(i.outcome == "completed" for i in invs)
        spans = [tuple(i.stages[Stage.COMPUTE]) for i in invs]
        assert all(e - b >= 2_500 for b, e in spans)           # each computes ~3 ms
        overlap = _max_overlap(spans)
        if slots is None:
            assert overlap >= 2          # (kernels on 8 hardware queues: some streams alias)
        else:
            assert overlap <= slots
            # FIFO: computes start in submission order
            starts = [b for b, _ in spans]
            assert starts == sorted(starts)

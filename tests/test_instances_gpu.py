"""Instance-per-invocation baselines on the device (csrc/fixedgsl.cu):
FixedGSL with a fresh context per instance -- on a library thread or in its
own OS process (sage_instance_worker) -- and DGSF in real pre-created CUDA
contexts.  Outputs and landed checksums must equal the oracle's; the stage
sets must be the reference's Serial plans (policies.py:102-276: FixedGSL
creates a GPU context per invocation, DGSF never does)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200.functions import Stage
from paper_2404_14691_b200.parboil import cfg2_functions
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation

pytestmark = pytest.mark.gpu


def check_outputs(invs, data):
    for i in invs:
        assert i.outcome == "completed", i.fail_reason
        fd = data[i.spec.name]
        lay = fd.layout
        seg, cs = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        assert i.ro_checksum == cs
        x = fd.input
        if fd.body == "sgemm":
            m, n, k = fd.args
            want = O.sgemm_ref(seg[:m * k * 4].view(np.float32).reshape(m, k), x.view(np.float32).reshape(n, k).T)
            np.testing.assert_allclose(i.result.view(np.float32).reshape(m, n), want, rtol=1e-3,
                                       atol=1e-4 * np.abs(want).max())
        elif fd.body == "stencil":
            nx, ny, nz, bits = fd.args
            want = O.stencil_ref(seg.view(np.float32)[:nx * ny * nz].reshape(nz, ny, nx),
                                 x.view(np.float32).reshape(nz, ny, nx), float(np.int32(bits).view(np.float32)))
            np.testing.assert_allclose(i.result.view(np.float32).reshape(nz, ny, nx), want, rtol=1e-3, atol=1e-5)
        else:
            rows, nnz, o_rp, o_col, o_val = fd.args
            want = O.spmv_ref(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32), seg[o_col:o_col + 4 * nnz].view(np.int32),
                              seg[o_val:o_val + 4 * nnz].view(np.float32), x.view(np.float32))
            np.testing.assert_allclose(i.result.view(np.float32)[:rows], want, rtol=1e-3, atol=1e-4)


@pytest.mark.parametrize("mode", ["thread", "process"])
def test_fixedgsl_fresh_context_instances(built, mode):
    table, data = cfg2_functions(scale=8)
    names = [sorted(table)[k % 3] for k in range(6)]
    with Simulation(ClusterSpec(gpus=1, instance_mode=mode), policy_preset("FixedGSL"), table, seed=1,
                    function_data=data) as sim:
        invs = sim.submit_many(names)
        sim.drain()
        check_outputs(invs, data)
        for i in invs:
            st = i.stages
            assert Stage.GPU_CTX in st and Stage.CPU_LOAD in st
            # serial: each stage after the previous one
            order = [Stage.CPU_CTX, Stage.CPU_LOAD, Stage.GPU_CTX, Stage.GPU_LOAD, Stage.COMPUTE, Stage.RETURN]
            ends = [st[s] for s in order]
            assert all(a[1] <= b[0] for a, b in zip(ends, ends[1:])), (mode, ends)
            assert i.setup_us >= st[Stage.GPU_CTX][1] - st[Stage.GPU_CTX][0] > 0
        sim.check_no_leaks()


def test_dgsf_runs_in_precreated_contexts(built):
    table, data = cfg2_functions(scale=8)
    names = [sorted(table)[k % 3] for k in range(9)]
    with Simulation(ClusterSpec(gpus=1), policy_preset("DGSF"), table, seed=1, function_data=data) as sim:
        handles = {c.handle for p in sim.policy.pools.values() for c in p.contexts}
        assert len(handles) == 3 * 4 and all(handles)           # 4 real contexts per function
        invs = sim.submit_many(names)
        sim.drain()
        check_outputs(invs, data)
        for i in invs:
            assert Stage.GPU_CTX not in i.stages and Stage.GPU_LOAD in i.stages
        # the contexts outlive the invocations and are reused
        assert {c.handle for p in sim.policy.pools.values() for c in p.contexts} == handles
        invs = sim.submit_many(names)
        sim.drain()
        check_outputs(invs, data)
        sim.check_no_leaks()

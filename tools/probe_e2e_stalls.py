"""Do e2e burst outliers correlate with the NVML clock sampler?  Runs the
bench's e2e leg (pinned store + pinned payloads) for N steps per mode:
sampler off / NVML every 5 ms / every 50 ms; prints step-time stats.
python tools/probe_e2e_stalls.py [steps]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
table, data = cfg2_functions()
names = bench.burst_names(table, 64)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
_lib.check(_lib.lib().sage_stats_enable(0), "stats")
pls = []
for n in names:
    pb = D.PinnedBuffer(data[n].input_bytes)
    pb.view()[:] = data[n].input
    pls.append(pb)
sim.dataplane.pin_host_store()
try:
    for mode in ("off", "nvml5", "nvml50", "off", "nvml5"):
        cs = None
        if mode != "off":
            cs = bench.ClockSampler(0)
            if mode == "nvml50":
                orig = cs._poll

                def slow(cs=cs):
                    nv, h, _ = cs._nvml
                    while not cs._stop.is_set():
                        cs.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                           nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                        cs._stop.wait(0.05)
                cs._poll = slow
            cs.start()
        us, _ = bench.timed(sim, names, steps, 3, None, pls)
        st = bench.timed.step_ms
        if cs is not None:
            cs.stop()
        print(json.dumps({"mode": mode, "mean_ms": round(us / steps / 1e3, 3), "max_ms": max(st),
                          "over_25ms": sum(x > 25 for x in st), "median_ms": sorted(st)[len(st) // 2]}), flush=True)
finally:
    sim.dataplane.unpin_host_store()
    sim.close()

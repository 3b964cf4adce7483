#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 120 python tools/probe_peak.py 32 400 800 1200
timeout 120 python tools/probe_peak.py 8 400 800 1200
SAGE_PINNED_SLABS=0 timeout 120 python tools/probe_peak.py 32 400 800 1200

#!/bin/bash
# compute-sanitizer memcheck over the smoke path and the body / land parity tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/sanitize_smoke.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --error-exitcode 9 python -m pytest tests/test_bodies_gpu.py tests/test_land_gpu.py -x -q -k "not two_gib and not hundred and not round_trip" > gpurun_out/sanitize_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/sanitize_tests.log
SAGE_LAND_TMA=1 timeout 900 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --error-exitcode 9 python -m pytest tests/test_land_gpu.py -x -q -k "random_layouts or golden" > gpurun_out/sanitize_tma.log 2>&1; echo "tma rc=$?"; tail -5 gpurun_out/sanitize_tma.log
# the column-sliced spmv (TMA ring, mbarriers, DSMEM slice sum): memcheck + racecheck + synccheck
timeout 900 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --error-exitcode 9 python -m pytest tests/test_bodies_gpu.py -x -q -k "csb and not 1048576" > gpurun_out/sanitize_csb_mem.log 2>&1; echo "csb memcheck rc=$?"; tail -3 gpurun_out/sanitize_csb_mem.log
timeout 900 compute-sanitizer --tool racecheck --report-api-errors no --error-exitcode 9 python -m pytest tests/test_bodies_gpu.py -x -q -k "csb and not 1048576 and not 65536" > gpurun_out/sanitize_csb_race.log 2>&1; echo "csb racecheck rc=$?"; tail -3 gpurun_out/sanitize_csb_race.log
timeout 900 compute-sanitizer --tool synccheck --report-api-errors no --error-exitcode 9 python -m pytest tests/test_bodies_gpu.py -x -q -k "csb and not 1048576 and not 65536" > gpurun_out/sanitize_csb_sync.log 2>&1; echo "csb synccheck rc=$?"; tail -3 gpurun_out/sanitize_csb_sync.log

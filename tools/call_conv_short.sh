#!/bin/bash
# conv: 2-stage short-K variants (two+ CTAs per SM) -- parity + sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SAGE_CONV_SHORT_ALL=1 SAGE_CONV_SHORT_KB=18 timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_dnn_gpu.py -x -q > gpurun_out/pytest_conv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_conv.log
tail -2 gpurun_out/pytest_conv.log
for cfg in "0 0" "8 0" "16 0" "8 1" "36 0"; do set -- $cfg
  echo "short_kb=$1 all=$2 $(SAGE_CONV_SHORT_KB=$1 SAGE_CONV_SHORT_ALL=$2 timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1)"
done | tee gpurun_out/conv_short_sweep3.txt

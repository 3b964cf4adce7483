#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for w in 0 1 2; do
  echo "waves=$w $(SAGE_CONV_WAVES=$w timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1)"
done | tee gpurun_out/conv_waves.txt

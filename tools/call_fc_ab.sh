#!/bin/bash
# A/B: _ab (HEAD: previous pool + fc) vs this tree, ResNet-50 forwards (1 and 16 streams), alternating
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
(cd _ab && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1) || { echo "ab build failed"; exit 1; }
for i in 1 2 3; do
  echo "old1 $(cd _ab && timeout 300 python tools/prof_resnet_native.py 8 1 20 | tail -1)"
  echo "new1 $(timeout 300 python tools/prof_resnet_native.py 8 1 20 | tail -1)"
  echo "old16 $(cd _ab && timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1)"
  echo "new16 $(timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1)"
done | tee gpurun_out/fc_ab.txt

#!/bin/bash
# ncu launch lists (duration + grid) of the bench at staged chunk 8 / 32 MiB: the e2e leg's chunk lands
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in 8 32; do
  timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ch$c.csv python bench.py --steps 2 --warmup 3 --no-cfg1 --no-cpu-baseline --chunk-mb $c > /dev/null 2>&1
  echo "== chunk $c"; python tools/launch_summary.py gpurun_out/launches_ch$c.csv | tail -8
done

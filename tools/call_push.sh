#!/bin/bash
# split-K reduction: push (st.async into the owner's smem, default) vs pull (SAGE_SGEMM_PULL=1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_bodies_gpu.py tests/test_runtime_gpu.py -x -q -k "sgemm" 2>&1 | tail -2
SAGE_SGEMM_PULL=1 timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k "sgemm" 2>&1 | tail -1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include tools/sgemm_host_cost.cu -o /tmp/shc -lcuda || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DSAGE_GEMM_TRACE tools/gemm_phases.cu -o /tmp/gemm_phases -lcuda || exit 1
for i in 1 2 3; do
  echo "push: $(timeout 60 /tmp/shc | head -1)"
  echo "pull: $(SAGE_SGEMM_PULL=1 timeout 60 /tmp/shc | head -1)"
done | tee gpurun_out/sgemm_push_ab.txt
echo "== push phases"; timeout 60 /tmp/gemm_phases | tee -a gpurun_out/sgemm_push_ab.txt
echo "== pull phases"; SAGE_SGEMM_PULL=1 timeout 60 /tmp/gemm_phases | tee -a gpurun_out/sgemm_push_ab.txt

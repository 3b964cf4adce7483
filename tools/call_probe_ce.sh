#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/probe_ce.py > gpurun_out/probe_ce.json 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 120 python tools/probe_ce.py > gpurun_out/probe_ce_32.json 2>&1
cat gpurun_out/probe_ce.json gpurun_out/probe_ce_32.json

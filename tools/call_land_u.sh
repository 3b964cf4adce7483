#!/bin/bash
for cfg in "4 4" "8 2" "8 3" "6 3"; do set -- $cfg
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2404_14691_b200/csrc -DSAGE_LAND_U=$1 -DSAGE_LAND_MINB=$2 tools/land_micro.cu -o /tmp/lm_$1_$2 2>/dev/null
echo "U=$1 MINB=$2"; /tmp/lm_$1_$2 | grep '"land_u4"'; /tmp/lm_$1_$2 104857600 | grep '"land_u4"'
done

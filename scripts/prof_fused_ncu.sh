#!/bin/bash
# ncu --set full of the k_code_fused main launch (config 1, 45 samples) with source-level SASS
# counts; run from the repo root on the GPU box.  Output: gpurun_out/$1.ncu-rep
set -e
name=${1:-fused}
ncu --set full --clock-control none --import-source on -k regex:k_code_fused -s 2 -c 1 \
    -o gpurun_out/$name -f python scripts/prof_fused.py > gpurun_out/$name.log 2>&1

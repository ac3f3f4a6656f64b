#!/bin/bash
# fusion-depth sweep + ncu --set full (with source) of the S=2 fused kernel
mkdir -p gpurun_out
bash scripts/tune_variants.sh
QUAPI_FUSE_S=${PROF_S:-2} ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 2 -o gpurun_out/prof_fused -f \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fused.log 2>&1
tail -2 gpurun_out/ncu_fused.log

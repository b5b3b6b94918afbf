#!/bin/bash
# Runs on the GPU box: bench line, per-launch device times, one ncu --set full
# capture of the hot kernels.  Outputs into gpurun_out/prof/.
set -x
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/prof/gpu.txt
timeout 600 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    --depth 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"k_raster_quad|k_preprocess|k_col_pass|k_row_pass|k_depth_pass|k_pair_scan|k_depth_fixup|k_depth_hist" -s 40 -c 10 \
    -o gpurun_out/prof/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --depth 1 \
    > gpurun_out/prof/ncu_full.log 2>&1
cuobjdump -sass paper_2503_05168_b200/libseele_b200.so > gpurun_out/prof/sass.txt 2>/dev/null

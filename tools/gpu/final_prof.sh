# round evidence: bench line, launch list, one ncu --set full capture of every kernel of a C3 frame, a C4 raster capture
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches_final.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    --no-exact --depth 1 > /dev/null 2>&1; echo "launch list rc=$?"
python tools/launches.py gpurun_out/launches_final.csv
SKIP=44 COUNT=12 bash tools/gpu/prof_full.sh final 'k_'
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_raster_quad|k_preprocess|k_bin_expand" -s 6 -c 3 \
    -o gpurun_out/full_c4 python bench.py --n 6000000 --width 3840 --height 2160 --flat --steps 2 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 --no-exact --depth 1 > gpurun_out/full_c4.log 2>&1; echo "c4 ncu rc=$?"; tail -3 gpurun_out/full_c4.log

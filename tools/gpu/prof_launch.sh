# per-kernel device times of the C3 bench (ncu launch list, serialised, cold caches)
tag=${1:-x}
shift
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    --no-exact --depth 1 "$@" > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_$tag.csv

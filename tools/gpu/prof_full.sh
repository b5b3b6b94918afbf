# one ncu --set full capture of the kernels matching $2 (C3 bench, few frames), report $1
tag=$1; pat=$2; shift 2
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$pat" -s ${SKIP:-20} -c ${COUNT:-2} \
    -o gpurun_out/full_$tag python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-exact --depth 1 "$@" \
    > gpurun_out/full_$tag.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/full_$tag.log

# compute-sanitizer over a GPU-parity subset (every kernel of the render path incl. the fallbacks)
mkdir -p gpurun_out/san
K="small_cases_vs_reference and (rand64_s0 or edges80x48 or odd100x70) or random_scenes_vs_oracle or config1 or test_gpu_depth or overflow or no_binned or contribution_matrix"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 200 --error-exitcode 99 \
     python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/$tool.log | tail -3
done

# quick parity subset + bench A/B of the current build
python -m pytest tests -m gpu -q -x -k "small_cases or random_scenes or config1 or large_synth or c3_frames or fast_equals or depth or edge" > gpurun_out/quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/quick.log
bash tools/gpu/ab.sh base "$@"

python -m pytest tests -m gpu -q -x -k "small_cases or random_scenes or config1 or large_synth or fast_equals or edge" > gpurun_out/rab_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/rab_tests.log
bash tools/gpu/ab.sh base old pipe6 pipe5

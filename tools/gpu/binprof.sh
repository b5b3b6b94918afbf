python -m pytest tests -m gpu -q -x -k "small_cases or config1 or large_synth or c4 or c5 or overflow or plan or c3_frames" > gpurun_out/bp_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/bp_tests.log
SKIP=${SKIP:-30} COUNT=${COUNT:-7} bash tools/gpu/prof_full.sh bin 'k_bin'
bash tools/gpu/prof_launch.sh bp

# configuration sweep (C1-C5), streaming overhead, sanitizer summary
python tools/configs.py > gpurun_out/configs.log 2>&1; echo "configs rc=$?"; cat gpurun_out/configs.log
python tools/streaming_overhead.py > gpurun_out/streaming.log 2>&1; echo "streaming rc=$?"; tail -4 gpurun_out/streaming.log
TOOLS="memcheck racecheck synccheck" bash tools/gpu/sanitize.sh

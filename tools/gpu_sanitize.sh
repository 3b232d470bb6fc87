mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 240 compute-sanitizer --tool $tool --error-exitcode 3 python tools/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.txt
done
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader

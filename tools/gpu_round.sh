set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
for c in cfg2 cfg3 cfg4 cfg5 cfg1; do timeout 600 python bench.py --config $c $([ $c = cfg2 ] || echo --no-cpu) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 600 gpurun_out/bench_$c.json; done
timeout 900 bash tools/profile.sh cfg2 r03

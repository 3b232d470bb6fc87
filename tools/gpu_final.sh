# round-end style check without profilers: gpu tests, smoke, default bench, per-config bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in cfg2 cfg3 cfg4 cfg5 cfg1; do
  timeout 600 python bench.py --config $c $([ $c = cfg2 ] || echo --no-cpu) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['breakdown_ms'], (d.get('e2e') or {}).get('value'))"
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json

# GPU check: full gpu tests, smoke, default bench, other configs (no profilers)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in ${CFGS:-cfg2 cfg3 cfg4 cfg5 cfg5-hwt}; do
  timeout 900 python bench.py --config $c $([ $c = cfg2 ] || echo --no-cpu) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], {k: v for k, v in d.get('breakdown_ms', {}).items()}, 'frac', d['roofline']['frac'], 'warm', d.get('warm_l2_ms'), 'perm', d.get('perm_ms'), 'mask', d.get('mask_build_ms'), 'e2e', (d.get('e2e') or {}).get('value'))" || tail -5 gpurun_out/bench_$c.err
done
[ -n "$REF" ] && timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json

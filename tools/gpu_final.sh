# round-end style run without profilers: gpu tests, smoke, the default bench line, per-config
# lines, the oracle arm.  TAG names the saved JSON (gpurun_out/bench_<cfg>_<TAG>.json).
T=${TAG:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default_$T.json 2> gpurun_out/bench_default_$T.err
tail -1 gpurun_out/bench_default_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['breakdown_ms'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'))"
for c in cfg3 cfg4 cfg5 cfg5-hwt cfg1; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_${c}_$T.json 2> gpurun_out/bench_${c}_$T.err
  tail -1 gpurun_out/bench_${c}_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['breakdown_ms'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'))"
done
for c in cfg4 cfg5; do
  b=$([ $c = cfg4 ] && echo 64 || echo 128)
  timeout 600 python bench.py --config $c --block $b --no-cpu --no-e2e --no-variants > gpurun_out/bench_${c}_b${b}_$T.json 2> gpurun_out/bench_${c}_b${b}_$T.err
  tail -1 gpurun_out/bench_${c}_b${b}_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c b$b', d['value'], d['breakdown_ms'], d['roofline']['frac'])"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; tail -c 300 gpurun_out/bench_ref_$T.json

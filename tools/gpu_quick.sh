# quick GPU check under gpurun: full gpu tests + short benches (no variants / oracle / e2e)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in ${CFGS:-cfg2 cfg3 cfg4}; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e ${BENCH_ARGS:---no-variants} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['breakdown_ms'], 'frac', d['roofline']['frac'], {k:v.get('ms_per_step') for k,v in d.get('variants',{}).items() if isinstance(v,dict)})"
done

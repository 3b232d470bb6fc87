mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for a in "cfg4 --block 64" "cfg5" "cfg2"; do
  set -- $a
  timeout 900 python bench.py --config $a --no-cpu > gpurun_out/bench_$1$2$3.json 2> gpurun_out/bench_$1.err
  tail -1 gpurun_out/bench_$1$2$3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', d['value'], d['breakdown_ms'], 'frac', d['roofline']['frac'], 'tiles', d['config'].get('mask'), 'tpct', d.get('tensor_pct_executed'))" || tail -3 gpurun_out/bench_$1.err
done
ncu --query-metrics-mode all 2>/dev/null | grep -i -E "tensor|umma|utc|tcgen" > gpurun_out/ncu_tensor_metrics.txt
wc -l gpurun_out/ncu_tensor_metrics.txt

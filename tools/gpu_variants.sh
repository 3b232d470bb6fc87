# bench the default build and dev variants (libhla_<name>.so) back to back: VARIANTS="w1 w2" CFGS="cfg2 cfg3"
for v in default ${VARIANTS}; do
  for c in ${CFGS:-cfg2}; do
    if [ "$v" = default ]; then unset HLA_LIB_NAME; else export HLA_LIB_NAME=libhla_$v.so; fi
    timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-variants 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['value'], d['breakdown_ms'])"
  done
done

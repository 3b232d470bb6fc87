# bwd decomposition: default build + `make VARIANT=vN DEFS=-DHLA_BWD_VAR=N` builds,
# and the wait accounting of the HLA_BWD_PROF build
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
[ -n "$TESTS" ] && timeout 900 python -m pytest tests -m gpu -x -q $TESTS 2>&1 | tail -5
for v in default ${VARIANTS:-v1 v2 v8 v14 v15}; do
  if [ $v = default ]; then unset HLA_LIB_NAME; else export HLA_LIB_NAME=libhla_$v.so; fi
  timeout 300 python tools/probe_bwd_decomp.py 2>&1 | tail -1
done | tee gpurun_out/decomp_${TAG:-x}.txt
[ -f paper_2511_05832_b200/libhla_bprof.so ] && HLA_LIB_NAME=libhla_bprof.so timeout 300 python tools/probe_bwd_prof.py cfg2 cfg3 cfg4 dense2 2>&1 | tail -4 | tee gpurun_out/prof_${TAG:-x}.txt
[ -f paper_2511_05832_b200/libhla_fprof.so ] && HLA_LIB_NAME=libhla_fprof.so timeout 300 python tools/probe_fwd_prof.py cfg2 cfg3 cfg4 dense2 2>&1 | tail -8 | tee gpurun_out/fprof_${TAG:-x}.txt

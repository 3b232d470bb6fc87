#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU).
#   launches_<cfg>_<tag>.csv : every launch of our kernels with its device time
#                              (cold-cache, serialised -> compare SHARES, not absolutes)
#   prof_<cfg>_<kernel>_<tag>.ncu-rep : --set full capture of each hot kernel
CFG=${1:-cfg2}
TAG=${2:-r01}
B="python bench.py --config $CFG --steps 3 --warmup 1 --no-variants --no-cpu --no-e2e"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:attn_|hilbert_|bwd_pre|dq_fin" -c 200 --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $B > /dev/null 2>&1
for k in attn_bwd_kernel attn_fwd_kernel bwd_preprocess_kernel dq_finalize_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${CFG}_${k}_${TAG} -f $B > /dev/null 2>&1
done
ls gpurun_out

#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU).
#   launches_<cfg>_<tag>.csv : every launch of our kernels with its device time and DRAM bytes
#                              (cold-cache, serialised -> compare SHARES, not absolutes)
#   prof_<cfg>_<kernel>_<tag>.ncu-rep : --set full capture of each hot kernel
# usage: tools/profile.sh <cfg> <tag> [extra bench.py args, e.g. --block 64]
CFG=${1:-cfg2}
TAG=${2:-r01}
shift 2
B="python bench.py --config $CFG --steps 3 --warmup 1 --no-variants --no-cpu --no-e2e $*"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor.sum
ncu --metrics $M --clock-control none \
    -k "regex:attn_|hilbert_|bwd_pre|dq_fin|dq_zero" -c 400 --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $B > /dev/null 2>&1
for k in ${KERNELS:-attn_bwd_full_kernel attn_bwd_split_kernel attn_fwd_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${CFG}_${k}_${TAG} -f $B > /dev/null 2>&1
done
ls gpurun_out

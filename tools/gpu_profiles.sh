# ncu launch lists (time, DRAM bytes, tensor-path ops) + full captures for the bench configs.
# The full captures are summarised on the box (tools/ncu_summary.py) and only the cfg2 reports
# are kept, so gpurun_out/ stays under the 64 MiB copy-back limit.
T=${TAG:-r2}
bash tools/profile.sh cfg2 $T
bash tools/profile.sh cfg3 $T
bash tools/profile.sh cfg4 $T
bash tools/profile.sh cfg4 ${T}b64 --block 64
KERNELS="attn_bwd_split_kernel attn_fwd_kernel" bash tools/profile.sh cfg5 $T
KERNELS="attn_bwd_split_kernel attn_fwd_kernel" bash tools/profile.sh cfg5-hwt $T
python tools/ncu_summary.py gpurun_out/prof_*_${T}*.ncu-rep > gpurun_out/ncu_full_${T}.md 2> gpurun_out/ncu_full_${T}.err
for f in gpurun_out/launches_*_${T}*.csv; do echo "== $f"; python tools/launch_summary.py $f; done > gpurun_out/launches_${T}.txt 2>&1
find gpurun_out -name "prof_*_${T}*.ncu-rep" ! -name "prof_cfg2_*" -delete
ls -la gpurun_out | head -40

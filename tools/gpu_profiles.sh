# ncu launch lists (time, DRAM bytes, tensor-path ops) + full captures for the bench configs
T=${TAG:-r2}
bash tools/profile.sh cfg2 $T
bash tools/profile.sh cfg3 $T
bash tools/profile.sh cfg4 ${T}b64 --block 64
KERNELS="attn_bwd_split_kernel attn_fwd_kernel" bash tools/profile.sh cfg5 $T
KERNELS="attn_bwd_split_kernel" bash tools/profile.sh cfg5-hwt $T
ls -la gpurun_out | head -40

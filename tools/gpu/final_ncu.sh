# ncu evidence on HEAD: launch list, GEMM DRAM traffic, --set full captures (tools/ncu_profile.sh)
mkdir -p gpurun_out
bash tools/ncu_profile.sh r4l

set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_attn_(fwd|bwd)$" -s 2 -c 2 -o gpurun_out/prof_attn_r2k python tools/prof_attn.py > gpurun_out/ncu_attn_r2k.log 2>&1

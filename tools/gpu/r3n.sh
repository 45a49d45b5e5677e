set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_attn_fwd" -s 1 -c 1 -o gpurun_out/prof_attn_fwd_r3n python tools/prof_attn.py > gpurun_out/ncu_attn_r3n.log 2>&1

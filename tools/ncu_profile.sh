#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, 1 GPU; never multi-rank).
#   tools/ncu_profile.sh <tag>
# 1) every library launch of one bench step with its device time (cold-cache, serialised)
# 2) DRAM bytes of all 14 GEMM launches of one step (-> profiles/traffic.json)
# 3) one `--set full` capture each of the q-projection fwd/bwd GEMM, the forward shrink (q/k/v
#    group and down), the token reduction and the fused backward dY pass.
set -x
TAG=${1:-r1}
OUT=gpurun_out
K="regex:k_(gemm|gemm2|rowproj|shrink|shrink_planes|segred|finalize|finalize_multi|pad_cols|transpose_b|dypass|gfin|pack_a_group|meta_copy)"
B="python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
    --log-file $OUT/launches_$TAG.csv $B > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_gemm2 -s 14 -c 14 --csv --log-file $OUT/gemm_traffic_$TAG.csv \
    $B > $OUT/ncu_traffic_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm2 -s 0 -c 1 \
    -o $OUT/prof_gemm_fwd_$TAG $B > $OUT/ncu_gemm_fwd_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm2 -s 7 -c 1 \
    -o $OUT/prof_gemm_bwd_$TAG $B > $OUT/ncu_gemm_bwd_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_shrink -s 0 -c 1 \
    -o $OUT/prof_shrink_$TAG $B > $OUT/ncu_shrink_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_shrink -s 3 -c 1 \
    -o $OUT/prof_shrink_down_$TAG $B > $OUT/ncu_shrink_down_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segred -s 0 -c 1 \
    -o $OUT/prof_segred_$TAG $B > $OUT/ncu_segred_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dypass -s 0 -c 1 \
    -o $OUT/prof_dypass_$TAG $B > $OUT/ncu_dypass_$TAG.log 2>&1
ls -la $OUT

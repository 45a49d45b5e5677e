B="python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e"
for s in 4 6 11 13; do
timeout 600 ncu --set full --clock-control none -k regex:k_gemm2 -s $s -c 1 -o gpurun_out/prof_gemm_s${s}_r1c $B > gpurun_out/ncu_big_$s.log 2>&1
done

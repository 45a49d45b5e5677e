# GEMM raster: DRAM bytes per launch for more K = 11008 / N = 11008 orders, then A/B bench runs
set -x
mkdir -p gpurun_out
for cfg in "NBIG=16 KBIG=-8" "NBIG=16 KBIG=-6" "NBIG=8 KBIG=1" "NBIG=12 KBIG=-12"; do
  set -- $cfg
  n=${1#NBIG=}; k=${2#KBIG=}
  LOBRA_GEMM_GM_NBIG=$n LOBRA_GEMM_GM_KBIG=$k timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_gemm2 -s 14 -c 14 --csv --log-file gpurun_out/r2v_traffic_n${n}_k${k}.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2>&1
done
for r in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-c2 > gpurun_out/r2v_bench_default_$r.json 2>/dev/null
  LOBRA_GEMM_GM_KBIG=-8 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-c2 > gpurun_out/r2v_bench_k-8_$r.json 2>/dev/null
done

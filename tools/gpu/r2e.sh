set -x
python tools/gemm_raster_sweep.py --rounds 3 > gpurun_out/r2e_raster.jsonl 2> gpurun_out/r2e_raster.err
for cfg in "NBIG=16 KBIG=16" "NBIG=32 KBIG=1" "NBIG=-2 KBIG=-2" "NBIG=64 KBIG=-4" "NBIG=24 KBIG=2"; do
  set -- $cfg
  n=${1#NBIG=}; k=${2#KBIG=}
  LOBRA_GEMM_GM_NBIG=$n LOBRA_GEMM_GM_KBIG=$k timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_gemm2 -s 14 -c 14 --csv --log-file gpurun_out/r2e_traffic_n${n}_k${k}.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2>&1
done

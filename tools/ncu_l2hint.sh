# GEMM DRAM traffic and duration under the LOBRA_GEMM_L2HINT probe (ncu, 14 GEMMs of one step)
OUT=gpurun_out
for h in 0 1 2 3; do
  LOBRA_GEMM_L2HINT=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_gemm2 -s 14 -c 14 --csv --log-file $OUT/l2hint_$h.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2>&1
done
for h in 0 1 2 0 1 2; do
  LOBRA_GEMM_L2HINT=$h timeout 300 python bench.py --no-cpu --no-e2e --no-kernel-events 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('hint', $h, round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> $OUT/l2hint_bench.txt
done

set -x
python -m pytest tests/test_gpu_layer_parity.py -k launch_counter -x -q 2>&1 | tail -5 > gpurun_out/r2d_gputests.txt
python tools/gemm_raster_sweep.py --values 1,2,3,4,6,8,12,16,32 > gpurun_out/r2d_raster.jsonl 2> gpurun_out/r2d_raster.err
for gm in 1 4 6 16; do
  LOBRA_GEMM_GROUP_M=$gm timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_gemm2 -s 14 -c 14 --csv --log-file gpurun_out/r2d_traffic_gm$gm.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2>&1
done

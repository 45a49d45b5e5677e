set -x
python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py tests/test_gpu_layer_parity.py tests/test_gpu_tp70b.py -x -q 2>&1 | tail -5 > gpurun_out/r2g_gputests.txt
bash tools/ncu_skinny.sh r2g_c3
bash tools/ncu_skinny.sh r2g_c2 --workload c2
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err

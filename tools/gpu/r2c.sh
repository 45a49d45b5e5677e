set -x
python -m pytest tests/test_gpu_layer_parity.py tests/test_gpu_bench_dist.py -x -q 2>&1 | tail -15 > gpurun_out/r2c_gputests.txt
bash tools/ncu_skinny.sh r2c_c3
bash tools/ncu_skinny.sh r2c_c2 --workload c2
bash tools/ncu_profile.sh r2c

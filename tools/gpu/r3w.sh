set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_symm.py tests/test_gpu_comm.py tests/test_gpu_bench_dist.py -x -q > gpurun_out/r3w_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3w_tests.txt

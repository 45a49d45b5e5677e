set -x
mkdir -p gpurun_out
LOBRA_E2E_TRACE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-c2 > gpurun_out/r3s_e2e.json 2> gpurun_out/r3s_e2e.err
timeout 900 python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py -x -q > gpurun_out/r3s_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3s_tests.txt

set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_group.py tests/test_gpu_lora.py tests/test_gpu_layer_parity.py -x -q > gpurun_out/r3k_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests.txt
bash tools/ncu_skinny.sh r3k_c3

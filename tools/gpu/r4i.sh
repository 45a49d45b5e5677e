mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py tests/test_gpu_guards.py -x -q > gpurun_out/r4i_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r4i_tests.txt
bash tools/ncu_skinny.sh r4i_c3
bash tools/ncu_skinny.sh r4i_c2 --workload c2

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guards.py -q -rs > gpurun_out/r4e_guards.txt 2>&1; echo "rc=$?" >> gpurun_out/r4e_guards.txt

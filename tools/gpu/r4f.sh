mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_group.py tests/test_gpu_guards.py tests/test_gpu_layer_parity.py tests/test_gpu_decoder.py -x -q > gpurun_out/r4f_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r4f_tests.txt
bash tools/ncu_skinny.sh r4f_c3
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r4f_bench.json 2> gpurun_out/r4f_bench.err

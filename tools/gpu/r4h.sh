mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py tests/test_gpu_guards.py tests/test_gpu_layer_parity.py tests/test_gpu_trainer.py tests/test_gpu_tp70b.py -x -q > gpurun_out/r4h_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r4h_tests.txt
bash tools/ncu_skinny.sh r4h_c3
bash tools/ncu_skinny.sh r4h_c2 --workload c2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r4h_bench.json 2> gpurun_out/r4h_bench.err

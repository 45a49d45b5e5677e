set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py tests/test_gpu_layer_parity.py tests/test_gpu_tp70b.py -x -q > gpurun_out/r2x_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2x_tests.txt
rm -f gpurun_out/dy_trace_x.jsonl
LOBRA_TRACE_DY=gpurun_out/dy_trace_x.jsonl timeout 600 python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2> gpurun_out/r2x.err
python tools/trace_dy.py gpurun_out/dy_trace_x.jsonl > gpurun_out/r2x_dy.txt 2>&1
bash tools/ncu_skinny.sh r2x_c3
bash tools/ncu_skinny.sh r2x_c2 --workload c2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err

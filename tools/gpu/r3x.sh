set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py tests/test_gpu_layer_parity.py -x -q > gpurun_out/r3x_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3x_tests.txt
rm -f gpurun_out/dy_trace_r3x.jsonl
LOBRA_TRACE_DY=gpurun_out/dy_trace_r3x.jsonl timeout 600 python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2> gpurun_out/r3x.err
python tools/trace_dy.py gpurun_out/dy_trace_r3x.jsonl > gpurun_out/r3x_dy.txt 2>&1
bash tools/ncu_skinny.sh r3x_c3

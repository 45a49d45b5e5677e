set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lora.py tests/test_gpu_group.py tests/test_gpu_layer_parity.py tests/test_gpu_attn.py tests/test_gpu_decoder.py -x -q > gpurun_out/r2y_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2y_tests.txt
rm -f gpurun_out/dy_trace_y.jsonl
LOBRA_TRACE_DY=gpurun_out/dy_trace_y.jsonl timeout 600 python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2> gpurun_out/r2y.err
python tools/trace_dy.py gpurun_out/dy_trace_y.jsonl > gpurun_out/r2y_dy.txt 2>&1
timeout 600 python tools/bench_attn.py > gpurun_out/r2y_bench_attn.txt 2>&1
LOBRA_TRACE_ATTN=gpurun_out/attn_trace_fwd_raw.txt timeout 300 python tools/trace_attn_fwd.py > gpurun_out/r2y_trace_fwd.txt 2>&1

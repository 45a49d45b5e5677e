set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q > gpurun_out/r2o_attn_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2o_attn_tests.txt
LOBRA_TRACE_ATTN=gpurun_out/attn_trace_raw.txt timeout 300 python tools/trace_attn.py > gpurun_out/r2o_trace.txt 2>&1
timeout 600 python tools/bench_attn.py > gpurun_out/r2o_bench_attn.txt 2>&1

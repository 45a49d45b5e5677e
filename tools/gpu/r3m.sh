set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_decoder.py -x -q > gpurun_out/r3m_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.txt
timeout 600 python tools/bench_attn.py > gpurun_out/r3m_bench_attn.txt 2>&1
LOBRA_TRACE_ATTN=gpurun_out/attn_trace_fwd_raw.txt timeout 300 python tools/trace_attn_fwd.py > gpurun_out/r3m_trace_fwd.txt 2>&1

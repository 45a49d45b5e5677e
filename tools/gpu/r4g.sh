mkdir -p gpurun_out
LOBRA_ATTN_DQ_TMA=1 timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_guards.py -x -q -k "attn or attention" > gpurun_out/r4g_tests_tma.txt 2>&1; echo "rc=$?" >> gpurun_out/r4g_tests_tma.txt
timeout 600 python tools/bench_attn.py > gpurun_out/r4g_bench_attn_red.txt 2>&1
LOBRA_ATTN_DQ_TMA=1 timeout 600 python tools/bench_attn.py > gpurun_out/r4g_bench_attn_tma.txt 2>&1

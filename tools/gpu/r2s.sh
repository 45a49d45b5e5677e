set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_decoder.py -x -q > gpurun_out/r2s_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.txt
timeout 600 python tools/bench_attn.py > gpurun_out/r2s_bench_attn.txt 2>&1

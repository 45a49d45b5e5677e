# own attention backward: parity + timing vs cuDNN / FA2
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q > gpurun_out/r2j_attn_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2j_attn_tests.txt
timeout 600 python tools/bench_attn.py > gpurun_out/r2j_bench_attn.txt 2>&1

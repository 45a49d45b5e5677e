set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_decoder.py -x -q > gpurun_out/r3f_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3f_tests.txt

set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_decoder.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r3u_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3u_tests.txt
timeout 600 python tools/bench_layer.py --attn lobra > gpurun_out/r3u_layer_lobra.txt 2>&1
timeout 600 python tools/bench_layer.py --attn cudnn > gpurun_out/r3u_layer_cudnn.txt 2>&1

# NEXT-3 decoder layer (7B, cuDNN vs own attention; 70B GQA) and C4 70B TP shards, per rank
mkdir -p gpurun_out
TAG=${1:-layer}
for a in cudnn lobra; do
  timeout 600 python tools/bench_layer.py --attn $a --steps 10 > gpurun_out/${TAG}_layer7b_$a.txt 2>&1
done
timeout 600 python tools/bench_layer.py --attn cudnn --model 70b --steps 5 > gpurun_out/${TAG}_layer70b_cudnn.txt 2>&1
timeout 900 python tools/bench_tp_shapes.py --steps 10 > gpurun_out/${TAG}_tp_shapes.txt 2>&1

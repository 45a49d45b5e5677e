set -x
mkdir -p gpurun_out
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export LOBRA_META_MEMCPY=1; else unset LOBRA_META_MEMCPY; fi
  timeout 600 python tools/bench_layer.py --attn cudnn >> gpurun_out/r3v_layer_memcpy$v.txt 2>&1
done

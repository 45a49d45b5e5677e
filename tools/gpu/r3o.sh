set -x
mkdir -p gpurun_out
timeout 300 python tools/probe_h2d.py > gpurun_out/r3o_h2d.txt 2>&1
nvidia-smi topo -m > gpurun_out/r3o_topo.txt 2>&1
nproc >> gpurun_out/r3o_topo.txt; lscpu | head -30 >> gpurun_out/r3o_topo.txt 2>&1

# NVSwitch multicast (NVLS) availability on the box: fabric state, topology, tools/probe_nvls.cu
#   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_nvls_bin tools/probe_nvls.cu -L/usr/local/cuda/lib64/stubs -lcuda
mkdir -p gpurun_out
( nvidia-smi -q | grep -i -A4 "fabric"; nvidia-smi topo -m; timeout 120 ./tools/probe_nvls_bin ) > gpurun_out/nvls_probe.txt 2>&1

mkdir -p gpurun_out
( nvidia-smi -q | grep -i -A4 "fabric"; nvidia-smi topo -m; timeout 120 ./tools/probe_nvls_bin ) > gpurun_out/r4b_nvls.txt 2>&1

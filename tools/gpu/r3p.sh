set -x
mkdir -p gpurun_out
timeout 600 python tools/probe_e2e_copy.py > gpurun_out/r3p_copy.txt 2>&1

set -x
mkdir -p gpurun_out
LOBRA_TRACE_ATTN=gpurun_out/attn_trace_raw.txt timeout 300 python tools/trace_attn.py > gpurun_out/r2p_trace.txt 2>&1

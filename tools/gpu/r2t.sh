set -x
mkdir -p gpurun_out
LOBRA_TRACE_ATTN=gpurun_out/attn_trace_fwd_raw.txt timeout 300 python tools/trace_attn_fwd.py > gpurun_out/r2t_trace_fwd.txt 2>&1

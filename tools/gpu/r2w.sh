set -x
mkdir -p gpurun_out
rm -f gpurun_out/dy_trace.jsonl
LOBRA_TRACE_DY=gpurun_out/dy_trace.jsonl timeout 600 python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2> gpurun_out/r2w.err
python tools/trace_dy.py gpurun_out/dy_trace.jsonl > gpurun_out/r2w_dy.txt 2>&1
rm -f gpurun_out/dy_trace_c2.jsonl
LOBRA_TRACE_DY=gpurun_out/dy_trace_c2.jsonl timeout 600 python bench.py --workload c2 --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > /dev/null 2>> gpurun_out/r2w.err
python tools/trace_dy.py gpurun_out/dy_trace_c2.jsonl > gpurun_out/r2w_dy_c2.txt 2>&1

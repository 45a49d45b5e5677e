set -x
mkdir -p gpurun_out
nproc > gpurun_out/r3z_nproc.txt
timeout 900 python tools/dispatch_solve_times.py > gpurun_out/r3z_dispatch_solve_times.md 2>&1

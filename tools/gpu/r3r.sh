set -x
mkdir -p gpurun_out
LOBRA_E2E_TRACE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-c2 > gpurun_out/r3r_e2e.json 2> gpurun_out/r3r_e2e.err

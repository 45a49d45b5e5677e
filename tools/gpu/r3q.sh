set -x
mkdir -p gpurun_out
for cs in 2 4; do
  LOBRA_E2E_COPY_STREAMS=$cs timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-c2 > gpurun_out/r3q_e2e_cs$cs.json 2> gpurun_out/r3q_e2e_cs$cs.err
done

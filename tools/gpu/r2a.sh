set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_gputests.txt
python bench.py --steps 10 --warmup 3 --workload c3 > gpurun_out/r2a_bench_c3.json 2> gpurun_out/r2a_bench_c3.err
python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err
tail -3 gpurun_out/r2a_gputests.txt

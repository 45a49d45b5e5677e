# full GPU suite, smoke, default bench (C3 + C2), launch list + skinny DRAM tables
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3e_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3e_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err
bash tools/ncu_skinny.sh r3e_c3
bash tools/ncu_skinny.sh r3e_c2 --workload c2

# round 2 re-entry: GPU tests, smoke, default bench (C3 headline + C2 beside), ncu evidence
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2h_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
bash tools/ncu_profile.sh r2h

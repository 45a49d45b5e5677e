# round-2 final evidence: full GPU suite, smoke, default bench, ncu launch list + GEMM traffic + --set full captures
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3j_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3j_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3j_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3j_bench.json 2> gpurun_out/r3j_bench.err
bash tools/ncu_profile.sh r3j

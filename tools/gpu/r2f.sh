set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2f_gputests.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.txt 2>&1

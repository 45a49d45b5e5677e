set -x
python -m pytest tests/test_gpu_trainer.py tests/test_optim.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2b_gputests.txt
python tools/bench_tp_shapes.py --model 7b --workload c3 --tps 1,2,4,8 --chunk 8192,16384,32768,32768 --steps 10 > gpurun_out/r2b_tp_costs_7b.jsonl 2> gpurun_out/r2b_tp.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_ref.json 2>&1

# final evidence after the metadata-upload change: full GPU suite, smoke, default bench, launch list
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r4k_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/r4k_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4k_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r4k_bench.json 2> gpurun_out/r4k_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r4k_ref.json 2> gpurun_out/r4k_ref.err
K="regex:k_(gemm|gemm2|rowproj|shrink|shrink_planes|segred|finalize|finalize_multi|pad_cols|transpose_b|dypass|gfin|pack_a_group|meta_copy)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_r4k.csv python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > gpurun_out/ncu_launch_r4k.log 2>&1
bash tools/ncu_skinny.sh r4k_c3; bash tools/ncu_skinny.sh r4k_c2 --workload c2

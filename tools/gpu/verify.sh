# Full verification on one B200 (run under gpurun): GPU test suite, smoke, default bench line,
# reference arm, ncu launch list of one bench step, memory-bound kernel tables (C3, C2).
#   gpurun --timeout 3600 -- 'bash tools/gpu/verify.sh <tag>'
set -x
TAG=${1:-verify}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputests.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
K="regex:k_(gemm|gemm2|rowproj|shrink|shrink_planes|segred|finalize|finalize_multi|pad_cols|transpose_b|dypass|gfin|pack_a_group|meta_copy)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1
bash tools/ncu_skinny.sh ${TAG}_c3; bash tools/ncu_skinny.sh ${TAG}_c2 --workload c2

# durations of the memory-bound kernels of one bench step (ncu, serialised, cold cache)
#   tools/ncu_skinny.sh <tag> [extra bench.py args, e.g. --workload c3]
TAG=${1:-x}
shift
OUT=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(shrink|shrink_planes|rowproj|dypass|gfin|segred|finalize|pack_a_group|meta_copy)" --csv --log-file $OUT/skinny_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --profile-only --no-cpu --no-e2e "$@" > $OUT/skinny_$TAG.log 2>&1

# round-2 kernels under compute-sanitizer (memcheck / synccheck / racecheck), small cases
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20 --error-exitcode 7"
run() { name=$1; shift; timeout 1500 $CS "$@" > gpurun_out/r4d_$name.log 2>&1; echo "$name rc=$?" >> gpurun_out/r4d_summary.txt; }
: > gpurun_out/r4d_summary.txt
run memcheck_lora --tool memcheck python -m pytest tests/test_gpu_lora.py -q -x -k "edge_cases or medium or empty"
run memcheck_group --tool memcheck python -m pytest tests/test_gpu_group.py -q -x -k "not full_size and not full_batch and not c3"
run memcheck_attn --tool memcheck python -m pytest tests/test_gpu_attn.py -q -x -k "oracle"
run memcheck_layerops --tool memcheck python -m pytest tests/test_gpu_layer_ops.py -q -x
run synccheck_attn --tool synccheck python -m pytest tests/test_gpu_attn.py -q -x -k "bwd_matches_oracle"
run racecheck_attn --tool racecheck python -m pytest tests/test_gpu_attn.py -q -x -k "bwd_matches_oracle"
run racecheck_lora --tool racecheck python -m pytest tests/test_gpu_lora.py -q -x -k "bf16_medium"
run racecheck_group --tool racecheck python -m pytest tests/test_gpu_group.py -q -x -k "group_equals_single_sequence_bitwise"

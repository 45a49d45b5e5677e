set -x
OUT=gpurun_out
for d in 0 1 4 7; do
  LOBRA_DBG_RP=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__cycles_active.avg --clock-control none -k regex:k_rowproj -s 3 -c 3 --csv python tools/probe_rowproj.py child 4096 4096 > $OUT/ncu_rp_d$d.csv 2>&1
done
LOBRA_RP_SPLITS=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_rowproj -s 3 -c 3 --csv python tools/probe_rowproj.py child 4096 4096 > $OUT/ncu_rp_s1.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rowproj -s 3 -c 1 -o $OUT/rp_full python tools/probe_rowproj.py child 4096 4096 > $OUT/ncu_rp_full.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_tma -s 20 -c 1 -o $OUT/probe_full ./tools/probe_stream.bin > $OUT/ncu_probe_full.log 2>&1

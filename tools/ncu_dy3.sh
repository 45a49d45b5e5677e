# k_dypass on the C3 batch (ranks up to 64: 128-byte operand span) under the probe bits
OUT=gpurun_out
for cfg in "0" "7" "2" "4" "6" "1"; do
  echo "dbg $cfg" >> $OUT/ncu_dy3.txt
  LOBRA_DBG_DY=$cfg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dypass -s 2 -c 2 --csv python tools/probe_rowproj.py childb3 4096 4096 2>&1 | grep k_dypass | awk -F'","' '{print $NF}' | tr -d '"' >> $OUT/ncu_dy3.txt
done

# k_dypass duration vs operand span / stage count / probe bits (ncu, serialised)
OUT=gpurun_out
for cfg in "128 3 0" "128 8 0" "32 3 0" "32 8 0" "32 8 7" "32 8 2" "32 8 4" "64 8 0" "128 3 7"; do
  set -- $cfg
  echo "span $1 stages $2 dbg $3" >> $OUT/ncu_dy2.txt
  LOBRA_DY_SPAN=$1 LOBRA_DY_STAGES=$2 LOBRA_DBG_DY=$3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dypass -s 2 -c 2 --csv python tools/probe_rowproj.py childb 4096 4096 2>&1 | grep k_dypass | awk -F'","' '{print $NF}' | tr -d '"' >> $OUT/ncu_dy2.txt
done

# k_dypass duration under the LOBRA_DBG_DY probe bits (ncu, serialised)
OUT=gpurun_out
for d in 0 1 2 4 6 7; do
  for shp in "4096 4096" "4096 11008"; do
    echo "dbg $d shape $shp" >> $OUT/ncu_dy.txt
    LOBRA_DBG_DY=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dypass -s 2 -c 2 --csv python tools/probe_rowproj.py childb $shp 2>&1 | grep k_dypass | awk -F'","' '{print $NF}' | tr -d '"' >> $OUT/ncu_dy.txt
  done
done

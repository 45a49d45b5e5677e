# k_shrink vs k_rowproj kernel durations (ncu, serialised) on the C2 q and down shapes
OUT=gpurun_out
for sh in 0 1; do
  for shp in "4096 4096" "11008 4096"; do
    LOBRA_SHRINK=$sh timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_rowproj|k_shrink" -s 3 -c 3 --csv python tools/probe_rowproj.py child $shp 2>&1 | grep -E "k_rowproj|k_shrink" | awk -F'","' '{print $5, $(NF-2), $NF}' | tr -d '"' >> $OUT/ncu_shrink.txt
  done
done

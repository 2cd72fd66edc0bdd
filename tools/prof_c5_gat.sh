OUT=gpurun_out/prof; mkdir -p $OUT
B="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"k_gat_" -s 20 -c 8 -o $OUT/gat -f $B > $OUT/gat.log 2>&1
ncu -i $OUT/gat.ncu-rep --page details --csv > $OUT/gat_details.csv 2>/dev/null
ncu -i $OUT/gat.ncu-rep --page source --csv --print-source sass > $OUT/gat_sass.csv 2>/dev/null
rm -f $OUT/gat.ncu-rep

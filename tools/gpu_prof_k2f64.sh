# ncu --set full of the fp64 K2 (config 3's fp64 side line): summary + SASS mix
O=gpurun_out/k2f64
mkdir -p $O
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k2_tma_kernel<double" -s 3 -c 1 -o $O/prof \
  python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/prof.ncu-rep > $O/summary.txt
ncu -i $O/prof.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
python tools/sass_mix_csv.py $O/src.csv > $O/sassmix.txt 2>/dev/null
ncu -i $O/prof.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
rm -f $O/prof.ncu-rep $O/src.csv

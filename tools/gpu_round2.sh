ncu --set full --clock-control none --import-source on -k regex:mc_chunk -s 3 -c 1 -o gpurun_out/prof_mc python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_mc.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_mc.ncu-rep > gpurun_out/sum_mc.txt
ncu -i gpurun_out/prof_mc.ncu-rep --page source --csv --print-source sass > gpurun_out/src_mc.csv 2>/dev/null
rm -f gpurun_out/prof_mc.ncu-rep

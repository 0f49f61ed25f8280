ncu --set full --clock-control none --import-source on -k regex:gradmarch -s 3 -c 1 -o gpurun_out/prof_gm python bench.py --workload redsea --steps 3 --no-e2e --no-cpu > gpurun_out/ncu_gm.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_gm.ncu-rep > gpurun_out/sum_gm.txt
ncu -i gpurun_out/prof_gm.ncu-rep --page source --csv --print-source sass > gpurun_out/src_gm.csv 2>/dev/null
rm -f gpurun_out/prof_gm.ncu-rep

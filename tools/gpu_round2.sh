timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mc or MC or config2 or smoke" 2>&1 | tail -2 > gpurun_out/mctest.txt
bash tools/gpu_prof.sh mc mc_chunk --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/prof_mc.ncu-rep --page source --csv --print-source sass > gpurun_out/src_mc.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_mc.ncu-rep > gpurun_out/sum_mc.txt
rm gpurun_out/prof_mc.ncu-rep

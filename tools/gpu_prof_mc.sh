# ncu --set full of the MC chunk kernel (config 2) and the config-1 fused kernel
bash tools/gpu_prof.sh mc mc_chunk --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu
bash tools/gpu_prof.sh c1 k3_tma --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu
for n in mc c1; do ncu -i gpurun_out/prof_$n.ncu-rep --page source --print-source sass --csv > gpurun_out/src_$n.csv 2>/dev/null; done
ls -la gpurun_out

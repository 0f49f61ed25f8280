# usage: bash tools/gpu_prof.sh <name> <kernel-regex> <bench args...>
name=$1; shift; kre=$1; shift
python bench.py "$@" > gpurun_out/plain_$name.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 1 -o gpurun_out/prof_$name python bench.py "$@" > gpurun_out/ncu_$name.log 2>&1
tail -2 gpurun_out/ncu_$name.log

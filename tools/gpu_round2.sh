timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for c in 4 1 3; do timeout 300 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/b_c$c.json 2> gpurun_out/b_c$c.err || tail -5 gpurun_out/b_c$c.err; python -c "import json;d=json.load(open('gpurun_out/b_c$c.json'));print($c,d['ms_per_step'],d['roofline']['frac'],d['clocks'])"; done
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k3_rowmarch -s 3 -c 1 python bench.py --config 1 --no-cpu --no-e2e --steps 3 2>&1 | grep -E "dram__bytes_read|gpu__time_duration"

timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/alltest.txt 2>&1
timeout 300 python bench.py --workload redsea --steps 20 --no-cpu > gpurun_out/rs.json 2>gpurun_out/rs.err || tail -3 gpurun_out/rs.err; python -c "import json;d=json.load(open('gpurun_out/rs.json'));r=d['roofline'];print('rs',d['ms_per_step'],r['frac'],r.get('unfused_chain_ms'))"

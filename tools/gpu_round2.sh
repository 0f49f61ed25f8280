timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mc or MC or config2 or smoke or philox" > gpurun_out/mctest.txt 2>&1
timeout 300 python bench.py --config 2 --no-cpu --no-e2e --steps 20 > gpurun_out/mc.json 2>gpurun_out/mc.err || tail -3 gpurun_out/mc.err
python -c "import json;d=json.load(open('gpurun_out/mc.json'));print('mc',d['ms_per_step'],d['roofline']['frac'])"
tail -1 gpurun_out/mctest.txt

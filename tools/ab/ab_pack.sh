python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3.json 2>gpurun_out/c3.err; python tools/summ.py gpurun_out/c3.json
python -c "import json; d=json.load(open('gpurun_out/c3.json')); print(d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['roofline']['decode_step_ms'])"
python bench.py --no-cpu-baseline > gpurun_out/c2.json 2>&1; python tools/summ.py gpurun_out/c2.json

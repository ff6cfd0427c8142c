python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2 3; do python bench.py --no-cpu-baseline > gpurun_out/ab_f$i.log 2>&1; python tools/summ.py gpurun_out/ab_f$i.log; done

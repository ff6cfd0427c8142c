run() { tag=$1; envs=$2; shift 2; env $envs python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$tag.log 2>&1; python tools/summ.py gpurun_out/ab_$tag.log; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
run base X=1
run none ARBOR_EVICT_EXP=3
run nomove ARBOR_EVICT_EXP=1
run c4 X=1 --config c4

run() { tag=$1; envs=$2; shift 2; env $envs python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$tag.log 2>&1; python tools/summ.py gpurun_out/ab_$tag.log; }
run one X=1
run split ARBOR_SPLIT_NQ=1
run one2 X=1
run split2 ARBOR_SPLIT_NQ=1

run() { tag=$1; envs=$2; shift 2; env $envs python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$tag.log 2>&1; python tools/summ.py gpurun_out/ab_$tag.log; }
run base X=1
run rflush ARBOR_BENCH_READ_FLUSH=1
run base2 X=1
run rflush2 ARBOR_BENCH_READ_FLUSH=1

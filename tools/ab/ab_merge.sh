run() { tag=$1; envs=$2; shift 2; env $envs python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$tag.log 2>&1; python tools/summ.py gpurun_out/ab_$tag.log; }
run new ARBOR_BENCH_TWO_CALL=1
run old "ARBOR_BENCH_TWO_CALL=1 ARBOR_OLD_MERGE=1"
run new2 ARBOR_BENCH_TWO_CALL=1
run old2 "ARBOR_BENCH_TWO_CALL=1 ARBOR_OLD_MERGE=1"

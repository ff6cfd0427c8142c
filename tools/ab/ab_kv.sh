run() { tag=$1; envs=$2; shift 2; env $envs python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$tag.log 2>&1; python tools/summ.py gpurun_out/ab_$tag.log; }
ARBOR_TC_AHEAD=2 python -m pytest tests/test_gpu_attn_tc.py tests/test_gpu_decode_step.py -x -q 2>&1 | tail -1
run base X=1
run ahead2 ARBOR_TC_AHEAD=2
run base2 X=1
run ahead2b ARBOR_TC_AHEAD=2
for v in 1 2; do ARBOR_TC_AHEAD=$v python profiles/decode_step_prof.py c2 20; ARBOR_TC_AHEAD=$v python profiles/decode_step_prof.py c3 20; done

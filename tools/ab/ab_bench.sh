run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --steps 40 > gpurun_out/ab_$tag.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1]); print('$tag', round(d['ms_per_step']*1e3,1), [round(x*1e3,1) for x in d['step_ms_p10_p50_p90']], round(d['stage_ms_median']['attn']*1e3,1), round(d['stage_ms_median']['score_accum']*1e3,1), round(d['stage_ms_median']['attn_merge']*1e3,1), round(d['stage_ms_median']['allocate']*1e3,1), round(d['stage_ms_median']['select_compact']*1e3,1))"; }
run fused X=1
run two ARBOR_BENCH_TWO_CALL=1
run fused_postnopdl ARBOR_POST_NOPDL=1
run fused_nopdl ARBOR_NO_PDL=1
run two_nopdl ARBOR_NO_PDL=1 ARBOR_BENCH_TWO_CALL=1

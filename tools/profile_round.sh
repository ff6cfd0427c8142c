# Full measurement pass for profiles/ (round 2): ncu launch list of the C2 step, ncu --set full
# of the C2 step and of one C3 (DPTS loop state) decode step — their DRAM traffic regenerates
# profiles/ncu_traffic.json (tools/ncu_traffic.py) BEFORE the benches, so every bench line of
# the round carries this build's `traffic` — then benches C2 (with cpu_baseline), C3, C4, C5,
# the reference arm, the evict / decode_post timelines and the attention traces.
set -x
V=${V:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_step/" --csv \
    --log-file gpurun_out/${V}_launches.csv python bench.py --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "bench_step/" -c 4 \
    -o gpurun_out/${V}_full python bench.py --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_tc_kernel|decode_post" \
    --launch-skip 187 --launch-count 2 -o gpurun_out/${V}_c3dpts python profiles/decode_step_prof.py c3dpts 3 \
    > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_full.log gpurun_out/ncu_c3.log
python tools/ncu_traffic.py gpurun_out/${V}_full.ncu-rep gpurun_out/${V}_c3dpts.ncu-rep ${V} > /dev/null \
    && cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python bench.py > gpurun_out/${V}_bench.json 2> gpurun_out/bench_err.log; tail -c 300 gpurun_out/bench_err.log
python bench.py --config c3 --no-cpu-baseline > gpurun_out/${V}_bench_c3.json 2>>gpurun_out/bench_err.log
python bench.py --config c4 --no-cpu-baseline > gpurun_out/${V}_bench_c4.json 2>>gpurun_out/bench_err.log
python bench.py --config c5 --no-cpu-baseline > gpurun_out/${V}_bench_c5.json 2>>gpurun_out/bench_err.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${V}_bench_reference.json 2>>gpurun_out/bench_err.log
ARBOR_NVCC_FLAGS="-DARBOR_EVICT_TRACE_BUILD" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
python profiles/evict_trace.py c2 > gpurun_out/${V}_evict_trace_c2.json 2>&1
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
# the timelines are compiled only into diagnostic builds
ARBOR_NVCC_FLAGS="-DARBOR_TC_TRACE_BUILD -DARBOR_POST_TRACE_BUILD" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
POST_TRACE=1 python profiles/decode_step_prof.py c3dpts 10 > gpurun_out/${V}_post_trace_c3dpts.json 2>&1
POST_TRACE=1 python profiles/decode_step_prof.py c2 10 > gpurun_out/${V}_post_trace_c2.json 2>&1
python profiles/attn_trace.py c3dpts > gpurun_out/${V}_attn_trace_c3dpts.json 2>&1
python profiles/attn_trace.py c2 > gpurun_out/${V}_attn_trace_c2.json 2>&1
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
for f in gpurun_out/${V}_bench*.json; do python tools/summ.py $f; done

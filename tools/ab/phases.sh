# select-phase timeline of select_compact (debug build -DARBOR_EVICT_PHASES), then the normal build
ARBOR_NVCC_FLAGS="-DARBOR_EVICT_PHASES -DARBOR_EVICT_TRACE_BUILD" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
for cfg in "$@"; do python profiles/evict_trace.py $cfg > gpurun_out/phases_$cfg.json 2>&1; done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

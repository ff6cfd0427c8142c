# allocate phase timeline (debug build -DARBOR_ALLOC_TRACE), then the normal build
ARBOR_NVCC_FLAGS="-DARBOR_ALLOC_TRACE" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
for cfg in "$@"; do python profiles/alloc_trace.py $cfg > gpurun_out/alloc_$cfg.json 2>&1; cat gpurun_out/alloc_$cfg.json | tail -1; done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

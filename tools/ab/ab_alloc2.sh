python -m pytest tests/test_gpu_parity.py tests/test_gpu_controller.py tests/test_gpu_variants.py tests/test_gpu_shards.py tests/test_gpu_decode_step.py -x -q 2>&1 | tail -1
ARBOR_NVCC_FLAGS="-DARBOR_ALLOC_TRACE" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
python profiles/alloc_trace.py
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
for i in 1 2; do python bench.py --no-cpu-baseline > gpurun_out/b$i.log 2>&1; python tools/summ.py gpurun_out/b$i.log; done
python bench.py --no-cpu-baseline --config c5 > gpurun_out/b5.log 2>&1; python tools/summ.py gpurun_out/b5.log

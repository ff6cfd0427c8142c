for t in 512 1024 512 1024; do
  ARBOR_NVCC_FLAGS="-DARBOR_ALLOC_THREADS=$t -DARBOR_ALLOC_TRACE" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  echo "threads=$t"; python profiles/alloc_trace.py
  ARBOR_NVCC_FLAGS="-DARBOR_ALLOC_THREADS=$t" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  python bench.py --no-cpu-baseline > gpurun_out/ab_t$t.log 2>&1; python tools/summ.py gpurun_out/ab_t$t.log
done
ARBOR_NVCC_FLAGS="-DARBOR_ALLOC_THREADS=1024" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_controller.py tests/test_gpu_variants.py -x -q 2>&1 | tail -1

for js in 2 4 8 2 4; do
  ARBOR_NVCC_FLAGS=-DARBOR_JOB_SLOTS=$js python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  python bench.py --no-cpu-baseline > gpurun_out/ab_js$js.log 2>&1; echo "slots=$js"; python tools/summ.py gpurun_out/ab_js$js.log
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_step.py -x -q 2>&1 | tail -1
python bench.py --no-cpu-baseline --config c4 > gpurun_out/ab_c4.log 2>&1; python tools/summ.py gpurun_out/ab_c4.log

for u in 4 6 8 4 6; do
  ARBOR_NVCC_FLAGS="-DARBOR_KUW=$u" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  python bench.py --no-cpu-baseline > gpurun_out/ab_u$u.log 2>&1; echo "kUw=$u"; python tools/summ.py gpurun_out/ab_u$u.log
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

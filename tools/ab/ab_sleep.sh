# A/B: select_compact with sleeping mbarrier waits (ARBOR_EVICT_SLEEP_NS, default) vs spinning (0)
for v in 2000 0 2000 0; do
  ARBOR_NVCC_FLAGS="-DARBOR_EVICT_SLEEP_NS=$v" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  for cfg in c2 c5; do
    python bench.py --no-cpu-baseline --config $cfg > gpurun_out/ab_sleep_${v}_$cfg.log 2>&1
    echo "sleep=$v $cfg"; python tools/summ.py gpurun_out/ab_sleep_${v}_$cfg.log
  done
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

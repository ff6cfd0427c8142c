# Generic A/B of build-flag variants, alternating twice on one box:
#   CFGS="c2 c5" bash tools/ab/ab_flags.sh "-DX=1" "-DX=2" ...
CFGS=${CFGS:-"c2 c5"}
for rep in 1 2; do
  i=0
  for fl in "$@"; do
    i=$((i+1))
    ARBOR_NVCC_FLAGS="$fl" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
    for cfg in $CFGS; do
      python bench.py --no-cpu-baseline --config $cfg > gpurun_out/ab_v${i}_$cfg.log 2>&1
      echo "[$fl] $cfg $(python tools/summ.py gpurun_out/ab_v${i}_$cfg.log | cut -d' ' -f2-12,16-)"
    done
  done
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

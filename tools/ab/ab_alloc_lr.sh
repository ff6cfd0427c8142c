# allocate largest remainder: register/shuffle bitonic vs warp-per-node ranking vs smem bitonic
for v in "" "-DARBOR_ALLOC_LR_WARP_MAX=0" "-DARBOR_ALLOC_LR_SHFL=0"; do
  ARBOR_NVCC_FLAGS="-DARBOR_ALLOC_TRACE $v" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  for c in c2 c3dpts c5; do echo "[$v] $(python profiles/alloc_trace.py $c 2>&1 | tail -1)"; done
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

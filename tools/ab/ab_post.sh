# decode_post build variants on the C3 DPTS and C2 decode steps: bash tools/ab/ab_post.sh "-DX" ...
for rep in 1 2; do
for v in "" "$@"; do
  ARBOR_NVCC_FLAGS="$v" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  echo "[$v] $(python profiles/decode_step_prof.py c3dpts 20 2>&1 | tail -1 | cut -c1-150)"
  echo "[$v] $(python profiles/decode_step_prof.py c2 30 2>&1 | tail -1 | cut -c1-150)"
done
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

# decode_post residency A/B: min blocks per SM (registers) x parts, C3 DPTS decode step + C2 bench
for rep in 1 2; do
for m in 2 3 4; do
  ARBOR_NVCC_FLAGS="-DARBOR_POST_MINB=$m" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  for parts in 0 2; do
    echo "minb=$m parts=$parts $(ARBOR_POST_PARTS=$parts python profiles/decode_step_prof.py c3dpts 20 2>&1 | tail -1 | cut -c1-160)"
  done
  echo "minb=$m c2 $(python profiles/decode_step_prof.py c2 20 2>&1 | tail -1 | cut -c1-160)"
done
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

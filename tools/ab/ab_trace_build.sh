# production build (no trace code) vs the diagnostic trace builds of attn_tc / decode_post
for rep in 1 2; do
for v in "" "-DARBOR_TC_TRACE_BUILD -DARBOR_POST_TRACE_BUILD"; do
  ARBOR_NVCC_FLAGS="$v" python -m paper_2605_22106_b200.build --force > /dev/null 2>&1
  echo "[$v] $(python profiles/decode_step_prof.py c3dpts 20 2>&1 | tail -1 | cut -c1-150)"
  echo "[$v] $(python profiles/decode_step_prof.py c2 30 2>&1 | tail -1 | cut -c1-150)"
  python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; echo "[$v] $(python tools/summ.py gpurun_out/b.log | cut -d' ' -f2-9)"
done
done
python -m paper_2605_22106_b200.build --force > /dev/null 2>&1

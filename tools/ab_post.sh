for pp in 1 2 8; do
  echo "PARTS=$pp"; ARBOR_POST_PARTS=$pp python profiles/decode_step_prof.py c2 20; ARBOR_POST_PARTS=$pp python profiles/decode_step_prof.py c3 20
done
echo default; python profiles/decode_step_prof.py c2 20; python profiles/decode_step_prof.py c3 20
python bench.py --no-cpu-baseline > gpurun_out/ab_def.log 2>&1; python tools/summ.py gpurun_out/ab_def.log
ARBOR_BENCH_TWO_CALL=1 python bench.py --no-cpu-baseline > gpurun_out/ab_two.log 2>&1; python tools/summ.py gpurun_out/ab_two.log

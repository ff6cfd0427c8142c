python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for e in 0 2; do echo "EXP=$e"; ARBOR_POST_EXP=$e python profiles/decode_step_prof.py c3 20; ARBOR_POST_EXP=$e python profiles/decode_step_prof.py c2 20; done
python bench.py --no-cpu-baseline > gpurun_out/ab_c2.log 2>&1; python tools/summ.py gpurun_out/ab_c2.log

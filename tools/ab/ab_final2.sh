timeout 240 python profiles/stress_decode.py c3 2000 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 0 8; do echo "QSLOT=$v"; ARBOR_QSLOT=$v timeout 120 python profiles/decode_step_prof.py c3 20; done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c2q.log 2>&1; python tools/summ.py gpurun_out/c2q.log
for v in 0 8; do ARBOR_QSLOT=$v timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3q$v.log 2>&1; echo "c3 QSLOT=$v"; python tools/summ.py gpurun_out/c3q$v.log; done

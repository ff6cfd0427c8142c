timeout 300 python -m pytest tests/test_gpu_attn_tc.py tests/test_gpu_decode_step.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 0 8; do echo "QSLOT=$v"; ARBOR_QSLOT=$v python profiles/decode_step_prof.py c3 20; ARBOR_QSLOT=$v python profiles/decode_step_prof.py c2 20; done
ARBOR_QSLOT=0 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3d.log 2>&1; python tools/summ.py gpurun_out/c3d.log
ARBOR_QSLOT=8 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3e.log 2>&1; python tools/summ.py gpurun_out/c3e.log
python bench.py --config c4 --no-cpu-baseline > gpurun_out/c4d.log 2>&1; python tools/summ.py gpurun_out/c4d.log
python bench.py --no-cpu-baseline > gpurun_out/c2d.log 2>&1; python tools/summ.py gpurun_out/c2d.log

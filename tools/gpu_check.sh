# GPU parity suite + smoke + benches: bash tools/gpu_check.sh [notest] cfg...
if [ "$1" != "notest" ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
else
  shift
fi
for cfg in "$@"; do
  extra=""
  [ "$cfg" = "c3" ] && extra="--steps 10 --warmup 3"
  python bench.py --no-cpu-baseline --config $cfg $extra > gpurun_out/bench_$cfg.log 2>&1
  python tools/summ.py gpurun_out/bench_$cfg.log
done

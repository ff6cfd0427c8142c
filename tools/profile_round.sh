# Full measurement pass for profiles/ (round 1, v11): benches C2 (with cpu_baseline), C3, C4, C5,
# the reference arm, an ncu launch list of the C2 step and one ncu --set full capture.
set -x
V=${V:-v15}
python bench.py > gpurun_out/r01_bench_$V.json 2> gpurun_out/bench_err.log; tail -c 300 gpurun_out/bench_err.log
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3_$V.json 2>>gpurun_out/bench_err.log
python bench.py --config c4 --no-cpu-baseline > gpurun_out/r01_bench_c4_$V.json 2>>gpurun_out/bench_err.log
python bench.py --config c5 --no-cpu-baseline > gpurun_out/r01_bench_c5_$V.json 2>>gpurun_out/bench_err.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01_bench_reference_$V.json 2>>gpurun_out/bench_err.log
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_step/" --csv \
    --log-file gpurun_out/launches_$V.csv python bench.py --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "bench_step/" -c 4 \
    -o gpurun_out/full_$V python bench.py --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
for f in gpurun_out/r01_bench_*$V.json; do python tools/summ.py $f; done

# Bench + ncu launch list + one ncu --set full capture of the fused kernel, the
# inputs of tools/profile_summary.py.   usage: bash tools/gpu_profile_round.sh
set -x
python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_line.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-policy > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_observe -s 20 -c 1 \
    -o gpurun_out/prof_bench -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-policy \
    > gpurun_out/ncu_full.log 2>&1; echo full=$?

# Bench (default C1 line + the reference arm + short-K line) + ncu launch list +
# one ncu --set full capture of the fused kernel: the inputs of
# tools/profile_summary.py.   usage: bash tools/gpu_profile_round.sh
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_line.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
python bench.py --steps 20 --warmup 3 --no-policy --no-cpu-baseline > gpurun_out/bench_s20.json 2> gpurun_out/bench_s20.err; echo s20=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-policy > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_observe -s 4 -c 1 \
    -o gpurun_out/prof_bench -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-policy \
    > gpurun_out/ncu_full.log 2>&1; echo full=$?

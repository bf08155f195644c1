python tools/bench_step.py 64 50 > gpurun_out/bench_step.csv 2> gpurun_out/bench_step.err; echo bs=$?
timeout 900 python bench.py --config C3 --no-policy --no-cpu-baseline --no-e2e > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo c3=$?

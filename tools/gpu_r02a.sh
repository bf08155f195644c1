# round-2 check: tests, bench default, bench --steps 20, strong C3/C4 shards
set -x
free -g; nproc
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench=$?
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-policy > gpurun_out/bench_c1_s20.json 2> gpurun_out/bench_c1_s20.err; echo bench20=$?
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_s20.json 2> gpurun_out/bench_ref_s20.err; echo ref20=$?
timeout 900 python bench.py --config C3 --no-policy --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 1200 python bench.py --config C4 --scenarios 32768 --no-policy --no-cpu-baseline > gpurun_out/bench_c4_32k.json 2> gpurun_out/bench_c4_32k.err; echo c4=$?
free -g

for c in C2 C3 C4s; do
  timeout 1500 python bench.py --config $c --no-policy > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
done
timeout 2400 python bench.py --config C4 --no-policy --no-e2e > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo C4=$?

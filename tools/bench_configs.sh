# One bench line per single-GPU config (C2 dense, and the one-GPU shards of C3 / C4).
for c in C2 C3 C4; do
  timeout 1200 python bench.py --config $c --no-policy > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
done

# usage: bash tools/variant_bench_cfgs.sh "C1 C2 C4" variant...
cfgs=$1; shift
for c in $cfgs; do for v in base "$@"; do
  if [ $v = base ]; then L=paper_2312_15122_b200/libzsim_gpu.so; else L=paper_2312_15122_b200/_build/$v/libzsim_gpu.so; fi
  ZSIM_GPU_LIB=$L timeout 900 python bench.py --config $c --no-policy --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c $v\", d[\"value\"], d[\"ms_per_step\"])"
done; done

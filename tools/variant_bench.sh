# Run bench.py (device leg only) for the base library and each variant.
# usage: bash tools/variant_bench.sh [config] name1 name2 ...
cfg=${1:-C1}; shift
out=gpurun_out/variants_$cfg.txt; : > $out
for rep in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then lib=paper_2312_15122_b200/libzsim_gpu.so; else lib=paper_2312_15122_b200/_build/$v/libzsim_gpu.so; fi
  ZSIM_GPU_LIB=$lib timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1000,2), 'us/step', 'kernel', round(d['roofline']['kernel_ms']*1000,2), 'frac', round(d['roofline']['frac'],4))" >> $out
done
done
cat $out

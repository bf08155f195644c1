for rep in 1 2; do for v in base hc4; do
  if [ $v = base ]; then lib=paper_2312_15122_b200/libzsim_gpu.so; else lib=paper_2312_15122_b200/_build/$v/libzsim_gpu.so; fi
  ZSIM_GPU_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-policy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4e' % d['e2e']['value'])" >> gpurun_out/e2e.txt
done; done

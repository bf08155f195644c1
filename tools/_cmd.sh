for rep in 1 2; do for v in base gs; do
  if [ $v = base ]; then lib=paper_2312_15122_b200/libzsim_gpu.so; else lib=paper_2312_15122_b200/_build/$v/libzsim_gpu.so; fi
  echo $v $(ZSIM_GPU_LIB=$lib timeout 600 python tools/policy_bench.py 4096 20 fp32 2>&1 | tail -1) >> gpurun_out/pol_var.txt
done; done
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/gs/libzsim_gpu.so timeout 900 python -m pytest tests/test_policy.py tests/test_policy_reference.py -q -x > gpurun_out/pol_test.log 2>&1; echo rc=$? >> gpurun_out/pol_test.log

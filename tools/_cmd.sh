ZSIM_GPU_LIB=paper_2312_15122_b200/_build/pj2bchk/libzsim_gpu.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shapes.py -x -q > gpurun_out/var_chk.log 2>&1; echo rc=$? >> gpurun_out/var_chk.log
bash tools/variant_bench.sh C1 pj2b > /dev/null 2>&1
bash tools/variant_bench.sh C4s pj2b > /dev/null 2>&1

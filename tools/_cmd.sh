ZSIM_GPU_LIB=paper_2312_15122_b200/_build/rcpc/libzsim_gpu.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shapes.py tests/test_gpu_bench_shapes.py -x -q > gpurun_out/pytest_rcp.log 2>&1; echo pytest=$? >> gpurun_out/pytest_rcp.log
bash tools/variant_bench.sh C1 rcp > /dev/null 2>&1
bash tools/variant_bench.sh C4s rcp > /dev/null 2>&1

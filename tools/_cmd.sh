timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shapes.py tests/test_gpu_bench_shapes.py -x -q > gpurun_out/pytest_v1.log 2>&1; echo pytest=$? >> gpurun_out/pytest_v1.log
bash tools/variant_bench.sh C1 r01 > /dev/null 2>&1

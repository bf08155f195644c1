timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_bench_shapes.py tests/test_controlled.py -x -q > gpurun_out/pytest_fdiv.log 2>&1; echo pytest=$? >> gpurun_out/pytest_fdiv.log
bash tools/variant_bench.sh C2 kth > /dev/null 2>&1
bash tools/variant_bench.sh C4s kth > /dev/null 2>&1
bash tools/variant_bench.sh C1 kth > /dev/null 2>&1

timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_bench_shapes.py tests/test_controlled.py tests/test_gpu_comm.py -x -q > gpurun_out/pytest_sat.log 2>&1; echo pytest=$? >> gpurun_out/pytest_sat.log
bash tools/variant_bench.sh C2 sat0 > /dev/null 2>&1
bash tools/variant_bench.sh C4s sat0 > /dev/null 2>&1

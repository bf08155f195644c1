timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v4.log 2>&1; echo pytest=$? >> gpurun_out/pytest_v4.log
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/checked/libzsim_gpu.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_checked.log 2>&1; echo pytest_checked=$? >> gpurun_out/pytest_checked.log
bash tools/variant_bench.sh C2 prewin > /dev/null 2>&1

ZSIM_GPU_LIB=paper_2312_15122_b200/_build/checked/libzsim_gpu.so timeout 1500 python -m pytest tests -m gpu -q -k "not multiprocess and not multi_gpu_driver and not dropin" > gpurun_out/pytest_full_checked.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full_checked.log
timeout 900 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err

ZSIM_GPU_LIB=paper_2312_15122_b200/_build/checked/libzsim_gpu.so timeout 1500 python -m pytest tests -m gpu -q -k "not multiprocess and not multi_gpu_driver and not dropin" > gpurun_out/pytest_full_checked.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full_checked.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full.log
for c in C2 C3 C4 C4s; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done

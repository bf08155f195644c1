ZSIM_GPU_LIB=paper_2312_15122_b200/_build/checked/libzsim_gpu.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shapes.py tests/test_gpu_bench_shapes.py tests/test_gpu_rollout.py tests/test_gpu_stream.py -x -q > gpurun_out/var_chk.log 2>&1; echo rc=$? >> gpurun_out/var_chk.log
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --no-cpu-baseline --no-policy > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err

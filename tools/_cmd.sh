# final round-2 C1 profile after the <= 32-agent kernel instance
bash tools/gpu_profile_round.sh > gpurun_out/profile_round.log 2>&1
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/pathstats/libzsim_gpu_pathstats.so timeout 600 python tools/episode_profile.py 4096 --pathstats > gpurun_out/phases_c1.json 2> gpurun_out/phases_c1.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full.log
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/checked/libzsim_gpu.so timeout 1500 python -m pytest tests -m gpu -q -k "not multiprocess and not multi_gpu_driver and not dropin" > gpurun_out/pytest_full_checked.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full_checked.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log

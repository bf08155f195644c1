# final round-2 validation + profile
bash tools/gpu_profile_round.sh > gpurun_out/profile_round.log 2>&1
for c in C2 C3 C4 C4s; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_observe -s 2 -c 2 -o gpurun_out/prof_c4s -f python bench.py --config C4s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-policy > gpurun_out/ncu_c4s.log 2>&1; echo c4s=$? >> gpurun_out/ncu_c4s.log
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/pathstats/libzsim_gpu_pathstats.so timeout 600 python tools/episode_profile.py 4096 --pathstats > gpurun_out/phases_c1.json 2> gpurun_out/phases_c1.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full.log
ZSIM_GPU_LIB=paper_2312_15122_b200/_build/checked/libzsim_gpu.so timeout 1500 python -m pytest tests -m gpu -q -k "not multiprocess and not multi_gpu_driver and not dropin" > gpurun_out/pytest_full_checked.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full_checked.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log

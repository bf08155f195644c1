timeout 300 python -m pytest tests/test_policy.py -x -q -s 2>&1 | grep -E "error|passed|failed"
ncu --set full --import-source on --clock-control none -k regex:k_policy_tc -s 2 -c 1 -o gpurun_out/policy_tc -f python tools/policy_bench.py 4096 3 > gpurun_out/policy_ncu.log 2>&1; echo ncu=$?

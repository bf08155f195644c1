timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_observe -s 4 -c 1 \
    -o gpurun_out/prof_bench -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-policy \
    > gpurun_out/ncu_full.log 2>&1; echo full=$?
bash tools/variant_bench.sh C1 pf ilibm pfil > /dev/null 2>&1
bash tools/variant_bench.sh C4s pf ilibm pfil > /dev/null 2>&1

bash tools/variant_bench.sh C1 cap192 cap160 cap128 > /dev/null 2>&1
bash tools/variant_bench.sh C4s cap192 cap160 > /dev/null 2>&1

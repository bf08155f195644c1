bash tools/variant_bench.sh C1 blf1 blf4 > /dev/null 2>&1

bash tools/variant_bench.sh C1 l4 > /dev/null 2>&1

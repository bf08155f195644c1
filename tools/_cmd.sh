bash tools/variant_bench.sh C1 peel > /dev/null 2>&1

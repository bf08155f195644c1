bash tools/variant_bench.sh C1 tinl > /dev/null 2>&1
bash tools/variant_bench.sh C4s tinl > /dev/null 2>&1

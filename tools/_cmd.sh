bash tools/variant_bench.sh C1 bl2 bl4 > /dev/null 2>&1
bash tools/variant_bench.sh C4s bl2 bl4 > /dev/null 2>&1
bash tools/variant_bench.sh C2 bl2 bl4 > /dev/null 2>&1

bash tools/variant_bench.sh C4s blm4 blm8 > /dev/null 2>&1
bash tools/variant_bench.sh C2 blm4 blm8 > /dev/null 2>&1

bash tools/variant_bench.sh C4s kum6 kum12 > /dev/null 2>&1
bash tools/variant_bench.sh C2 kum6 kum12 > /dev/null 2>&1

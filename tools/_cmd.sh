bash tools/variant_bench.sh C2 s32 s40 s48 > /dev/null 2>&1

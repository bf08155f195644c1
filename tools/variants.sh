# Build experiment variants of libzsim_gpu.so (-D flags) under _build/<name>/.
# usage: bash tools/variants.sh name:FLAG1,FLAG2 name2:FLAG ...
set -e
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  args=""
  IFS=',' read -ra fl <<< "$flags"
  for f in "${fl[@]}"; do [ -n "$f" ] && args="$args -D$f"; done
  python paper_2312_15122_b200/build.py --variant=$name $args > /dev/null
  echo "built $name ($flags)"
done

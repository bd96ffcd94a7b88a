# bench A/B over environment settings: args = tag then "NAME=VAL ..." strings (use "-" for none)
tag=$1; shift
mkdir -p gpurun_out/$tag
i=0
for e in "$@"; do
  i=$((i+1))
  if [ "$e" = "-" ]; then e=""; fi
  env $e timeout 600 python bench.py --no-cpu-baseline --no-like --no-solve --no-batch --breakdown > gpurun_out/$tag/v$i.json 2>gpurun_out/$tag/v$i.err
  echo "v$i: $e" >> gpurun_out/$tag/index.txt
done

#!/bin/bash
# usage: scripts/ab_lib.sh <tag> <lib>...  -- bench each in-tree library variant (GMT_LIB)
out=gpurun_out/$1; mkdir -p $out; shift
for lib in "$@"; do
  b=$(basename $lib .so)
  GMT_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --breakdown --no-cpu-baseline --no-solve > $out/bench_$b.json 2> $out/bench_$b.err; echo "$b rc=$?"
done

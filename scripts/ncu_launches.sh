#!/bin/bash
# usage: scripts/ncu_launches.sh <tag> [bench args...]
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline $@"
$C > $out/plain.json 2> $out/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv $C > $out/ncu.log 2>&1
echo "launches rc=$?"

#!/bin/bash
# usage: scripts/ncu_one.sh <tag> <kernel-regex> <skip> [bench args]
tag=$1; kre=$2; skip=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline $@"
tmp=/tmp/ncu_$tag; mkdir -p $tmp
$C > $out/plain.json 2> $out/plain.err && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -o $tmp/prof $C > $out/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $tmp/prof.ncu-rep --page raw --csv > $out/prof.raw.csv 2>/dev/null
ncu -i $tmp/prof.ncu-rep --page source --csv --print-source cuda > $out/prof.cuda.csv 2>/dev/null
ncu -i $tmp/prof.ncu-rep --page details --csv > $out/prof.details.csv 2>/dev/null
du -sh $out

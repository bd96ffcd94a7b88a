#!/bin/bash
# usage: scripts/ncu_full.sh <tag> <kernel-regex> <skip> <count> [bench args...]
# One `ncu --set full` capture of the selected launches of the bench command,
# run only after the same command exited 0 without ncu.  Exports raw/source/
# details CSVs next to the plain run (reports stay in /tmp: gpurun_out <= 64 MiB).
tag=$1; kre=$2; skip=$3; cnt=$4; shift 4
out=gpurun_out/$tag; mkdir -p $out
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline $@"
tmp=/tmp/ncu_$tag; mkdir -p $tmp
$C > $out/plain.json 2> $out/plain.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $cnt -o $tmp/prof $C > $out/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $tmp/prof.ncu-rep --page raw --csv > $out/prof.raw.csv 2>/dev/null
ncu -i $tmp/prof.ncu-rep --page source --csv --print-source sass > $out/prof.sass.csv 2>/dev/null
ncu -i $tmp/prof.ncu-rep --page details --csv > $out/prof.details.csv 2>/dev/null
du -sh $out

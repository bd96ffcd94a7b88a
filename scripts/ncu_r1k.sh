#!/bin/bash
out=gpurun_out/r1m; mkdir -p $out
C2="python bench.py --res 256 --steps 1 --warmup 1 --no-cpu-baseline"
tmp=/tmp/ncu_r1m; mkdir -p $tmp
$C2 > $out/plain256.json 2> $out/plain256.err && \
ncu --set full --clock-control none --import-source on -k regex:"k_fine_tiled|k_iface" -s 2 -c 2 -o $tmp/prof_tiled $C2 > $out/ncu1.log 2>&1
echo "ncu rc=$?"
ncu -i $tmp/prof_tiled.ncu-rep --page raw --csv > $out/prof_tiled.raw.csv 2>/dev/null
ncu -i $tmp/prof_tiled.ncu-rep --page source --csv --print-source cuda > $out/prof_tiled.cuda.csv 2>$out/src_err.log
ncu -i $tmp/prof_tiled.ncu-rep --page details --csv > $out/prof_tiled.details.csv 2>/dev/null
du -sh $out

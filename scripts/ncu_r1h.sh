#!/bin/bash
out=gpurun_out/r1h; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --breakdown > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
C2="python bench.py --res 256 --steps 1 --warmup 1 --no-cpu-baseline"
tmp=/tmp/ncu_r1h; mkdir -p $tmp
$C2 > $out/plain256.json 2> $out/plain256.err && \
ncu --set full --clock-control none --import-source on -k regex:"k_fine_tiled" -s 1 -c 1 -o $tmp/prof_tiled $C2 > $out/ncu1.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_effective" -c 1 -o $tmp/prof_ch $C2 > $out/ncu2.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_coarse" -s 2 -c 1 -o $tmp/prof_coarse $C2 > $out/ncu3.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_stencil_l1" -c 1 -o $tmp/prof_l1 $C2 > $out/ncu4.log 2>&1
echo "ncu rc=$?"
for f in $tmp/*.ncu-rep; do b=$(basename $f .ncu-rep); ncu -i $f --page raw --csv > $out/$b.raw.csv 2>/dev/null; ncu -i $f --page details --csv > $out/$b.details.csv 2>/dev/null; done
ncu -i $tmp/prof_tiled.ncu-rep --page source --csv > $out/prof_tiled.source.csv 2>/dev/null
du -sh $out

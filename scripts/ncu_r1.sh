#!/bin/bash
out=gpurun_out/r1c; mkdir -p $out
C1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$C1 > $out/plain512.json 2> $out/plain512.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches512.csv $C1 > $out/ncu512.log 2>&1
echo "launches rc=$?"
C2="python bench.py --res 256 --steps 1 --warmup 1 --no-cpu-baseline"
$C2 > $out/plain256.json 2> $out/plain256.err && \
ncu --set full --clock-control none --import-source on -k regex:"k_fine|k_coarse|k_galerkin|k_effective|k_stencil|k_restrict|k_prolong" -c 14 -o $out/prof256 $C2 > $out/ncu256.log 2>&1
echo "full rc=$?"

#!/bin/bash
out=gpurun_out/r1g; mkdir -p $out
C2="python bench.py --res 256 --steps 1 --warmup 1 --no-cpu-baseline"
$C2 > $out/plain256.json 2> $out/plain256.err && \
ncu --set full --clock-control none --import-source on -k regex:"k_fine_tiled|k_stencil_l1|k_elem_l2|k_galerkin_elem|k_effective|k_coarse|k_stencil_from" -c 12 -o $out/prof256 $C2 > $out/ncu256.log 2>&1
echo "full rc=$?"

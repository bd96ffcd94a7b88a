# ncu --set full of the level-1 tiled coarse sweep (first k_coarse_tiled launch of a V-cycle, 512^3 gyroid)
mkdir -p gpurun_out/ct
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/ct/build.log 2>&1
B="--steps 1 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $B > gpurun_out/ct/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_tiled -s 0 -c 1 \
  -o gpurun_out/ct/ct python bench.py $B > gpurun_out/ct/ncu.log 2>&1
echo done

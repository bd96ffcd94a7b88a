# ncu --set full of the level-0 restriction / prolongation and the level-1 interface kernel (512^3 gyroid)
mkdir -p gpurun_out/xfer
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/xfer/build.log 2>&1
B="--steps 1 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $B > gpurun_out/xfer/plain.log 2>&1 || exit 1
for spec in "k_restrict 0 r" "k_prolong_cell 6 p" "k_coarse_iface 0 i"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
    -o gpurun_out/xfer/$3 python bench.py $B > gpurun_out/xfer/ncu_$3.log 2>&1
done
echo done

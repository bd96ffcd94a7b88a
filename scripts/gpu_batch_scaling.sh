# batch V-cycle time vs batch size (scripts/batch_scaling.py)
mkdir -p gpurun_out/bs2
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/bs2/build.log 2>&1
for m in 256; do
  GMT_L0_SPLIT_MIN=$m timeout 900 python scripts/batch_scaling.py > gpurun_out/bs2/scaling_$m.log 2>&1
done

echo done

# halo / interior overlap of the slab level-0 sweeps: slab tests, then V-cycle times with and without
mkdir -p gpurun_out/ovl3
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/ovl3/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/ovl3/pytest.log 2>&1
for cfg in "256 2" "256 4" "512 2" "512 4"; do
  set -- $cfg
  timeout 600 python scripts/slab_overlap_time.py $1 $2 >> gpurun_out/ovl3/times.log 2>&1
done
echo done

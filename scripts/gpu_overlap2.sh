mkdir -p gpurun_out/ovl2
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/ovl2/build.log 2>&1
OVL_SETTINGS=0 timeout 300 python scripts/slab_overlap_time.py 256 2 > gpurun_out/ovl2/a_ovl0.log 2>&1
OVL_SETTINGS=1 GMT_SLAB_MIN_PLANES=8 timeout 300 python scripts/slab_overlap_time.py 256 2 > gpurun_out/ovl2/b_ovl1_min8.log 2>&1
OVL_SETTINGS=1 timeout 300 python scripts/slab_overlap_time.py 128 2 > gpurun_out/ovl2/c_128.log 2>&1
OVL_SETTINGS=1 OVL_CYCLES=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/slab_overlap_time.py 256 2 > gpurun_out/ovl2/d_san.log 2>&1
echo done

# A/B of the level-0 z-chunk (GMT_L0_ZC = 16 / 32 / 48 builds)
mkdir -p gpurun_out/zc2
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/zc2/build.log 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve"
for v in zc48 zc40 zc56 zc48 zc56; do
  if [ $v = def ]; then unset GMT_LIB; else export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_$v.so; fi
  timeout 600 python bench.py $B >> gpurun_out/zc2/$v.json 2>>gpurun_out/zc2/$v.err
  timeout 600 python bench.py $B --res 256 --geometry stochastic >> gpurun_out/zc2/${v}_sto.json 2>>gpurun_out/zc2/$v.err
done
GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_zc56.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/zc2/pytest56.log 2>&1
echo done

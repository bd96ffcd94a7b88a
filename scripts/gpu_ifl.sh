# A/B of lanes per interface node in k_l0 (L0_IFL = 4 default vs 8 and 2): parity subset, then
# stochastic 256^3 / gyroid 512^3 sweeps
mkdir -p gpurun_out/ifl
cd paper_2604_26518_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -shared -Xcompiler -fvisibility=hidden -I ../../include"
nvcc $F -DL0_IFL=8 -o ../libgmt_ifl8.so gmt_api.cu gmt_fem.cpp > /dev/null 2>&1 &
nvcc $F -DL0_IFL=2 -o ../libgmt_ifl2.so gmt_api.cu gmt_fem.cpp > /dev/null 2>&1 &
cd ../..
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/ifl/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "level0 or vcycle or sweep" > gpurun_out/ifl/pytest.log 2>&1
wait
for v in def ifl8 ifl2; do
  if [ $v = def ]; then unset GMT_LIB; else export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_$v.so; fi
  timeout 300 python bench.py --res 256 --geometry stochastic --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/ifl/${v}_sto.json 2>gpurun_out/ifl/${v}_sto.err
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve > gpurun_out/ifl/${v}_gyr.json 2>gpurun_out/ifl/${v}_gyr.err
done
unset GMT_LIB
echo done

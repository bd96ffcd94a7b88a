# A/B of the transfer kernels (working tree vs the last commit's library), gyroid 512^3 and stochastic 256^3
tag=${1:-xf}
mkdir -p gpurun_out/$tag
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/$tag/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_batch.py -m gpu -x -q > gpurun_out/$tag/pytest.log 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve"
for v in new old new old; do
  if [ $v = old ]; then export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_old.so; else unset GMT_LIB; fi
  timeout 300 python bench.py $B >> gpurun_out/$tag/$v.json 2>>gpurun_out/$tag/$v.err
  timeout 300 python bench.py $B --res 256 --geometry stochastic >> gpurun_out/$tag/${v}_sto.json 2>>gpurun_out/$tag/${v}_sto.err
done
echo done

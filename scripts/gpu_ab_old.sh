# A/B of the working tree's libgmt.so against libgmt_old.so (built from the last commit):
# parity subset first, then stochastic 256^3 and gyroid 512^3 sweeps for both
tag=${1:-ab}
mkdir -p gpurun_out/$tag
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/$tag/build.log 2>&1
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/$tag/pytest.log 2>&1
for v in def old def old; do
  if [ $v = def ]; then unset GMT_LIB; else export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_old.so; fi
  timeout 300 python bench.py --res 256 --geometry stochastic --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve >> gpurun_out/$tag/${v}_sto.json 2>>gpurun_out/$tag/${v}_sto.err
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve >> gpurun_out/$tag/${v}_gyr.json 2>>gpurun_out/$tag/${v}_gyr.err
done
unset GMT_LIB
echo done

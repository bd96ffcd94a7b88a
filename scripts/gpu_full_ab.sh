# A/B (working tree vs last commit): all GPU tests, then V-cycle breakdowns for 512^3 elastic and heat, 256^3 stochastic
tag=${1:-fa}
mkdir -p gpurun_out/$tag
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/$tag/build.log 2>&1
timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/$tag/pytest.log 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve"
for v in new old; do
  if [ $v = old ]; then export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_old.so; else unset GMT_LIB; fi
  timeout 600 python bench.py $B >> gpurun_out/$tag/${v}_ela.json 2>>gpurun_out/$tag/$v.err
  timeout 600 python bench.py $B --res 256 --geometry stochastic >> gpurun_out/$tag/${v}_sto.json 2>>gpurun_out/$tag/$v.err
  timeout 600 python bench.py $B --physics thermal >> gpurun_out/$tag/${v}_heat.json 2>>gpurun_out/$tag/$v.err
done
echo done

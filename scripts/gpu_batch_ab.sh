# A/B (working tree vs last commit): GPU tests, V-cycle breakdown, batch screening line
tag=${1:-bt}
mkdir -p gpurun_out/$tag
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/$tag/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/$tag/pytest.log 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-like --breakdown --no-solve"
for v in new old; do
  if [ $v = old ]; then export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_old.so; else unset GMT_LIB; fi
  timeout 600 python bench.py $B >> gpurun_out/$tag/$v.json 2>>gpurun_out/$tag/$v.err
done
echo done

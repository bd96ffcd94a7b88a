# A/B of k_prolong_cell component groups (GMT_PROLONG_G) against the last commit's library
mkdir -p gpurun_out/pg
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/pg/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/pg/pytest.log 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve"
for v in 2 3 6 old; do
  if [ $v = old ]; then export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_old.so; else export GMT_PROLONG_G=$v; fi
  timeout 300 python bench.py $B > gpurun_out/pg/g$v.json 2>gpurun_out/pg/g$v.err
done
echo done

# A/B of k_coarse_iface load-case groups (GMT_IFACE_G) and the last commit's library
mkdir -p gpurun_out/ig
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/ig/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_batch.py -m gpu -x -q > gpurun_out/ig/pytest.log 2>&1
B="--steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve"
for v in 1 2 3 6 old; do
  if [ $v = old ]; then export GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_old.so; else export GMT_IFACE_G=$v; fi
  timeout 300 python bench.py $B > gpurun_out/ig/g$v.json 2>gpurun_out/ig/g$v.err
  timeout 300 python bench.py $B --res 256 --geometry stochastic > gpurun_out/ig/s$v.json 2>gpurun_out/ig/s$v.err
done
echo done

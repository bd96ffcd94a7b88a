# A/B two in-tree builds: bench gyroid + solid for each lib given as args (paths relative to repo)
tag=$1; shift
mkdir -p gpurun_out/$tag
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "level0_vcycle_kernel or vcycle_matches" > gpurun_out/$tag/pytest_k.log 2>&1; echo "k rc=$?"
for lib in "$@"; do
  nm=$(basename $lib .so)
  for g in gyroid solid; do
    GMT_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown --no-solve --geometry $g > gpurun_out/$tag/${nm}_$g.json 2>gpurun_out/$tag/${nm}_$g.err
  done
done
echo done

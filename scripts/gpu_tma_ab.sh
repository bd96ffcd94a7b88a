tag=$1
mkdir -p gpurun_out/$tag
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_refine.py -m gpu -q -x -k "tma or sweep_sampled or auto_switch" > gpurun_out/$tag/pytest.log 2>&1; echo "pytest rc=$?"
for g in gyroid solid; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve --geometry $g > gpurun_out/$tag/tma_$g.json 2>gpurun_out/$tag/tma_$g.err
  GMT_NO_TMA=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve --geometry $g > gpurun_out/$tag/cpa_$g.json 2>gpurun_out/$tag/cpa_$g.err
done
echo done

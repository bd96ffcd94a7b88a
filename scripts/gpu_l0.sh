# level-0 kernel iteration: build, parity of the kernel, bench gyroid/solid, ncu of k_l0
tag=${1:-l0}
mkdir -p gpurun_out/$tag
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/$tag/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "level0_vcycle_kernel or vcycle_matches" > gpurun_out/$tag/pytest_k.log 2>&1; echo "k rc=$?"
for g in gyroid solid; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown --no-solve --geometry $g > gpurun_out/$tag/def_$g.json 2>gpurun_out/$tag/def_$g.err
done
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/$tag/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_l0 -s 4 -c 1 -o gpurun_out/$tag/l0 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/$tag/ncu.log 2>&1
echo done

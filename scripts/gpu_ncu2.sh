tag=$1
mkdir -p gpurun_out/$tag
for g in solid gyroid; do
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve --geometry $g > gpurun_out/$tag/plain_$g.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_l0 -s 4 -c 1 -o gpurun_out/$tag/l0_$g python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve --geometry $g > gpurun_out/$tag/ncu_$g.log 2>&1
done
for g in gyroid solid; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown --no-solve --geometry $g > gpurun_out/$tag/b_$g.json 2>gpurun_out/$tag/b_$g.err
done
echo done

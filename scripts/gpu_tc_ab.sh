tag=$1
mkdir -p gpurun_out/$tag
for k in 0 1; do for g in gyroid solid; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-like --breakdown --no-solve --geometry $g --l0-kernel $k > gpurun_out/$tag/k${k}_$g.json 2>gpurun_out/$tag/k${k}_$g.err
done; done
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-like --no-solve --l0-kernel 1 > gpurun_out/$tag/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_l0_tc -s 4 -c 1 -o gpurun_out/$tag/tc python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-like --no-solve --l0-kernel 1 > gpurun_out/$tag/ncu.log 2>&1
echo done

# bench lines for the other BASELINE workloads (configs[3] 256^3 stochastic, heat 512^3, configs[1] 64^3)
tag=$1
mkdir -p gpurun_out/$tag
timeout 600 python bench.py --res 256 --geometry stochastic --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/$tag/bench_256_stochastic.json 2>gpurun_out/$tag/e1.err
timeout 600 python bench.py --physics thermal --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/$tag/bench_512_thermal.json 2>gpurun_out/$tag/e2.err
timeout 600 python bench.py --res 64 --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/$tag/bench_64_elastic.json 2>gpurun_out/$tag/e3.err
echo done

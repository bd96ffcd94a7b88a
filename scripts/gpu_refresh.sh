# Round-2 evidence refresh: GPU tests, default bench line, heat / stochastic / 64^3 lines,
# ncu --set full of one level-0 sweep (interior TMA launch + boundary-ring launch), launch list
tag=${1:-rf}
mkdir -p gpurun_out/$tag
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/$tag/build.log 2>&1
timeout 1200 python -m pytest tests/ -m gpu -q > gpurun_out/$tag/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/$tag/bench_512_elastic.json 2>gpurun_out/$tag/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/$tag/bench_512_elastic_breakdown.json 2>>gpurun_out/$tag/bench.err
timeout 600 python bench.py --physics thermal --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/$tag/bench_512_thermal.json 2>>gpurun_out/$tag/bench.err
timeout 600 python bench.py --res 256 --geometry stochastic --no-cpu-baseline --no-like --no-batch --breakdown > gpurun_out/$tag/bench_256_stochastic.json 2>>gpurun_out/$tag/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/$tag/bench_reference.json 2>>gpurun_out/$tag/bench.err
B="--steps 1 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $B > gpurun_out/$tag/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l0 -s 8 -c 2 -o gpurun_out/$tag/l0 python bench.py $B > gpurun_out/$tag/ncu_l0.log 2>&1
B2="--steps 2 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $B2 > gpurun_out/$tag/plain2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches.csv python bench.py $B2 > gpurun_out/$tag/ncu_launches.log 2>&1
echo done

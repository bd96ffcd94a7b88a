# ncu launch list of bench.py steps (cold-cache, serialised: compare shares)
tag=$1
mkdir -p gpurun_out/$tag
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $ARGS > gpurun_out/$tag/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches.csv python bench.py $ARGS > gpurun_out/$tag/ncu.log 2>&1
echo done $?

# ncu --set full of the stochastic 256^3 level-0 interior launch (interface-heavy)
mkdir -p gpurun_out/sto2
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/sto2/build.log 2>&1
B="--res 256 --geometry stochastic --steps 1 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $B > gpurun_out/sto2/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l0 -s 8 -c 1 -o gpurun_out/sto2/l0 python bench.py $B > gpurun_out/sto2/ncu.log 2>&1
echo done

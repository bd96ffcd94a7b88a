# stochastic 256^3: k_l0 with vs without the interface pass, and one ncu --set full capture of the
# k_l0 interior-tile launch (source-level stalls of the interface pass)
mkdir -p gpurun_out/sto
cd paper_2604_26518_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -shared -Xcompiler -fvisibility=hidden -I ../../include"
nvcc $F -DL0_NO_IFACE -o ../libgmt_noif.so gmt_api.cu gmt_fem.cpp > /dev/null 2>&1 &
cd ../..
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/sto/build.log 2>&1
wait
A="--res 256 --geometry stochastic --steps 5 --warmup 3 --no-cpu-baseline --no-like --no-batch --breakdown --no-solve"
timeout 300 python bench.py $A > gpurun_out/sto/def.json 2>gpurun_out/sto/def.err
GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_noif.so timeout 300 python bench.py $A > gpurun_out/sto/noif.json 2>gpurun_out/sto/noif.err
B="--res 256 --geometry stochastic --steps 1 --warmup 1 --no-cpu-baseline --no-like --no-batch --no-solve"
timeout 300 python bench.py $B > gpurun_out/sto/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l0 -s 6 -c 1 -o gpurun_out/sto/l0 python bench.py $B > gpurun_out/sto/ncu.log 2>&1
echo done

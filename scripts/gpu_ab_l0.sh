# A/B of the level-0 kernel: default vs no interface processing; gyroid and solid; ncu of k_l0
mkdir -p gpurun_out/ab
cd paper_2604_26518_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -shared -Xcompiler -fvisibility=hidden -I ../../include"
nvcc $F -DL0_NO_IFACE -o ../libgmt_noif.so gmt_api.cu gmt_fem.cpp > /dev/null 2>&1 &
cd ../..
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/ab/build.log 2>&1
wait
for g in gyroid solid; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown --no-solve --geometry $g > gpurun_out/ab/def_$g.json 2>gpurun_out/ab/def_$g.err
  GMT_LIB=$PWD/paper_2604_26518_b200/libgmt_noif.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown --no-solve --geometry $g > gpurun_out/ab/noif_$g.json 2>gpurun_out/ab/noif_$g.err
done
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ab/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_l0 -s 4 -c 1 -o gpurun_out/ab/l0 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ab/ncu.log 2>&1
echo done

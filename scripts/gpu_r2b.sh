mkdir -p gpurun_out/r2b
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/r2b/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "level0_vcycle_kernel" > gpurun_out/r2b/pytest_k.log 2>&1; echo "k rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2b/pytest.log 2>&1; echo "all rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown --no-solve > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo "bench rc=$?"

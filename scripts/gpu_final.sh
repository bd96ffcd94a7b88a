# final check of the tree: all GPU tests, smoke, default bench line
mkdir -p gpurun_out/fin
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/fin/build.log 2>&1
timeout 1500 python -m pytest tests/ -m gpu -q > gpurun_out/fin/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin/bench.json 2>gpurun_out/fin/bench.err
echo done

# full GPU test suite + smoke on the current tree
mkdir -p gpurun_out/${1:-t}
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/${1:-t}/build.log 2>&1
timeout 1500 python -m pytest tests/ -m gpu -q > gpurun_out/${1:-t}/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${1:-t}/smoke.log 2>&1
echo done

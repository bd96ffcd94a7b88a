# robustness sweep (scripts/config_sweep.py): odd / non-power-of-2 resolutions, both physics, slabs
mkdir -p gpurun_out/sw
python -c "from paper_2604_26518_b200 import build; build.build()" > gpurun_out/sw/build.log 2>&1
timeout 2400 python scripts/config_sweep.py > gpurun_out/sw/sweep.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sw/smoke.log 2>&1
echo done

#!/bin/bash
# usage: scripts/gpu_round.sh <tag> [steps...]; runs selected steps, logs under gpurun_out/<tag>/
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
for stepname in "$@"; do
  case $stepname in
    build) timeout 300 python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?" ;;
    test) timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    testall) timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench64) timeout 300 python bench.py --res 64 --steps 10 --warmup 3 --breakdown > $out/bench64.json 2> $out/bench64.err; echo "bench64 rc=$?" ;;
    bench128) timeout 300 python bench.py --res 128 --steps 10 --warmup 3 --breakdown > $out/bench128.json 2> $out/bench128.err; echo "bench128 rc=$?" ;;
    bench256) timeout 400 python bench.py --res 256 --steps 5 --warmup 3 --breakdown > $out/bench256.json 2> $out/bench256.err; echo "bench256 rc=$?" ;;
    bench) timeout 600 python bench.py --breakdown > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" ;;
    benchdef) timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "benchdef rc=$?" ;;
  esac
done

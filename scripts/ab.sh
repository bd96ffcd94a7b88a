#!/bin/bash
out=gpurun_out/$1; mkdir -p $out; shift
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for v in "$@"; do
  GMT_TILED_VARIANT=$v timeout 600 python bench.py --steps 5 --warmup 3 --breakdown --no-cpu-baseline > $out/bench_v$v.json 2> $out/bench_v$v.err; echo "v$v rc=$?"
done

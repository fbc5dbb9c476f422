#!/bin/bash
# One GPU development iteration (run through gpurun): build, GPU parity, the
# default bench line, and an ncu --set full capture of the mover / deposit on a
# C3-structure clone restricted to the timed steps.
# usage: tools/gpu_iter.sh TAG [extra bench args]
TAG=${1:-iter}; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { cat gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.log 2>&1
CMD="python bench.py --config c3 --c3-cells 96 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --graph 0 $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "bench_steps/" \
  -k regex:"mover_tiled|deposit_tiled" -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -n 2 gpurun_out/pytest_$TAG.log

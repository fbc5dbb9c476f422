#!/bin/bash
# One GPU iteration: build, GPU parity, bench, ncu of the fused kernel.
# usage: tools/gpu_iter.sh TAG [extra bench args]
TAG=${1:-iter}; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { cat gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"mover_tiled|deposit_tiled" -s 4 -c 3 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -n 2 gpurun_out/pytest_$TAG.log; grep '^{' gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.3e ms/step %.2f'%(d['value'],d['ms_per_step']), d['phase_ms'], 'frac %.3f'%d['roofline']['frac'])"

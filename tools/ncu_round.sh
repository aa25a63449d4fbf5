#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU). The bench command
# runs first without ncu; the launch-list pass profiles the SAME command.
# usage: tools/ncu_round.sh [tag]
set -u
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3"
timeout 600 $CMD > gpurun_out/bench_${TAG}.jsonl 2> gpurun_out/bench_${TAG}.err
echo "bench_rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref_${TAG}.jsonl 2> gpurun_out/bench_ref_${TAG}.err
echo "ref_rc=$?"
timeout 2000 ncu --metrics gpu__time_duration.sum --clock-control none -c 46000 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD --no-cpu-baseline > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo "launches_rc=$?"

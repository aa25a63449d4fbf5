#!/bin/bash
# Round-2 closing run (one GPU): GPU tests, smoke, the bench (both arms),
# a full small-config contraction through the bench, the eigensolver timings.
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.txt 2>&1
tail -3 gpurun_out/final/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
tail -2 gpurun_out/final/smoke.txt
timeout 300 python tools/eig_bench.py --sizes 1024 2048 4096 8192 > gpurun_out/final/eb.txt 2>&1
timeout 900 python bench.py > gpurun_out/final/bench.jsonl 2> gpurun_out/final/bench.err
tail -c 600 gpurun_out/final/bench.jsonl
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.jsonl 2> gpurun_out/final/bench_ref.err
tail -c 300 gpurun_out/final/bench_ref.jsonl
timeout 600 python bench.py --config c20 --prefix-steps 0 --no-cpu-baseline > gpurun_out/final/bench_c20_full.jsonl 2> gpurun_out/final/bench_c20.err
tail -c 400 gpurun_out/final/bench_c20_full.jsonl

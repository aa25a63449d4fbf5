#!/bin/bash
# ncu --set full of the final tridiagonalization kernels at p = 4096 (no CUDA
# graph above 2048 columns, so every launch is visible); plain run first.
mkdir -p gpurun_out/ncu2
EIG="python tools/eig_bench.py --sizes 4096"
MB_TRY_JACOBI_P=0 $EIG > gpurun_out/ncu2/plain.log 2>&1 || exit 1
MB_TRY_JACOBI_P=0 ncu --set full --clock-control none --import-source on -k regex:k_symv_tiles2 \
    -s 1500 -c 2 -o gpurun_out/ncu2/symv2 $EIG > gpurun_out/ncu2/symv2.log 2>&1
MB_TRY_JACOBI_P=0 ncu --set full --clock-control none --import-source on -k regex:k_trd_upd2 \
    -s 1500 -c 2 -o gpurun_out/ncu2/upd2 $EIG > gpurun_out/ncu2/upd2.log 2>&1
ls -la gpurun_out/ncu2

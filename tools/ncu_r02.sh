#!/bin/bash
# Round-2 ncu evidence (run under gpurun on ONE GPU; every ncu command is
# preceded by the same command line run plainly, exit 0):
#   full captures of the large-SVD kernels at p = 4096 (tools/eig_bench.py),
#   launch lists of the eigensolver at p = 2048 and of the bench command.
mkdir -p gpurun_out/ncu
EIG="python tools/eig_bench.py --sizes 4096"
$EIG > gpurun_out/ncu/plain_eig.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:k_symv_tiles \
    -s 3000 -c 2 -o gpurun_out/ncu/symv $EIG > gpurun_out/ncu/symv.log 2>&1
ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:k_gemm_cm \
    -s 30 -c 4 -o gpurun_out/ncu/gemm $EIG > gpurun_out/ncu/gemm.log 2>&1
ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:"k_trd_upd|k_trd_vec" \
    -s 3000 -c 2 -o gpurun_out/ncu/panel $EIG > gpurun_out/ncu/panel.log 2>&1
EIG2="python tools/eig_bench.py --sizes 2048"
$EIG2 > gpurun_out/ncu/plain_eig2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node -c 60000 --csv \
    --log-file gpurun_out/ncu/launches_eig2048.csv $EIG2 > gpurun_out/ncu/launches_eig.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/ncu/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node -c 60000 --csv \
    --log-file gpurun_out/ncu/launches_bench.csv $B > gpurun_out/ncu/launches_bench.log 2>&1
ls -la gpurun_out/ncu

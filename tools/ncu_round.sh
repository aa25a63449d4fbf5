#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; each ncu only after the same
# command exited 0 without ncu).
set -u
cd "${GRAFT_REPO_ROOT:-.}"
CMD="python tools/profile_run.py --config c20 --max-steps 120"
timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 4000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi_pair_cl \
    -s 20 -c 2 -o gpurun_out/prof_jacobi_pair $CMD > gpurun_out/ncu_full1.log 2>&1
echo "full_jacobi_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_svd_small \
    -s 2000 -c 2 -o gpurun_out/prof_svd_small $CMD > gpurun_out/ncu_full2.log 2>&1
echo "full_small_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm \
    -s 2000 -c 2 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_full3.log 2>&1
echo "full_gemm_rc=$?"
ls -la gpurun_out/

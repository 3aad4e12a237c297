#!/bin/bash
# ncu evidence for one round (run under gpurun from the repo root):
#   launch list of a two-grid step at cfg4, and --set full captures of the
#   subdomain-solve kernels (FDM and dense GEMM) and the residual kernel.
set -e
mkdir -p gpurun_out
python tools/run_once.py --what step --reps 2 > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_step.csv python tools/run_once.py --what step --reps 2 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dd_fdm -c 1 -o gpurun_out/prof_fdm \
    python tools/run_once.py --what sweep --reps 1 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_residual -c 1 -o gpurun_out/prof_k1 \
    python tools/run_once.py --what sweep --reps 1 > gpurun_out/ncu3.log 2>&1
HTG_FDM=0 python tools/run_once.py --what sweep --reps 1 > gpurun_out/plain_dense.log 2>&1
HTG_FDM=0 ncu --set full --clock-control none --import-source on -k regex:k_dd_gemm -c 1 -o gpurun_out/prof_gemm \
    python tools/run_once.py --what sweep --reps 1 > gpurun_out/ncu4.log 2>&1
echo done

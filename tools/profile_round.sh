#!/bin/bash
# ncu evidence for one round (run under gpurun from the repo root, one GPU):
#   launch lists (time + DRAM bytes) of a two-grid step and a coarse solve at cfg4,
#   and --set full captures of the top kernels. Each ncu command runs only after
#   the same command exited 0 without ncu.
set -e
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/run_once.py --what step --reps 2 > gpurun_out/plain_step.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_step.csv \
    python tools/run_once.py --what step --reps 2 > gpurun_out/ncu_step.log 2>&1
python tools/run_once.py --what sweep --reps 2 > gpurun_out/plain_sweep2.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_sweep.csv \
    python tools/run_once.py --what sweep --reps 2 > gpurun_out/ncu_sweep.log 2>&1
python tools/run_once.py --what coarse --reps 1 > gpurun_out/plain_coarse.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_coarse.csv \
    python tools/run_once.py --what coarse --reps 1 > gpurun_out/ncu_coarse.log 2>&1
python tools/run_once.py --what sweep --reps 1 > gpurun_out/plain_sweep.log 2>&1
for K in k_dd_fdm k1_cells k_dd_combine; do
  ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K -f \
      python tools/run_once.py --what sweep --reps 1 > gpurun_out/ncu_$K.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_nd_fwd_warp --launch-skip 1 -c 1 \
    -o gpurun_out/prof_k_nd_fwd_warp -f python tools/run_once.py --what coarse --reps 1 > gpurun_out/ncu_nd.log 2>&1
HTG_FDM=0 python tools/run_once.py --what sweep --reps 1 > gpurun_out/plain_dense.log 2>&1
HTG_FDM=0 ncu --set full --clock-control none --import-source on -k regex:k_dd_gemm -c 1 -o gpurun_out/prof_k_dd_gemm -f \
    python tools/run_once.py --what sweep --reps 1 > gpurun_out/ncu_gemm.log 2>&1
echo done

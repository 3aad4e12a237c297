#!/bin/bash
# ncu evidence for one round (run under gpurun from the repo root, one GPU):
#   launch lists (time + DRAM bytes) of a smoother sweep, a two-grid step and a
#   coarse solve at cfg4, and --set full captures of every kernel family. Each ncu
#   command runs only after the same command exited 0 without ncu.
set -e
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for W in sweep step coarse; do
  python tools/run_once.py --what $W --reps 2 > gpurun_out/plain_$W.log 2>&1
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
      python tools/run_once.py --what $W --reps 2 > gpurun_out/ncu_$W.log 2>&1
done
full() {  # name regex what [skip]
  ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip ${4:-0} -c 1 \
      -o gpurun_out/prof_$1 -f python tools/run_once.py --what $3 --reps 2 > gpurun_out/ncu_$1.log 2>&1
}
full k_dd_fdm_w k_dd_fdm_w sweep
# the same kernel at cfg3 (80 wavelengths: five 3-warp teams per SM)
python tools/run_once.py --what sweep --reps 2 --wavelengths 80 > gpurun_out/plain_sweep_cfg3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dd_fdm_w -c 1 -o gpurun_out/prof_k_dd_fdm_w_cfg3 -f \
    python tools/run_once.py --what sweep --reps 2 --wavelengths 80 > gpurun_out/ncu_k_dd_fdm_w_cfg3.log 2>&1
full k1_cells k1_cells sweep
full k_dd_combine k_dd_combine sweep
full k1_restrict k1_cells step 2
full k_prolong k_prolong step
full k_nd_fwd_warp k_nd_fwd_warp coarse 1
python tools/run_once.py --what capply --reps 2 > gpurun_out/plain_capply.log 2>&1
full k_coarse_apply k_coarse_apply capply
BAND_REPS=2 python tools/bench_band.py > gpurun_out/plain_band.log 2>&1
BAND_REPS=2 ncu --set full --clock-control none --import-source on -k regex:k_band_solve -c 1 \
    -o gpurun_out/prof_k_band_solve -f python tools/bench_band.py > gpurun_out/ncu_band.log 2>&1
HTG_FDM=0 python tools/run_once.py --what sweep --reps 1 > gpurun_out/plain_dense.log 2>&1
HTG_FDM=0 full k_dd_gemm k_dd_gemm sweep
echo done

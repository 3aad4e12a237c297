python tools/run_once.py --what sweep --reps 1 > gpurun_out/p_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dd_fdm_w -c 1 -o gpurun_out/prof_fdm_perm -f python tools/run_once.py --what sweep --reps 1 > gpurun_out/p1.log 2>&1

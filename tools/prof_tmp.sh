python tools/run_once.py --what sweep --reps 1 > gpurun_out/p_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_cells -c 1 -o gpurun_out/prof_k1_hmaj -f python tools/run_once.py --what sweep --reps 1 > gpurun_out/p1.log 2>&1

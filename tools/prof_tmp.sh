python tools/run_once.py --what capply --reps 2 > gpurun_out/p_plain2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_coarse_apply -c 1 -o gpurun_out/prof_k4 -f python tools/run_once.py --what capply --reps 1 > gpurun_out/p3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_prolong -c 1 -o gpurun_out/prof_k3b -f python tools/run_once.py --what prolong --reps 1 > gpurun_out/p4.log 2>&1

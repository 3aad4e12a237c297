SWEEP_LEAF=16,36,64,100,144 SWEEP_WARPF=96 SWEEP_MID=16384 python tools/coarse_sweep.py 160
SWEEP_LEAF=16 SWEEP_WARPF=64,128 SWEEP_MID=16384,65536 python tools/coarse_sweep.py 160
bash tools/nd_split_sweep.sh
